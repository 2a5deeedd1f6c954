"""The FP32 march kernel (pd_march32.cu; the reference's T = float path,
solver.hpp:385-455 in float) and the FP64 march kernel's uniform-chunk path
against the reference run in-process on the same inputs: u, u_next and every diagnostics row bit for bit, on grids with many
chunks per warp — sink band, volumetric source with a time factor, walls,
Dirichlet faces — and the non-finite error path (message and post-error
state). conftest.py sets PD_MARCH_MIN_CHUNKS=0, so every 3-D FP32 step here
runs the march kernel."""
import numpy as np
import pytest

import cases
from cases import dt_of, oracle_config, sim_config, time_factor

pytestmark = pytest.mark.gpu

SPECS = {
    "pack61_fp32_vol": dict(dims=3, n=61, box=(0.0, 1.0), geom="pack", pack=(40, 0.06, 0.14, 91),
                            channels=["phi", "u", "D", "u_next", "f"], profile=(0.05, 1.0, 0.0, 60.0),
                            u0=("hash_unit", 4), fp32=True, reaction=("volumetric", "f", "exp"), dt_frac=0.45,
                            steps=40, record=8),
    # steep sigmoid: D saturates exactly, most chunks take the uniform path
    "pack64_fp32_unif": dict(dims=3, n=64, box=(0.0, 1.0), geom="pack", pack=(6, 0.05, 0.09, 3),
                             channels=["phi", "u", "D", "u_next"], profile=(0.05, 1.0, 0.0, 4000.0),
                             u0=("hash_unit", 2), fp32=True, reaction=("surface_sink", 1.5, 1.0), dt_frac=0.45,
                             steps=40, record=10),
    "pack56_fp32_walls": dict(dims=3, n=56, box=(0.0, 1.0), geom="pack", pack=(30, 0.07, 0.15, 12),
                              channels=["phi", "u", "D", "u_next"], profile=("anchored", 0.05, 0.95, 200.0, 0.02),
                              u0=("hash_unit", 6), fp32=True, eps=0.5 / 56, reaction=("surface_sink", 2.0, 1.0),
                              dirichlet={0: 1.0, 5: 0.25}, dt_frac=0.45, steps=60, record=60),
}


@pytest.fixture
def spec_cases(monkeypatch):
    for k, v in SPECS.items():
        monkeypatch.setitem(cases.CASES, k, v)
    return cases.CASES


def _compare(ours, g, res, rows):
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u) for d in res.diagnostics]
    for c in ("u", "u_next"):
        a, b = ours.channel_data(c), g.prop(c)
        assert a.dtype == np.float32
        diff = np.nonzero(a.view(np.uint32) != b.view(np.uint32))
        assert diff[0].size == 0, (c, diff[0][:5], diff[1][:5], a[diff][:5], b[diff][:5])


@pytest.mark.parametrize("name", list(SPECS))
def test_fp32_march_equals_reference(name, spec_cases, ref, cuda):
    from paper_2304_11165_b200 import porediff as pd
    spec = spec_cases[name]
    g = cases.ref_case(name, ref)
    keys, masks = g.layout()
    assert len(keys) > 200  # many chunks per launch
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = dt_of(spec, g.max_diffusivity())
    geom = pd.GridGeometry.cell_centered_box(spec["n"], *spec["box"], spec["dims"])
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data, np.float32)
    code, msg, rows = g.run(oracle_config(spec, dt), time_factor(spec))
    assert code == 0, msg
    res = pd.run_simulation(ours, sim_config(spec, dt))
    _compare(ours, g, res, rows)


def test_fp32_march_nonfinite_error_and_state(spec_cases, ref, cuda):
    """An overflow mid-run: same numeric_error text (first step, lowest
    ordinal node) and the same post-error u / u_next as the reference."""
    from paper_2304_11165_b200 import porediff as pd
    name = "pack56_fp32_walls"
    spec = dict(spec_cases[name])
    g = cases.ref_case(name, ref)
    keys, masks = g.layout()
    u = g.prop("u")
    act = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(len(masks), -1).astype(bool)
    j, off = [int(v[len(v) // 2]) for v in np.nonzero(act)]
    u[j, off] = np.float32(3e38)
    g.set_prop("u", u)
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = 3.0 * dt_of(spec, g.max_diffusivity())
    spec["steps"] = 30
    ocfg = oracle_config(spec, dt)
    ocfg.enforce_stability = 0
    code, msg, _ = g.run(ocfg, None)
    assert code == 6, msg
    geom = pd.GridGeometry.cell_centered_box(spec["n"], *spec["box"], spec["dims"])
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data, np.float32)
    cfg = sim_config(spec, dt)
    cfg.enforce_stability = False
    with pytest.raises(pd.NumericError) as ei:
        pd.run_simulation(ours, cfg)
    assert str(ei.value) == msg
    for c in ("u", "u_next"):
        assert np.array_equal(ours.channel_data(c).view(np.uint32), g.prop(c).view(np.uint32)), c


# FP64 march: uniform chunks (kFlagUnif — every node fluid, one D_eff value in
# the chunk and its six neighbours) load no D_eff and use (dv + dv) * 0.5 for
# every face. A steep sigmoid saturates D to exactly d_min + d_max a few cells
# from the interface, so most chunks of a coarse-grained pack are uniform.
SPECS64 = {
    "pack64_unif_sink": dict(dims=3, n=64, box=(0.0, 1.0), geom="pack", pack=(6, 0.05, 0.09, 3),
                             channels=["phi", "u", "D", "u_next"], profile=(0.05, 1.0, 0.0, 4000.0),
                             u0=("hash_unit", 2), reaction=("surface_sink", 1.5, 1.0), dt_frac=0.45,
                             steps=40, record=10),
    "pack64_unif_vol": dict(dims=3, n=64, box=(0.0, 1.0), geom="pack", pack=(6, 0.05, 0.09, 5),
                            channels=["phi", "u", "D", "u_next", "f"], profile=(0.1, 2.0, 0.0, 4000.0),
                            u0=("hash_unit", 8), reaction=("volumetric", "f", "exp"), dirichlet={1: 0.5},
                            dt_frac=0.45, steps=30, record=30),
}


@pytest.mark.parametrize("name", list(SPECS64))
def test_fp64_uniform_chunks_equal_reference(name, monkeypatch, ref, cuda):
    from paper_2304_11165_b200 import porediff as pd
    for k, v in SPECS64.items():
        monkeypatch.setitem(cases.CASES, k, v)
    spec = cases.CASES[name]
    g = cases.ref_case(name, ref)
    keys, masks = g.layout()
    D = g.prop("D")
    full = np.all(masks == np.uint64(0xFFFFFFFFFFFFFFFF), axis=1)
    assert (full & (D.min(axis=1) == D.max(axis=1))).mean() > 0.3  # plenty of uniform chunks
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = dt_of(spec, g.max_diffusivity())
    geom = pd.GridGeometry.cell_centered_box(spec["n"], *spec["box"], spec["dims"])
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data)
    code, msg, rows = g.run(oracle_config(spec, dt), time_factor(spec))
    assert code == 0, msg
    res = pd.run_simulation(ours, sim_config(spec, dt))
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u) for d in res.diagnostics]
    for c in ("u", "u_next"):
        a, b = ours.channel_data(c), g.prop(c)
        diff = np.nonzero(a.view(np.uint64) != b.view(np.uint64))
        assert diff[0].size == 0, (c, diff[0][:5], diff[1][:5], a[diff][:5], b[diff][:5])


def test_fp64_uniform_chunk_nonfinite_error_and_state(monkeypatch, ref, cuda):
    """An overflow that starts inside a uniform chunk (the rare path runs with
    the chunk's dv instead of D_eff from the ring): same numeric_error text
    and post-error u / u_next as the reference."""
    from paper_2304_11165_b200 import porediff as pd
    for k, v in SPECS64.items():
        monkeypatch.setitem(cases.CASES, k, v)
    name = "pack64_unif_sink"
    spec = dict(cases.CASES[name])
    g = cases.ref_case(name, ref)
    keys, masks = g.layout()
    D = g.prop("D")
    full = np.all(masks == np.uint64(0xFFFFFFFFFFFFFFFF), axis=1)
    uni = np.nonzero(full & (D.min(axis=1) == D.max(axis=1)) & np.all(keys > 0, axis=1)
                     & np.all(keys < 7, axis=1))[0]
    j = int(uni[len(uni) // 2])
    u = g.prop("u")
    u[j, 9 * 64 // 2 + 3] = 1e300
    g.set_prop("u", u)
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = 3.0 * dt_of(spec, g.max_diffusivity())
    spec["steps"] = 40
    ocfg = oracle_config(spec, dt)
    ocfg.enforce_stability = 0
    code, msg, _ = g.run(ocfg, None)
    assert code == 6, msg
    geom = pd.GridGeometry.cell_centered_box(spec["n"], *spec["box"], spec["dims"])
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data)
    cfg = sim_config(spec, dt)
    cfg.enforce_stability = False
    with pytest.raises(pd.NumericError) as ei:
        pd.run_simulation(ours, cfg)
    assert str(ei.value) == msg
    for c in ("u", "u_next"):
        assert np.array_equal(ours.channel_data(c).view(np.uint64), g.prop(c).view(np.uint64)), c


def test_fp64_march_128_pack_equals_reference(monkeypatch, ref, cuda):
    """A C5-shaped case at 128^3 (overlapping spheres, sigmoid D with exact
    saturation, surface sink): thousands of chunks through the march kernel's
    claim pipeline, uniform and generic chunks mixed, against the reference."""
    from paper_2304_11165_b200 import porediff as pd
    spec = dict(dims=3, n=128, box=(0.0, 1.0), geom="pack", pack=(60, 0.04, 0.09, 2048),
                channels=["phi", "u", "D", "u_next"], profile=(0.0, 1.0, 0.0, 512.0), u0=("hash_unit", 1),
                reaction=("surface_sink", 1.0, 1.0), dt_frac=0.4, steps=30, record=15)
    monkeypatch.setitem(cases.CASES, "pack128", spec)
    g = cases.ref_case("pack128", ref)
    keys, masks = g.layout()
    assert len(keys) > 2000
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = dt_of(spec, g.max_diffusivity())
    geom = pd.GridGeometry.cell_centered_box(128, 0.0, 1.0, 3)
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data)
    code, msg, rows = g.run(oracle_config(spec, dt), None)
    assert code == 0, msg
    res = pd.run_simulation(ours, sim_config(spec, dt))
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u) for d in res.diagnostics]
    for c in ("u", "u_next"):
        assert np.array_equal(ours.channel_data(c).view(np.uint64), g.prop(c).view(np.uint64)), c


@pytest.mark.parametrize("dtype,n", [(np.float64, 48), (np.float32, 40), (np.float64, 37)])
def test_free_box_dense_kernel_equals_reference(dtype, n, ref, cuda, monkeypatch):
    """A free box (every node active and fluid, one D, no-flux box — the FRAP
    fit's probes): interior chunks take the uniform path, box-boundary chunks
    the generic one (n = 37: partial chunks); equal to the reference."""
    from paper_2304_11165_b200 import porediff as pd
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    sdf = np.ones(n ** 3)
    rg = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf, tbytes=np.dtype(dtype).itemsize)
    keys, masks = rg.layout()
    D = np.full((len(keys), 512), 0.7, dtype)
    rg.set_prop("D", D)
    rg.fill_hash("u", 5)
    data = {c: rg.prop(c) for c in pd.solver_channels()}
    dt = 0.45 * pd.stability_dt(geom, 0.7)
    ours = pd.SparseBlockGrid.from_layout(geom, pd.solver_channels(), keys, masks, data, dtype)
    from oracle.pyoracle import make_config
    code, msg, rows = rg.run(make_config(dt, 25, record_every=5), None)
    assert code == 0, msg
    cfg = pd.SimulationConfig(dt=dt, n_steps=25, record_every=5)
    res = pd.run_simulation(ours, cfg)
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u) for d in res.diagnostics]
    view = np.uint64 if dtype == np.float64 else np.uint32
    for c in ("u", "u_next"):
        assert np.array_equal(ours.channel_data(c).view(view), rg.prop(c).view(view)), c


@pytest.mark.parametrize("dtype,tiny", [(np.float64, 1e-310), (np.float32, 1e-39)])
def test_subnormal_diffusivity_disables_halving_and_stays_exact(dtype, tiny, monkeypatch, ref, cuda):
    """A fluid node with a subnormal D: halving D_eff would not be exact, so
    the plan keeps D unhalved (plan.half = false); results still equal the
    reference bit for bit."""
    from paper_2304_11165_b200 import porediff as pd
    spec = dict(dims=3, n=40, box=(0.0, 1.0), geom="pack", pack=(20, 0.05, 0.12, 9),
                channels=["phi", "u", "D", "u_next"], profile=(0.05, 1.0, 0.0, 160.0), u0=("hash_unit", 3),
                fp32=dtype == np.float32, reaction=("surface_sink", 1.0, 1.0), dt_frac=0.4, steps=12, record=4)
    monkeypatch.setitem(cases.CASES, "tinyD", spec)
    g = cases.ref_case("tinyD", ref)
    keys, masks = g.layout()
    D = g.prop("D")
    phi = g.prop("phi")
    act = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(len(masks), -1).astype(bool)
    j, off = [int(v[len(v) // 2]) for v in np.nonzero(act & (phi > 0.05))]
    D[j, off] = dtype(tiny)
    g.set_prop("D", D)
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = dt_of(spec, g.max_diffusivity())
    geom = pd.GridGeometry.cell_centered_box(40, 0.0, 1.0, 3)
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data, dtype)
    code, msg, rows = g.run(oracle_config(spec, dt), None)
    assert code == 0, msg
    res = pd.run_simulation(ours, sim_config(spec, dt))
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u) for d in res.diagnostics]
    view = np.uint64 if dtype == np.float64 else np.uint32
    for c in ("u", "u_next"):
        assert np.array_equal(ours.channel_data(c).view(view), g.prop(c).view(view)), c
