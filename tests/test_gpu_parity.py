"""GPU parity: the sm_100a FTCS path, driven through the C ABI (via the Python
mirror of the reference API), reproduces the reference bit for bit — fields
u and u_next, and every diagnostics row — on all golden cases."""
import math

import numpy as np
import pytest

from cases import CASES, dt_of, host_case, oracle_config, sha, sim_config, time_factor

pytestmark = pytest.mark.gpu


def _row_hex(d):
    return [int(d.step), float(d.time).hex(), float(d.total_mass).hex(), float(d.min_u).hex(),
            float(d.max_u).hex()]


def _first_diff(a, b):
    a = np.ascontiguousarray(a).reshape(-1)
    b = np.ascontiguousarray(b).reshape(-1)
    bad = np.nonzero(a.view(np.uint8 if a.dtype.itemsize == 1 else (np.uint64 if a.dtype.itemsize == 8 else np.uint32))
                     != b.view(np.uint64 if b.dtype.itemsize == 8 else np.uint32))[0]
    return bad[:5], a[bad[:5]], b[bad[:5]]


@pytest.mark.parametrize("name", list(CASES))
def test_run_simulation_bitwise_equal_to_reference(name, golden, cuda):
    from paper_2304_11165_b200 import porediff as pd
    spec, gold = CASES[name], golden[name]
    grid = host_case(name)
    dt = float.fromhex(gold["dt"])
    assert pd.max_diffusivity(grid) == float.fromhex(gold["dmax"])
    cfg = sim_config(spec, dt)
    res = pd.run_simulation(grid, cfg)
    assert [_row_hex(d) for d in res.diagnostics] == gold["rows"]
    u = grid.channel_data("u")
    un = grid.channel_data("u_next")
    assert sha(u) == gold["sha_outputs"]["u"], _first_diff(u, u)
    assert sha(un) == gold["sha_outputs"]["u_next"]


@pytest.mark.parametrize("name", ["contract40", "pack27_fp32", "disk24_sink"])
def test_against_reference_arrays(name, ref, cuda):
    """Full-array comparison with the reference run in the same process
    (oracle/_ref travels to the GPU box as a prebuilt .so)."""
    from cases import ref_case
    from paper_2304_11165_b200 import porediff as pd
    spec = CASES[name]
    g = ref_case(name, ref)
    keys, masks = g.layout()
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = dt_of(spec, g.max_diffusivity())
    geom = pd.GridGeometry.cell_centered_box(spec["n"], *spec["box"], spec["dims"])
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data, g.dtype)
    code, msg, rows = g.run(oracle_config(spec, dt), time_factor(spec))
    assert code == 0, msg
    res = pd.run_simulation(ours, sim_config(spec, dt))
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u)
                                        for d in res.diagnostics]
    for c in ("u", "u_next"):
        a, b = ours.channel_data(c), g.prop(c)
        bits = a.dtype.itemsize * 8
        view = np.uint64 if bits == 64 else np.uint32
        diff = np.nonzero(a.view(view) != b.view(view))
        assert diff[0].size == 0, (c, diff[0][:5], diff[1][:5], a[diff][:5], b[diff][:5])


def test_segmented_runs_equal_one_run(cuda, golden):
    """Observers force per-record segments; results must not change."""
    from paper_2304_11165_b200 import porediff as pd
    name = "contract40"
    spec, gold = CASES[name], golden[name]
    grid = host_case(name)
    cfg = sim_config(spec, float.fromhex(gold["dt"]))
    seen = []
    pd.run_simulation(grid, cfg, [lambda g, d: seen.append((d.step, g.get((20, 20, 3), "u")))])
    assert [s for s, _ in seen] == [int(r[0]) for r in gold["rows"]]
    assert sha(grid.channel_data("u")) == gold["sha_outputs"]["u"]


def test_ftcs_step_sequence_equals_run(cuda, golden):
    """ftcs_step (solver.hpp:470-475) repeated == run_simulation (no gate)."""
    from paper_2304_11165_b200 import porediff as pd
    name = "disk24_sink"
    spec, gold = CASES[name], golden[name]
    grid = host_case(name)
    cfg = sim_config(spec, float.fromhex(gold["dt"]))
    for s in range(spec["steps"]):
        d = pd.ftcs_step(grid, cfg, s)
        assert d.step == s + 1
    assert sha(grid.channel_data("u")) == gold["sha_outputs"]["u"]


def test_error_messages_match_oracle(cuda, port):
    """numeric_error / stability_error / input_error text and codes equal the
    plain-C oracle (itself pinned to the reference by test_oracle.py)."""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import porediff as pd
    base = host_case("disk24_sink")
    keys, masks = base.keys(), base.masks()
    props = {c: base.channel_data(c).copy() for c in ("phi", "u", "D", "u_next")}
    act = base.active_bool()
    j, off = [int(v[len(v) // 2]) for v in np.nonzero(act)]
    props["u"][j, off] = np.inf
    h = 2.0 / 24
    dmax = float(props["D"][base.active_bool()].max())
    bound = pd.stability_dt(base.geom, dmax)
    cases = [(0.3 * bound, 5, {}), (10 * bound, 5, {}), (bound, 5, {}), (-1.0, 5, {}),
             (0.3 * bound, 0, {}), (0.3 * bound, 5, {"reaction": "surface_sink", "rate": -1.0})]
    for dt, n, kw in cases:
        ocfg = make_config(dt, n, **kw)
        pc, pmsg, _, pu, pun = port.run((24, 24), (h, h), keys, masks, props["phi"], props["u"], props["D"],
                                        props["u_next"], ocfg)
        g = pd.SparseBlockGrid.from_layout(base.geom, pd.solver_channels(), keys, masks, props)
        cfg = pd.SimulationConfig(dt=dt, n_steps=n)
        if kw:
            cfg.reaction = pd.ReactionSpec.surface_sink(kw["rate"])
        with pytest.raises(pd.PorediffError) as ei:
            pd.run_simulation(g, cfg)
        kind = {1: pd.InputError, 5: pd.StabilityError, 6: pd.NumericError}[pc]
        assert isinstance(ei.value, kind), (ei.value, pc, pmsg)
        assert str(ei.value) == pmsg
        if pc == 6:  # state left exactly as the reference leaves it
            assert np.array_equal(g.channel_data("u").view(np.uint64), pu.view(np.uint64))
            assert np.array_equal(g.channel_data("u_next").view(np.uint64), pun.view(np.uint64))


def test_nonfinite_after_several_steps_keeps_state(cuda, port):
    """A value that overflows mid-run: the error names the first step and the
    lowest-ordinal node, earlier steps' swaps stay applied."""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import porediff as pd
    base = host_case("disk24_sink")
    keys, masks = base.keys(), base.masks()
    props = {c: base.channel_data(c).copy() for c in ("phi", "u", "D", "u_next")}
    act = base.active_bool()
    j, off = [int(v[len(v) // 3]) for v in np.nonzero(act)]
    props["u"][j, off] = 1e300
    h = 2.0 / 24
    dt = 0.9 * pd.stability_dt(base.geom, float(props["D"][base.active_bool()].max()))
    ocfg = make_config(dt * 3.0, 40, enforce_stability=False)  # unstable: grows until overflow
    pc, pmsg, prows, pu, pun = port.run((24, 24), (h, h), keys, masks, props["phi"], props["u"], props["D"],
                                        props["u_next"], ocfg)
    assert pc == 6, pmsg
    g = pd.SparseBlockGrid.from_layout(base.geom, pd.solver_channels(), keys, masks, props)
    cfg = pd.SimulationConfig(dt=dt * 3.0, n_steps=40, enforce_stability=False)
    with pytest.raises(pd.NumericError) as ei:
        pd.run_simulation(g, cfg)
    assert str(ei.value) == pmsg
    assert np.array_equal(g.channel_data("u").view(np.uint64), pu.view(np.uint64))
    assert np.array_equal(g.channel_data("u_next").view(np.uint64), pun.view(np.uint64))


def test_device_sphere_pack_builder_matches_reference_builder(cuda, ref):
    """north_star subsystem 1: block activation, indexing, masks and phi are
    bit-exact against build_sparse_grid(field_from(pack.fluid_sdf))."""
    from paper_2304_11165_b200 import porediff as pd
    for n, args, dtype in [(40, (30, 0.08, 0.16, 777), np.float64), (37, (60, 0.03, 0.12, 5), np.float64),
                           (33, (20, 0.1, 0.2, 8), np.float32)]:
        geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
        c, r = ref.sphere_packing((0, 0, 0), (1, 1, 1), *args)
        sdf = ref.field_sphere_pack(geom.size, geom.spacing, geom.origin, c, r)
        g = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf, tbytes=np.dtype(dtype).itemsize)
        dev = pd.DeviceGrid.sphere_pack(geom, c, r, dtype=dtype)
        keys, masks = dev.layout()
        rk, rm = g.layout()
        assert np.array_equal(keys, rk) and np.array_equal(masks, rm)
        phi = dev.download(0)
        assert np.array_equal(phi, g.prop("phi"))
        assert dev.info()[1] == g.active_count()
        dev.close()


def test_device_fill_hash_matches_reference(cuda, ref):
    from cases import ref_case
    from paper_2304_11165_b200 import porediff as pd
    g = ref_case("contract40", ref)
    keys, masks = g.layout()
    geom = pd.GridGeometry.cell_centered_box(40, 0.0, 1.0, 3)
    dev = pd.DeviceGrid.create(geom, np.float64, keys, masks, 4)
    dev.fill_hash(1, 5)
    assert np.array_equal(dev.download(1), g.prop("u"))
    dev.close()


@pytest.mark.parametrize("seed", range(6))
def test_random_packs_and_bands_builder_matches_reference(seed, cuda, ref):
    """Seeded random sphere packs with random phase bands (including bands
    that exclude the pore space's far field), FP64 / FP32, odd box sizes:
    keys, masks, phi and the active count equal the reference builder's."""
    from paper_2304_11165_b200 import porediff as pd
    r = np.random.default_rng(77 + seed)
    n = int(r.integers(17, 50))
    dtype = np.float32 if seed % 2 else np.float64
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    c, rad = ref.sphere_packing((0, 0, 0), (1, 1, 1), int(r.integers(5, 60)), 0.03, float(r.uniform(0.08, 0.25)),
                                int(r.integers(1, 10 ** 6)))
    b_low = float(r.choice([0.0, -0.05, 0.02]))
    b_up = float(r.choice([np.inf, 0.1, 0.3]))
    sdf = ref.field_sphere_pack(geom.size, geom.spacing, geom.origin, c, rad)
    g = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf, b_low, b_up, tbytes=np.dtype(dtype).itemsize)
    dev = pd.DeviceGrid.sphere_pack(geom, c, rad, pd.PhaseBand(b_low, b_up), dtype=dtype)
    keys, masks = dev.layout()
    rk, rm = g.layout()
    assert np.array_equal(keys, rk) and np.array_equal(masks, rm)
    assert np.array_equal(dev.download(0), g.prop("phi"))
    assert dev.info()[1] == g.active_count()
    dev.close()
