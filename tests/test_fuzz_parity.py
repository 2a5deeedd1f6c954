"""Seeded random configurations through run_simulation on the B200 against
the reference run in-process on identical inputs: geometry (ball or sphere
pack, box not a multiple of 8), rank (2-D / 3-D), scalar type, diffusion
profile (plain or anchored sigmoid, steep enough for uniform chunks or not),
boundary epsilon (walls), reaction (none / surface sink / volumetric with
exp(-t)), Dirichlet faces and values, record interval. Every u / u_next bit
and every diagnostics row must match. conftest.py forces the march kernels
for 3-D grids; 2-D grids take the tile kernel."""
import numpy as np
import pytest

import cases
from cases import dt_of, oracle_config, sim_config, time_factor

pytestmark = pytest.mark.gpu


def _spec(seed):
    r = np.random.default_rng(seed)
    dims = int(r.choice([2, 3], p=[0.3, 0.7]))
    n = int(r.integers(17, 45) if dims == 3 else r.integers(20, 70))
    fp32 = bool(r.random() < 0.35)
    chans = ["phi", "u", "D", "u_next"]
    spec = dict(dims=dims, n=n, box=(0.0, 1.0), channels=chans, u0=("hash_unit", int(r.integers(1, 99))),
                fp32=fp32, dt_frac=float(r.uniform(0.2, 0.49)), steps=int(r.integers(5, 40)))
    spec["record"] = int(r.integers(1, spec["steps"] + 1))
    if dims == 3 and r.random() < 0.7:
        spec.update(geom="pack", pack=(int(r.integers(4, 40)), 0.05, float(r.uniform(0.1, 0.25)),
                                       int(r.integers(1, 10 ** 6))))
    else:
        c = tuple(float(v) for v in r.uniform(0.35, 0.65, dims))
        spec.update(geom="ball", center=c, radius=float(r.uniform(0.2, 0.4)), sign=float(r.choice([-1.0, 1.0])))
    if r.random() < 0.5:
        spec["profile"] = (float(r.uniform(0.0, 0.2)), float(r.uniform(0.5, 2.0)), 0.0,
                           float(r.choice([1.0, 8.0 * n, 400.0 * n])))
    else:
        spec["profile"] = ("anchored", 0.05, 0.95, float(r.uniform(2.0, 40.0)) * n, 0.02)
    if r.random() < 0.4:
        spec["eps"] = float(r.uniform(0.0, 1.5)) / n
    kind = r.choice(["none", "sink", "vol"], p=[0.35, 0.4, 0.25])
    if kind == "sink":
        spec["reaction"] = ("surface_sink", float(r.uniform(0.1, 5.0)), float(r.uniform(0.5, 2.5)))
    elif kind == "vol":
        spec["channels"] = chans + ["f"]
        spec["reaction"] = ("volumetric", "f", "exp")
    faces = [f for f in range(2 * dims) if r.random() < 0.25]
    spec["dirichlet"] = {f: float(r.uniform(0.0, 1.0)) for f in faces}
    return spec


@pytest.mark.parametrize("seed", range(48))
def test_random_configuration_equals_reference(seed, monkeypatch, ref, cuda):
    from paper_2304_11165_b200 import porediff as pd
    spec = _spec(1000 + seed)
    name = f"fuzz{seed}"
    monkeypatch.setitem(cases.CASES, name, spec)
    g = cases.ref_case(name, ref)
    keys, masks = g.layout()
    dtype = np.float32 if spec["fp32"] else np.float64
    data = {c: g.prop(c) for c in spec["channels"]}
    dt = dt_of(spec, g.max_diffusivity())
    geom = pd.GridGeometry.cell_centered_box(spec["n"], *spec["box"], spec["dims"])
    ours = pd.SparseBlockGrid.from_layout(geom, spec["channels"], keys, masks, data, dtype)
    code, msg, rows = g.run(oracle_config(spec, dt), time_factor(spec))
    assert code == 0, (spec, msg)
    res = pd.run_simulation(ours, sim_config(spec, dt))
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u)
                                        for d in res.diagnostics], spec
    view = np.uint32 if spec["fp32"] else np.uint64
    for c in ("u", "u_next"):
        a, b = ours.channel_data(c), g.prop(c)
        diff = np.nonzero(a.view(view) != b.view(view))
        assert diff[0].size == 0, (spec, c, diff[0][:5], diff[1][:5])
