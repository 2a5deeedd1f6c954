"""Shared parity cases: each builds its inputs with the REFERENCE (oracle/_ref)
when available, and with this repo's host builders otherwise; the golden
fixtures pin that both produce identical bits (tests/golden/make_golden.py).

A case is a dict with geometry, channel list, layout, input slabs and the
run configuration (the SimulationConfig fields of solver.hpp:80-97).
"""
from __future__ import annotations

import hashlib
import math
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def solver_test_hash(ix, iy, iz, lo, hi):
    """hash_value of solver_test.cpp:26-36 (fixture helper of the reference
    tests; differs from config.hpp's hash_unit_value)."""
    m = (1 << 64) - 1
    h = 0x9E3779B97F4A7C15
    for v in (ix, iy, iz):
        h ^= ((v & m) + 0x9E3779B97F4A7C15 + ((h << 6) & m) + (h >> 2)) & m
        h = (h * 0xBF58476D1CE4E5B9) & m
        h ^= h >> 27
    unit = float(h >> 11) * 2.0 ** -53
    return lo + (hi - lo) * unit


# ---------------------------------------------------------------------------
# host construction (this repo's builders: numpy + libm exp)
# ---------------------------------------------------------------------------


def host_case(name: str):
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import synthetic as sy

    spec = CASES[name]
    dims, n = spec["dims"], spec["n"]
    lo, hi = spec["box"]
    dtype = np.float32 if spec.get("fp32") else np.float64
    geom = pd.GridGeometry.cell_centered_box(n, lo, hi, dims)
    if spec["geom"] == "ball":
        sdf = sy.ball_sdf_field(geom, spec["center"], spec["radius"], spec.get("sign", 1.0))
    elif spec["geom"] == "pack":
        pk = sy.SpherePacking.random((0, 0, 0), (1, 1, 1), *spec["pack"])
        sdf = pk.fluid_sdf_field(geom)
    else:
        raise ValueError(spec["geom"])
    channels = list(spec["channels"])
    grid = pd.build_sparse_grid(sdf, geom, pd.PhaseBand(), channels, dtype)
    prof = spec["profile"]
    if prof[0] == "anchored":
        p = pd.DiffusionProfile.anchored(*prof[1:])
    else:
        p = pd.DiffusionProfile(*prof)
    pd.populate_diffusion_channel(grid, p)
    act = grid.active_bool()
    u = grid.channel_data("u", writable=True)
    if spec["u0"][0] == "hash_unit":
        seed = spec["u0"][1]
        vals = np.array([pd.hash_unit_value(seed, int(f)) for f in grid.flat_indices()[act]])
    else:
        z = spec["u0"][1]
        idx = grid.node_indices()[act]
        vals = np.array([solver_test_hash(int(i[0]), int(i[1]), z if dims == 2 else int(i[2]), 0.0, 1.0)
                         for i in idx])
    u[act] = vals.astype(dtype)
    if "f" in channels:
        f = grid.channel_data("f", writable=True)
        idx = grid.node_indices()[act]
        f[act] = (0.5 + 0.25 * idx[:, 0].astype(np.float64)).astype(dtype)
    return grid


# ---------------------------------------------------------------------------
# reference construction (oracle/_ref)
# ---------------------------------------------------------------------------


def ref_case(name: str, R):
    spec = CASES[name]
    dims, n = spec["dims"], spec["n"]
    lo, hi = spec["box"]
    h = (hi - lo) / n
    size, sp, org = (n,) * dims, (h,) * dims, (lo + 0.5 * h,) * dims
    if spec["geom"] == "ball":
        sdf = R.field_ball(size, sp, org, spec["center"], spec["radius"], spec.get("sign", 1.0))
    else:
        c, r = R.sphere_packing((0, 0, 0), (1, 1, 1), *spec["pack"])
        sdf = R.field_sphere_pack(size, sp, org, c, r)
    tbytes = 4 if spec.get("fp32") else 8
    g = R.grid_from_sdf(size, sp, org, sdf, channels=spec["channels"], tbytes=tbytes)
    prof = spec["profile"]
    if prof[0] == "anchored":
        dmin, dmax, g2, anchor = prof[1:]
        g.populate_diffusion(dmin, dmax, -g2 * anchor, g2)
    else:
        g.populate_diffusion(*prof)
    if spec["u0"][0] == "hash_unit":
        g.fill_hash("u", spec["u0"][1])
    else:
        keys, masks = g.layout()
        u = g.prop("u")
        _fill_solver_hash(u, keys, masks, dims, spec["u0"][1])
        g.set_prop("u", u)
    if "f" in spec["channels"]:
        keys, masks = g.layout()
        f = g.prop("f")
        V = 512 if dims == 3 else 64
        for j in range(len(keys)):
            for off in range(V):
                if (int(masks[j, off >> 6]) >> (off & 63)) & 1:
                    x = (int(keys[j, 0]) << 3) | (off & 7)
                    f[j, off] = 0.5 + 0.25 * float(x)
        g.set_prop("f", f)
    return g


def _fill_solver_hash(u, keys, masks, dims, z0):
    V = 512 if dims == 3 else 64
    for j in range(len(keys)):
        for off in range(V):
            if (int(masks[j, off >> 6]) >> (off & 63)) & 1:
                ix = (int(keys[j, 0]) << 3) | (off & 7)
                iy = (int(keys[j, 1]) << 3) | ((off >> 3) & 7)
                iz = z0 if dims == 2 else ((int(keys[j, 2]) << 3) | (off >> 6))
                u[j, off] = solver_test_hash(ix, iy, iz, 0.0, 1.0)


def dt_of(spec, dmax):
    dims, n = spec["dims"], spec["n"]
    lo, hi = spec["box"]
    h = (hi - lo) / n
    inv = 0.0
    for _ in range(dims):
        inv += 1.0 / (h * h)
    return spec["dt_frac"] * (1.0 / (2.0 * dmax) / inv)


def oracle_config(spec, dt):
    from oracle.pyoracle import make_config
    r = spec.get("reaction", ("none",))
    kw = {}
    if r[0] == "surface_sink":
        kw = dict(reaction="surface_sink", rate=r[1], band_half_width=r[2])
    elif r[0] == "volumetric":
        kw = dict(reaction="volumetric", source_prop=spec["channels"].index(r[1]))
    bc = {f: ("dirichlet", v) for f, v in spec.get("dirichlet", {}).items()}
    return make_config(dt, spec["steps"], boundary_epsilon=spec.get("eps", 0.0), bc=bc,
                       record_every=spec.get("record", 1), **kw)


def time_factor(spec):
    r = spec.get("reaction", ("none",))
    if r[0] == "volumetric" and len(r) > 2 and r[2] == "exp":
        return lambda t: math.exp(-t)
    return None


def sim_config(spec, dt):
    from paper_2304_11165_b200 import porediff as pd
    cfg = pd.SimulationConfig()
    cfg.dt = dt
    cfg.n_steps = spec["steps"]
    cfg.record_every = spec.get("record", 1)
    cfg.boundary_epsilon = spec.get("eps", 0.0)
    r = spec.get("reaction", ("none",))
    if r[0] == "surface_sink":
        cfg.reaction = pd.ReactionSpec.surface_sink(r[1], r[2])
    elif r[0] == "volumetric":
        cfg.reaction = pd.ReactionSpec.volumetric(r[1], time_factor(spec))
    for f, v in spec.get("dirichlet", {}).items():
        cfg.outer_bc[f] = pd.FaceBc.dirichlet(v)
    return cfg


SOLVER = ["phi", "u", "D", "u_next"]

CASES = {
    # BASELINE.json configs[0] / SURVEY §8d C1: 64^3, pore outside a ball,
    # sigmoid D{0,1,0,1}, u0 = hash_unit_value(1, flat), 1000 steps no-flux.
    "c1_ball64": dict(dims=3, n=64, box=(0.0, 1.0), geom="ball", center=(0.5, 0.5, 0.5), radius=0.3,
                      sign=-1.0, channels=SOLVER, profile=(0.0, 1.0, 0.0, 1.0), u0=("hash_unit", 1),
                      dt_frac=0.4, steps=1000, record=1000),
    # SURVEY §8a contract check: 40^3 sphere pack (n not a multiple of 8),
    # walls via boundary_epsilon, surface sink, two Dirichlet faces.
    "contract40": dict(dims=3, n=40, box=(0.0, 1.0), geom="pack", pack=(30, 0.08, 0.16, 777),
                       channels=SOLVER, profile=("anchored", 0.05, 0.95, 160.0, 0.02), u0=("hash_unit", 5),
                       eps=0.5 / 40, reaction=("surface_sink", 3.0, 1.5), dirichlet={0: 1.0, 5: 0.25},
                       dt_frac=0.45, steps=300, record=50),
    # solver_test.cpp disk_grid(24) (:40-53) with the determinism test's sink
    # (:427-452): 2-D, record every 10.
    "disk24_sink": dict(dims=2, n=24, box=(-1.0, 1.0), geom="ball", center=(0.0, 0.0), radius=0.8,
                        channels=SOLVER, profile=(0.05, 1.0, 0.0, 16.0), u0=("solver_hash", 0),
                        reaction=("surface_sink", 0.4, 1.5), dt_frac=0.45, steps=150, record=10),
    # volumetric source with time factor exp(-t) (solver_test.cpp:265-286,
    # verification.hpp:229-231), 2-D, Dirichlet on the high-y face.
    "disk20_volumetric": dict(dims=2, n=20, box=(-1.0, 1.0), geom="ball", center=(0.1, -0.05),
                              radius=0.75, channels=SOLVER + ["f"], profile=(0.05, 1.0, 0.0, 16.0),
                              u0=("solver_hash", 1), reaction=("volumetric", "f", "exp"),
                              dirichlet={3: 0.5}, dt_frac=0.4, steps=60, record=7),
    # FP32 mode (solver_test.cpp:611-646)
    "disk24_fp32": dict(dims=2, n=24, box=(-1.0, 1.0), geom="ball", center=(0.0, 0.0), radius=0.8,
                        channels=SOLVER, profile=(0.05, 1.0, 0.0, 16.0), u0=("solver_hash", 2), fp32=True,
                        dt_frac=0.4, steps=200, record=20),
    # 3-D pack with a sink band and a non-multiple-of-8 box, FP32
    "pack27_fp32": dict(dims=3, n=27, box=(0.0, 1.0), geom="pack", pack=(12, 0.1, 0.2, 31),
                        channels=SOLVER, profile=("anchored", 0.1, 1.0, 100.0, 0.03), u0=("hash_unit", 9),
                        fp32=True, reaction=("surface_sink", 1.0, 2.0), dirichlet={2: 0.75}, dt_frac=0.45,
                        steps=80, record=20),
}
