"""Parity on the exact headline (bench) configuration, and of the device
D(phi) (VERDICT r1 "next" item 1).

The bench (bench.py, BASELINE.json configs[4]) builds on the device: a
2048^3 cell-centred box on [0,1]^3, pore space = complement of
pack_for_porosity(0.2, 128/2048, 12345), D from DiffusionProfile(0, 1, 0,
4*2048) (geometry.hpp:182-206), u0 = hash_unit_value(1, flat), surface sink
k = 1, w = 1, dt = 0.4 * stability bound. Here a [0, E)^3 crop of that
geometry (same spheres, same spacing and origin; the crop's faces are the box
faces) goes through the device builder, the device D, the device hash fill
and the march kernel, and the unmodified reference (oracle/_ref) runs the same
crop from its own SDF (field_from over the spheres that can reach the crop,
selected exactly), builder, populate_diffusion_channel (glibc exp) and
run_simulation. Everything is compared bit for bit.
"""
import math

import numpy as np
import pytest

N_BOX = 2048
PSI, R_VOX, SEED = 0.2, 128.0, 12345


def bench_spheres(ref):
    """pack_for_porosity(0.2, 128/2048, 12345) drawn by the reference's own
    SpherePacking::random (synthetic.hpp:42-55)."""
    r = R_VOX / N_BOX
    count = int(round(math.log(1.0 / PSI) / (4.0 / 3.0 * math.pi * r ** 3)))
    return ref.sphere_packing((0, 0, 0), (1, 1, 1), count, r, r, SEED)


def exact_crop_spheres(ref, centers, radii, size, h, origin):
    """The spheres that can be the minimum of fluid_sdf somewhere in the
    crop: with M an upper bound of the true field over the crop (the field of
    the spheres meeting the crop box), a sphere whose box distance minus
    radius exceeds M is never the minimum, not even tied. Exact, so
    field_from over the subset equals field_from over all spheres."""
    lo = np.asarray(origin, float)
    hi = lo + (np.asarray(size) - 1) * h
    d = np.linalg.norm(np.maximum(0.0, np.maximum(lo - centers, centers - hi)), axis=1) - radii
    first = d <= 0.0
    if not first.any():
        return centers, radii
    f0 = ref.field_sphere_pack(size, (h,) * 3, origin, centers[first], radii[first])
    keep = d <= float(np.max(f0))
    return centers[keep], radii[keep]


@pytest.mark.gpu
def test_device_diffusion_coefficient_is_libm_bitwise(cuda):
    """pd_smooth_diffusion_coefficients == d_min + d_max/(1+exp(-(g1+g2 phi)))
    with the host libm exp (what the reference calls), over phi spanning every
    exp branch: saturated both ways, the subnormal and overflow scalings and
    the transition band."""
    import ctypes as C
    from paper_2304_11165_b200 import _lib
    libm = C.CDLL("libm.so.6")  # the exp the reference links (Python's math.exp raises on overflow)
    libm.exp.restype, libm.exp.argtypes = C.c_double, [C.c_double]
    rng = np.random.default_rng(5)
    phi = np.concatenate([rng.uniform(-0.6, 0.6, 100000), rng.uniform(-0.002, 0.002, 100000),
                          rng.uniform(-0.0915, -0.0860, 20000), rng.uniform(0.0860, 0.0870, 20000),
                          [0.0, -0.0, 1e-300, -1e-300, np.inf, -np.inf]])
    for prof in [(0.0, 1.0, 0.0, 4.0 * N_BOX), (0.05, 0.95, 1.5, 256.0), (1e-3, 2.0, -3.0, 8192.0)]:
        out = np.empty_like(phi)
        rc = _lib.lib.pd_smooth_diffusion_coefficients(phi.ctypes.data, len(phi), *prof, out.ctypes.data, 0)
        assert rc == 0
        dmin, dmax, g1, g2 = prof
        want = np.array([dmin + dmax / (1.0 + libm.exp(-(g1 + g2 * float(p)))) for p in phi])
        bad = np.nonzero(out.view(np.uint64) != want.view(np.uint64))[0]
        assert bad.size == 0, (prof, phi[bad[:5]], out[bad[:5]], want[bad[:5]])


@pytest.mark.gpu
@pytest.mark.parametrize("edge,steps,corner", [(160, 50, 0), (256, 40, 0), (192, 30, 900)])
def test_headline_config_crop_bitwise(edge, steps, corner, cuda, ref):
    """corner > 0: the crop [corner, corner + edge)^3 of the box (origin
    shifted by corner nodes), an interior window of the bench domain."""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import porediff as pd
    h = 1.0 / N_BOX
    size, origin = (edge,) * 3, ((0.5 + corner) * h,) * 3
    geom = pd.GridGeometry.make(size, (h,) * 3, origin)
    centers, radii = bench_spheres(ref)
    # ours: the bench's device pipeline, fed the whole sphere list
    dev = pd.DeviceGrid.sphere_pack(geom, centers, radii, n_props=4, prop_phi=0)
    dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * N_BOX))
    dev.fill_hash(1, 1)
    # reference: its own SDF, builder, D (glibc exp) and hash fill
    sc, sr = exact_crop_spheres(ref, centers, radii, size, h, origin)
    sdf = ref.field_sphere_pack(size, (h,) * 3, origin, sc, sr)
    g = ref.grid_from_sdf(size, (h,) * 3, origin, sdf)
    g.populate_diffusion(0.0, 1.0, 0.0, 4.0 * N_BOX)
    g.fill_hash("u", 1)
    keys, masks = dev.layout()
    rk, rm = g.layout()
    assert len(keys) > 1000 and np.array_equal(keys, rk) and np.array_equal(masks, rm)
    for p, name in enumerate(("phi", "u", "D")):
        a, b = dev.download(p), g.prop(name)
        bad = np.nonzero(a.view(np.uint64) != b.view(np.uint64))
        assert bad[0].size == 0, (name, a[bad][:5], b[bad][:5])
    dmax = g.max_diffusivity()
    assert dev.max_active(2) == dmax
    dt = 0.4 * pd.stability_dt(geom, dmax)
    rec = 10
    code, msg, rows = g.run(make_config(dt, steps, reaction="surface_sink", rate=1.0, band_half_width=1.0,
                                        record_every=rec))
    assert code == 0, msg
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    cfg = pd.SimulationConfig(dt=dt, n_steps=steps, record_every=rec)
    cfg.reaction = pd.ReactionSpec.surface_sink(1.0, 1.0)
    res = pd.run_simulation(grid, cfg)
    assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u) for d in res.diagnostics]
    for c in ("u", "u_next"):
        a, b = grid.channel_data(c), g.prop(c)
        bad = np.nonzero(a.view(np.uint64) != b.view(np.uint64))
        assert bad[0].size == 0, (c, bad[0][:5], a[bad][:5], b[bad][:5])
    grid.close()


@pytest.mark.gpu
@pytest.mark.parametrize("log2h,u_exp", [(40, 900), (0, 1000), (-30, 1015)])
def test_nonfinite_total_mass_on_unrecorded_step_matches_reference(log2h, u_exp, cuda, ref):
    """run_simulation checks pairwise_sum(partials) * cell_volume on EVERY
    step (solver.hpp:514-515). With a large cell volume (h = 2^40: 2^120) the
    mass overflows while every |u| is far below 2^990, on a step that records
    nothing: the error (step number, type, text) and the state left behind
    must be the reference's. (the huge-value trigger now derives
    from the slot count and cell_volume.)"""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import porediff as pd
    n = 24
    h = math.ldexp(1.0, log2h)
    size, origin = (n,) * 3, (0.5 * h,) * 3
    sdf = ref.field_ball(size, (h,) * 3, origin, (12 * h, 11 * h, 12.5 * h), 9 * h, -1.0)
    g = ref.grid_from_sdf(size, (h,) * 3, origin, sdf)
    g.populate_diffusion(0.05, 1.0, 0.0, 4.0 / h)
    g.fill_hash("u", 3)
    u = g.prop("u")
    g.set_prop("u", np.ldexp(u, u_exp))  # |u| ~ 2^u_exp
    keys, masks = g.layout()
    geom = pd.GridGeometry.make(size, (h,) * 3, origin)
    data = {c: g.prop(c) for c in ("phi", "u", "D", "u_next")}
    ours = pd.SparseBlockGrid.from_layout(geom, pd.solver_channels(), keys, masks, data)
    dt = 0.3 * pd.stability_dt(geom, g.max_diffusivity())
    code, msg, rows = g.run(make_config(dt, 12, record_every=5))
    cfg = pd.SimulationConfig(dt=dt, n_steps=12, record_every=5)
    if code == 0:
        res = pd.run_simulation(ours, cfg)
        assert [tuple(r) for r in rows] == [(d.step, d.time, d.total_mass, d.min_u, d.max_u)
                                            for d in res.diagnostics]
    else:
        assert code == 6, msg  # (40, 900): "non-finite total mass at step 1"
        with pytest.raises(pd.NumericError) as ei:
            pd.run_simulation(ours, cfg)
        assert str(ei.value) == msg
    for c in ("u", "u_next"):
        assert np.array_equal(ours.channel_data(c).view(np.uint64), g.prop(c).view(np.uint64)), c
    ours.close()


@pytest.mark.gpu
@pytest.mark.parametrize("tbytes", [8, 4])
def test_huge_diffusivity_is_not_halved(tbytes, cuda, ref):
    """with |D| >= 2^1022 (2^126 in FP32) the reference's face sum
    d_a + d_b overflows while the march path's halved h_a + h_b would not;
    the plan must keep D unhalved so the result (here a numeric error) and
    the state left behind are the reference's."""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import porediff as pd
    n = 24
    h = 1.0 / n
    size, origin = (n,) * 3, (0.5 * h,) * 3
    dt_np = np.float64 if tbytes == 8 else np.float32
    sdf = ref.field_ball(size, (h,) * 3, origin, (0.5, 0.45, 0.5), 0.35, -1.0)
    g = ref.grid_from_sdf(size, (h,) * 3, origin, sdf, tbytes=tbytes)
    g.fill_hash("u", 4)
    big = 2.0 ** 1023 if tbytes == 8 else 2.0 ** 127
    d = g.prop("D")
    keys, masks = g.layout()
    act = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(len(masks), -1).astype(bool)
    d[act] = big * (0.5 + 0.5 * g.prop("u")[act])
    g.set_prop("D", d.astype(dt_np))
    geom = pd.GridGeometry.make(size, (h,) * 3, origin)
    data = {c: g.prop(c) for c in ("phi", "u", "D", "u_next")}
    ours = pd.SparseBlockGrid.from_layout(geom, pd.solver_channels(), keys, masks, data, dt_np)
    dt = 1e-300 if tbytes == 8 else 1e-40
    code, msg, rows = g.run(make_config(dt, 3, record_every=1, enforce_stability=False))
    cfg = pd.SimulationConfig(dt=dt, n_steps=3, record_every=1, enforce_stability=False)
    if code == 0:
        res = pd.run_simulation(ours, cfg)
        assert [tuple(r) for r in rows] == [(x.step, x.time, x.total_mass, x.min_u, x.max_u) for x in res.diagnostics]
    else:
        with pytest.raises(pd.PorediffError) as ei:
            pd.run_simulation(ours, cfg)
        assert str(ei.value) == msg
    # bitwise, except that a NaN is compared as NaN: x86 SSE creates the
    # default NaN 0xFFC00000 for float inf - inf, the GPU the canonical
    # 0x7FFFFFFF (FP64 agrees on 0xFFF8000000000000)
    view = np.uint64 if tbytes == 8 else np.uint32
    for c in ("u", "u_next"):
        a, b = ours.channel_data(c), g.prop(c)
        assert np.array_equal(np.isnan(a), np.isnan(b)), c
        keep = ~np.isnan(a)
        assert np.array_equal(a[keep].view(view), b[keep].view(view)), c
        if tbytes == 8:
            assert np.array_equal(a.view(view), b.view(view)), c
    ours.close()
