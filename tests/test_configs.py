"""BASELINE.json configs C3 and C4 as end-to-end pipelines at parity-test
sizes: every stage on the device (image -> indicator -> Sussman redistancing
-> band activation -> FTCS with the reactive sink and a Dirichlet inlet; or a
two-phase level set with sigmoid D and a hot sphere), compared bit for bit
with the unmodified reference (oracle/_ref) fed the same image / level set.
The full-size runs (512^3, 1024^3) are timed by scripts/configs_demo.py."""
import numpy as np
import pytest

from paper_2304_11165_b200 import porediff as pd

pytestmark = pytest.mark.gpu


def _hexrows(rows):
    return [(int(r[0]), float(r[1]).hex(), float(r[2]).hex(), float(r[3]).hex(), float(r[4]).hex()) for r in rows]


def _our_rows(res):
    return [(d.step, d.time.hex(), d.total_mass.hex(), d.min_u.hex(), d.max_u.hex()) for d in res.diagnostics]


def test_c3_soil_grf_reactive_sink_pipeline(ref, cuda):
    """C3: thresholded Gaussian random field (porosity 0.35), indicator,
    redistancing, band activation, anchored sigmoid D, u0 = hash, surface
    sink k=2 on |phi| <= h, Dirichlet inlet u=1 at x=0."""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import levelset as ls
    from paper_2304_11165_b200.synthetic import grf_mask
    n = 40
    bits = grf_mask((n, n, n), 0.35, n_modes=24, k_max=4.0, seed=3)
    h = 1.0 / n
    mask = ls.VoxelMask((n, n, n), (h, h, h), bits)
    phi_f = ls.mask_to_indicator(mask)
    geom = phi_f.geom
    diag = ls.sussman_redistance(phi_f)
    phi = phi_f.download()
    code, msg, phi_ref, (it, res, conv) = ref.field_redistance(geom.size, geom.spacing,
                                                                np.where(bits > 0, 1.0, -1.0), (1000, 1e-3, 0.5, 4, 6, 1))
    assert code == 0, msg
    assert (diag.iterations, diag.final_residual) == (it, res)
    assert np.array_equal(phi.view(np.uint64), phi_ref.view(np.uint64))

    grid = ls.build_sparse_grid(phi_f, pd.PhaseBand(), pd.solver_channels())
    prof = pd.DiffusionProfile.anchored(0.05, 0.95, 4.0 / h, 0.02)
    pd.populate_diffusion_channel(grid, prof)  # host libm exp: bit-identical
    u = grid.channel_data("u", writable=True)
    act = grid.active_bool()
    u[act] = np.array([pd.hash_unit_value(9, int(f)) for f in grid.flat_indices()[act]])
    dmax = pd.max_diffusivity(grid)
    cfg = pd.SimulationConfig(dt=0.45 * pd.stability_dt(geom, dmax), n_steps=40, record_every=10)
    cfg.reaction = pd.ReactionSpec.surface_sink(2.0, 1.0)
    cfg.outer_bc[0] = pd.FaceBc.dirichlet(1.0)

    rg = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, phi_ref)
    rg.populate_diffusion(prof.d_min, prof.d_max, prof.gamma1, prof.gamma2)
    rg.fill_hash("u", 9)
    assert np.array_equal(grid.channel_data("D").view(np.uint64), rg.prop("D").view(np.uint64))
    res_ours = pd.run_simulation(grid, cfg)
    code, msg, rows = rg.run(make_config(cfg.dt, 40, reaction="surface_sink", rate=2.0, band_half_width=1.0,
                                         bc={0: ("dirichlet", 1.0)}, record_every=10))
    assert code == 0, msg
    assert _our_rows(res_ours) == _hexrows(rows)
    assert np.array_equal(grid.channel_data("u").view(np.uint64), rg.prop("u").view(np.uint64))


def test_c4_two_phase_ceramic_pipeline(ref, cuda):
    """C4: gyroid-shell ceramic, band spanning both phases (every node
    active), sigmoid D from D_min (solid) to D_min + D_max (pore), surface
    sink k=0.1, hot sphere u0."""
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import levelset as ls
    n = 32
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    xs = geom.positions()
    k = 2.0 * np.pi / 0.5
    g = (np.sin(k * xs[0]) * np.cos(k * xs[1]) + np.sin(k * xs[1]) * np.cos(k * xs[2])
         + np.sin(k * xs[2]) * np.cos(k * xs[0]))
    sdf = (0.4 - np.abs(g)).reshape(-1)  # the same level set goes to both sides
    band = pd.PhaseBand(-1e9, 1e9)
    f = ls.DeviceField.from_host(geom, sdf)
    grid = ls.build_sparse_grid(f, band, pd.solver_channels())
    assert grid.active_node_count() == n ** 3
    prof = pd.DiffusionProfile(0.1, 1.0, 0.0, 8.0 * n)
    pd.populate_diffusion_channel(grid, prof)
    hot = np.zeros(n ** 3)
    r2 = sum((xs[a] - 0.5) ** 2 for a in range(3)).reshape(-1)
    hot[r2 < 0.15 ** 2] = 1.0
    idx = grid.flat_indices()
    u = grid.channel_data("u", writable=True)
    u[:] = hot[idx]
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, pd.max_diffusivity(grid)), n_steps=30,
                              record_every=15, phase_band=band)
    cfg.reaction = pd.ReactionSpec.surface_sink(0.1, 1.0)
    res_ours = pd.run_simulation(grid, cfg)

    rg = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf, band.b_low, band.b_up)
    rg.populate_diffusion(prof.d_min, prof.d_max, prof.gamma1, prof.gamma2)
    rg.set_prop("u", hot[idx].reshape(-1, 512))
    code, msg, rows = rg.run(make_config(cfg.dt, 30, b_low=band.b_low, b_up=band.b_up, reaction="surface_sink",
                                         rate=0.1, band_half_width=1.0, record_every=15))
    assert code == 0, msg
    assert _our_rows(res_ours) == _hexrows(rows)
    assert np.array_equal(grid.channel_data("u").view(np.uint64), rg.prop("u").view(np.uint64))
