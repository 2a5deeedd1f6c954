"""Full-size runs of BASELINE.json configs C1-C4 on one B200, every stage on
the device, with per-stage wall times (C5 is bench.py). Parity for each
pipeline is established at smaller sizes by the tests (test_gpu_parity,
test_frap, test_levelset, test_configs); these runs show the same code paths
at the configured sizes.

    python scripts/configs_demo.py [--only C2] > profiles/r01_configs_demo.txt
"""
import argparse
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2304_11165_b200 import analysis as an
from paper_2304_11165_b200 import levelset as ls
from paper_2304_11165_b200 import porediff as pd
from paper_2304_11165_b200 import synthetic as sy


class Timer:
    def __init__(self):
        self.rows = []

    def __call__(self, name, fn, *a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        self.rows.append((name, dt))
        print(f"    {name:38s} {dt * 1e3:10.1f} ms", flush=True)
        return out


def steps_rate(grid, cfg, label, T):
    st = pd.FtcsStepper(grid, cfg)
    T(label, st.run, 0, cfg.n_steps, cfg.n_steps)
    ms = st.last_ms()
    act = grid.device().info()[1]
    st.close()
    print(f"    -> {act} active nodes x {cfg.n_steps} steps: {act * cfg.n_steps / (ms / 1e3) / 1e9:.1f} G upd/s "
          f"(device time {ms:.1f} ms)", flush=True)


def c1(T):
    print("C1: 64^3 single-sphere obstacle, no-flux, 1000 steps (golden: mass 0.4449934885835134)")
    n = 64
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    sdf = sy.ball_sdf_field(geom, (0.5, 0.5, 0.5), 0.3, -1.0)
    grid = T("build_sparse_grid (host numpy)", pd.build_sparse_grid, sdf, geom, pd.PhaseBand(), pd.solver_channels())
    T("populate D (host libm)", pd.populate_diffusion_channel, grid, pd.DiffusionProfile(0.0, 1.0, 0.0, 1.0))
    u = grid.channel_data("u", writable=True)
    act = grid.active_bool()
    u[act] = np.array([pd.hash_unit_value(1, int(f)) for f in grid.flat_indices()[act]])
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, pd.max_diffusivity(grid)), n_steps=1000,
                              record_every=1000)
    res = T("run_simulation (1000 steps)", pd.run_simulation, grid, cfg)
    d = res.diagnostics[-1]
    print(f"    -> mass {d.total_mass!r} min {d.min_u!r} max {d.max_u!r}")


def c2(T, n=256, t_final=0.04):
    print(f"C2: {n}^3 random overlapping-sphere pack, FRAP to recovery >= 0.99 + golden-section D_eff / tortuosity "
          f"fit, and the steady-state flux estimate")
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = sy.pack_for_porosity(0.3, 16.0 / n, 12345)
    c, r = pack.arrays()
    box = an.central_bleach_box(geom, 0.1)
    dt = 0.4 * pd.stability_dt(geom, 1.2)
    while True:  # "run to steady state": the recovery curve reaches 0.99
        dev = T(f"device sphere-pack build ({len(r)} spheres)", pd.DeviceGrid.sphere_pack, geom, c, r, n_props=4)
        grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
        exp = T(f"run_frap (porous, D_mol = 1, t_final {t_final})", an.run_frap, grid, box, 1.0,
                an.FrapSchedule(t_final, 50, dt))
        print(f"    -> {len(exp.curve)} samples, final recovery {exp.curve[-1].recovery:.6f}, "
              f"region {exp.region_nodes} / phase {exp.phase_nodes} nodes")
        grid.close(keep=False)
        if exp.curve[-1].recovery >= 0.99:
            break
        t_final *= 2
    fit = T("fit_effective_D (free-box runs on device)", an.fit_effective_D, exp, geom, box, 0.2, 1.2,
            an.FitOptions(rel_tol=1e-3, dt=dt))
    print(f"    -> D_eff {fit.d_eff!r}  tau_d {fit.tau_d!r}  residual {fit.fit_residual:.3e}  "
          f"edge_warning {fit.edge_warning}")
    # steady-state through-diffusion (north_star (3); no reference counterpart)
    dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4)
    dev.fill_const(2, 1.0)
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    ss = T("steady_state_diffusivity (x, c 1 -> 0, device observers)", an.steady_state_diffusivity, grid, 0,
           1.0, 0.0, 1.0, 0.0, 1e-6, 2000)
    print(f"    -> {ss.steps} steps, converged {ss.converged} (rate {ss.rate:.2e}), porosity {ss.porosity:.4f}, "
          f"D_bulk {ss.d_bulk:.6f}, D_eff {ss.d_eff:.6f}, tau {ss.tau:.6f}, plane-flux spread "
          f"{(max(ss.plane_fluxes) - min(ss.plane_fluxes)) / ss.flux:.2e}")
    grid.close(keep=False)


def c3(T, n=512, steps=1000):
    print(f"C3: {n}^3 soil-CT-like pore space (thresholded GRF, porosity 0.35), reactive sink + Dirichlet inlet")
    h = 1.0 / n
    bits = T("GRF mask (torch, input generator)", sy.grf_mask, (n, n, n), 0.35, 48, 6.0, 7)
    mask = ls.VoxelMask((n, n, n), (h, h, h), bits)
    phi = T("mask_to_indicator", ls.mask_to_indicator, mask)
    phi2 = T("filter_thin_features (w = 2)", ls.filter_thin_features, phi, 2)
    phi.close()
    diag = T("sussman_redistance", ls.sussman_redistance, phi2)
    print(f"    -> {diag.iterations} sweeps, residual {diag.final_residual:.3e} h, converged {diag.converged}")
    grid = T("build_sparse_grid (device)", ls.build_sparse_grid, phi2, pd.PhaseBand(), pd.solver_channels())
    phi2.close()
    dev = grid.device()
    prof = pd.DiffusionProfile.anchored(0.05, 0.95, 4.0 / h, 0.02)
    T("populate D (device exp)", dev.populate_diffusion, 0, 2, prof)
    T("u0 = hash", dev.fill_hash, 1, 7)
    grid._mark_device_newer()
    nch, act = dev.info()
    print(f"    -> {nch} chunks, {act} active nodes")
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(grid.geometry(), 1.0), n_steps=steps, record_every=steps)
    cfg.reaction = pd.ReactionSpec.surface_sink(2.0, 1.0)
    cfg.outer_bc[0] = pd.FaceBc.dirichlet(1.0)
    steps_rate(grid, cfg, f"{steps} FTCS steps (sink + inlet)", T)
    if os.environ.get("C3_NO_INLET"):
        cfg.outer_bc[0] = pd.FaceBc.no_flux()
        steps_rate(grid, cfg, f"{steps} FTCS steps (sink, no inlet)", T)
    grid.close()


def c4(T, n=1024, steps=200):
    print(f"C4: {n}^3 porous ceramic (gyroid shell), two-phase sigmoid D, surface sink, u0 = 0.5")
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)

    def gyroid():
        x = (torch.arange(n, dtype=torch.float64, device="cuda") + 0.5) / n
        k = 2 * math.pi / 0.25
        sx, cx = torch.sin(k * x), torch.cos(k * x)
        g = (sx[None, None, :] * cx[None, :, None] + sx[None, :, None] * cx[:, None, None]
             + sx[:, None, None] * cx[None, None, :])
        return (0.35 - g.abs()).contiguous()

    sdf = T("gyroid level set (torch)", gyroid)
    f = ls.DeviceField(geom)
    T("upload level set (device to device)", f.upload_device, sdf.data_ptr())
    del sdf
    band = pd.PhaseBand(-1e9, 1e9)
    grid = T("build_sparse_grid (device, all nodes)", ls.build_sparse_grid, f, band, pd.solver_channels())
    f.close()
    dev = grid.device()
    T("populate D (device exp)", dev.populate_diffusion, 0, 2, pd.DiffusionProfile(0.1, 1.0, 0.0, 8.0 * n))
    T("u0 = 0.5", dev.fill_const, 1, 0.5)
    grid._mark_device_newer()
    nch, act = dev.info()
    print(f"    -> {nch} chunks, {act} active nodes")
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.1), n_steps=steps, record_every=steps,
                              phase_band=band)
    cfg.reaction = pd.ReactionSpec.surface_sink(0.1, 1.0)
    steps_rate(grid, cfg, f"{steps} FTCS steps (two-phase, sink)", T)
    grid.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    print(torch.cuda.get_device_name(0))
    T = Timer()
    for name, fn in (("C1", c1), ("C2", c2), ("C3", c3), ("C4", c4)):
        if a.only and name not in a.only.split(","):
            continue
        t0 = time.perf_counter()
        fn(T)
        print(f"  {name} total {time.perf_counter() - t0:.1f} s\n", flush=True)


if __name__ == "__main__":
    main()
