"""2-D step throughput (the generic staged-tile kernel: one CTA per 8x8
chunk) on a large disk-array pore space.

    python scripts/dims2_timing.py [--n 8192] [--steps 50]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np

from paper_2304_11165_b200 import porediff as pd
from paper_2304_11165_b200 import levelset as ls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    n = a.n
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 2)
    import torch
    x = (torch.arange(n, dtype=torch.float64, device="cuda") + 0.5) / n
    per, rad = 1.0 / 32, 0.4 / 32
    dx = torch.remainder(x, per) - per / 2
    sdf = (torch.sqrt(dx[None, :] ** 2 + dx[:, None] ** 2) - rad).contiguous()  # pore outside disks
    for dt_ in (np.float64, np.float32):
        f = ls.DeviceField(geom, dt_)
        f.upload_device(sdf.to(torch.float64 if dt_ == np.float64 else torch.float32).data_ptr())
        grid = ls.build_sparse_grid(f, pd.PhaseBand(), pd.solver_channels())
        f.close()
        dev = grid.device()
        dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n))
        dev.fill_hash(1, 3)
        grid._mark_device_newer()
        cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.05), n_steps=1 << 30, record_every=1 << 30)
        st = pd.FtcsStepper(grid, cfg)
        st.run(0, 5, 1 << 30)
        st.run(5, a.steps, 1 << 30)
        ms = st.last_ms() / a.steps
        act = dev.info()[1]
        bpu = 24 if dt_ == np.float64 else 12
        print(f"2-D {np.dtype(dt_).name}: {n}^2, {act} active, {ms:.3f} ms/step, {act / ms / 1e6:.1f} G upd/s, "
              f"{act * bpu / ms / 1e6:.0f} GB/s algorithmic", flush=True)
        st.close()
        grid.close()


if __name__ == "__main__":
    main()
