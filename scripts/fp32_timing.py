"""FP32 vs FP64 step throughput on the same device-built sphere pack (both
take their march kernels: pd_march32.cu / pd_march.cu).

    python scripts/fp32_timing.py [--n 1024] [--steps 50]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np

from paper_2304_11165_b200 import porediff as pd
from paper_2304_11165_b200 import synthetic as sy


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    n = a.n
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = sy.pack_for_porosity(0.2, 128.0 / 2048, 12345)
    c, r = pack.arrays()
    for dt_ in (np.float64, np.float32):
        dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4, dtype=dt_)
        dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n))
        dev.fill_hash(1, 1)
        grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev, dt_)
        cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.05), n_steps=1 << 30, record_every=1 << 30)
        cfg.reaction = pd.ReactionSpec.surface_sink(1.0, 1.0)
        st = pd.FtcsStepper(grid, cfg)
        st.run(0, 5, 1 << 30)
        st.run(5, a.steps, 1 << 30)
        ms = st.last_ms() / a.steps
        act = dev.info()[1]
        bpu = 24 if dt_ == np.float64 else 12
        print(f"{np.dtype(dt_).name}: {n}^3, {act} active, {ms:.3f} ms/step, {act / ms / 1e6:.1f} G upd/s, "
              f"{act * bpu / ms / 1e6:.0f} GB/s algorithmic ({bpu} B/update)", flush=True)
        st.close()
        grid.close()


if __name__ == "__main__":
    main()
