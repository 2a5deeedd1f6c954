"""Per-step device time of small grids (launch-bound regime): C1 64^3 and the
32^3 FRAP free box."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2304_11165_b200 import porediff as pd, synthetic as sy, analysis as an

for n in (128, 192, 256, 320):
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    dev = pd.DeviceGrid.full(geom, 4, prop_phi=0, phi_value=1.0)
    dev.fill_const(2, 1.0)
    dev.fill_hash(1, 3)
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.0), n_steps=2000, record_every=2000)
    st = pd.FtcsStepper(grid, cfg)
    st.run(0, 200, 2000)
    t0 = time.perf_counter(); st.run(200, 1000, 2000); wall = time.perf_counter() - t0
    ms = st.last_ms()
    print(f"{n}^3 free box: {1000} steps device {ms:.2f} ms ({ms:.3f} us/step x1000), wall {wall*1e3:.1f} ms", flush=True)
    st.close(); grid.close()
