"""Per-step device time of free-box (every node active, uniform D) runs —
the FRAP / D_eff fit's probes (analysis.hpp:147-153) — at several sizes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_11165_b200 import porediff as pd

for n in (64, 128, 256, 512):
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    dev = pd.DeviceGrid.full(geom, 4, prop_phi=0, phi_value=1.0)
    dev.fill_const(2, 1.0)
    dev.fill_hash(1, 3)
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.0), n_steps=1 << 30, record_every=1 << 30)
    st = pd.FtcsStepper(grid, cfg)
    st.run(0, 50, 1 << 30)
    steps = 2000 if n <= 128 else 300
    st.run(50, steps, 1 << 30)
    ms = st.last_ms() / steps
    print(f"{n}^3 free box: {ms * 1e3:.1f} us/step, {n ** 3 / ms / 1e6:.1f} G upd/s", flush=True)
    st.close()
    grid.close()
