"""Cost of recording diagnostics every step (run_simulation's default
record_every = 1) vs never, at 512^3 (C5 crop)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_11165_b200 import porediff as pd, synthetic as sy

n_box, n = 2048, 512
pack = sy.pack_for_porosity(0.2, 128 / n_box, 12345)
h = 1.0 / n_box
geom = pd.GridGeometry.make((n,) * 3, (h,) * 3, (0.5 * h,) * 3)
c, r = pack.arrays()
dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4, prop_phi=0)
dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n_box))
dev.fill_hash(1, 1)
grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
act = dev.info()[1]
for rec in (1000, 1):
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.0), n_steps=200, record_every=rec)
    st = pd.FtcsStepper(grid, cfg)
    st.run(0, 20, 200)
    rows = st.run(20, 100, 200)
    ms = st.last_ms()
    print(f"record_every={rec}: {len(rows)} rows, {ms / 100:.3f} ms/step, {act * 100 / (ms / 1e3) / 1e9:.1f} G upd/s")
    st.close()
