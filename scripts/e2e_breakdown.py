"""Timing breakdown of one end-to-end run_simulation call on host buffers
(the bench's e2e leg) — where the host-side time goes."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2304_11165_b200 import porediff as pd, synthetic as sy

n_box = 2048
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 500
pack = sy.pack_for_porosity(0.2, 128 / n_box, 12345)
h = 1.0 / n_box
geom = pd.GridGeometry.make((n,) * 3, (h,) * 3, (0.5 * h,) * 3)
c, r = pack.arrays()
dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4, prop_phi=0)
dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n_box))
dev.fill_hash(1, 1)
keys, masks = dev.layout()
host = {}
for p, name in enumerate(pd.solver_channels()):
    t = torch.empty((len(keys), 512), dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = dev.download(p)
    host[name] = t.numpy()
dev.close()
cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, float(host["D"].max())), n_steps=steps, record_every=steps)
cfg.reaction = pd.ReactionSpec.surface_sink(1.0, 1.0)
for rep in range(2):
    T = {}
    t0 = time.perf_counter()
    g = pd.SparseBlockGrid.from_layout(geom, pd.solver_channels(), keys, masks, None)
    for name in pd.solver_channels():
        g._data[name] = host[name]
    T["from_layout"] = time.perf_counter() - t0
    t1 = time.perf_counter(); d = g.device(); torch.cuda.synchronize(); T["upload"] = time.perf_counter() - t1
    t1 = time.perf_counter(); st = pd.FtcsStepper(g, cfg); T["stepper_create"] = time.perf_counter() - t1
    t1 = time.perf_counter(); b = st.stability_bound(); T["gate"] = time.perf_counter() - t1
    t1 = time.perf_counter(); d0 = st.snapshot_diagnostics(); T["row0"] = time.perf_counter() - t1
    t1 = time.perf_counter(); rows = st.run(0, steps, steps); T["steps"] = time.perf_counter() - t1
    T["kernel_ms"] = st.last_ms() / 1e3
    t1 = time.perf_counter(); u = g.channel_data("u"); T["download_u"] = time.perf_counter() - t1
    t1 = time.perf_counter(); un = g.channel_data("u_next"); T["download_u_next"] = time.perf_counter() - t1
    st.close(); g.close()
    T["total"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in T.items()}, "ms")
