"""One Sussman redistancing run on an n^3 indicator field (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import time
import numpy as np
import torch
from paper_2304_11165_b200 import porediff as pd, levelset as ls
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
it = int(sys.argv[2]) if len(sys.argv) > 2 else 50
geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
x = (torch.arange(n, dtype=torch.float64, device="cuda") + 0.5) / n
r = torch.sqrt((x[None, None, :] - 0.5) ** 2 + (x[None, :, None] - 0.5) ** 2 + (x[:, None, None] - 0.5) ** 2)
ind = torch.where(r < 0.3, -1.0, 1.0).contiguous()
f = ls.DeviceField(geom)
f.upload(ind.cpu().numpy())
torch.cuda.synchronize()
t0 = time.perf_counter()
d = ls.sussman_redistance(f, ls.LevelSetOptions(max_iterations=it, tolerance=1e-300))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{n}^3: {d.iterations} sweeps in {dt*1e3:.1f} ms = {dt*1e3/d.iterations:.3f} ms/sweep")
