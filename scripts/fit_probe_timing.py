"""Time one free-box FRAP probe of the D_eff fit at 256^3 (C2) by phase."""
import sys, time, cProfile, pstats
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2304_11165_b200 import porediff as pd, analysis as an
n = 256
geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
box = an.central_bleach_box(geom, 0.1)
dt = 0.4 * pd.stability_dt(geom, 1.2)
sched = an.FrapSchedule(0.01, 50, dt)
for rep in range(2):
    t0 = time.perf_counter()
    g = an.build_free_box_grid(geom)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    pr = cProfile.Profile(); pr.enable()
    exp = an.run_frap(g, box, 0.7, sched)
    pr.disable()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    g.close(); t3 = time.perf_counter()
    print(f"rep {rep}: build {1e3*(t1-t0):.1f} ms, run_frap {1e3*(t2-t1):.1f} ms, close {1e3*(t3-t2):.1f} ms", flush=True)
    if rep == 1:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
