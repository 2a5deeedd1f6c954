"""VTK export timing: write_grid_vtk (node texts formatted on the device,
streamed through pinned buffers) vs the reference's
write_vtk(vtk_from_sparse(grid)) (oracle/_ref, single host thread as in the
reference), same grid state, files compared byte for byte.

    python scripts/vtk_timing.py [--n 192] [--dir /tmp]
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np

from paper_2304_11165_b200 import porediff as pd
from paper_2304_11165_b200 import synthetic as sy
from paper_2304_11165_b200 import vtk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=192)
    ap.add_argument("--dir", default="/tmp")
    a = ap.parse_args()
    from oracle.pyoracle import Ref
    ref = Ref()
    n = a.n
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = sy.pack_for_porosity(0.3, 16.0 / n, 12345)
    c, r = pack.arrays()
    dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4)
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.05, 1.0, 0.0, 4.0 * n))
    dev.fill_hash(1, 3)
    grid._mark_device_newer()
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, 1.05), n_steps=3, record_every=3)
    pd.run_simulation(grid, cfg)
    keys, masks = grid.keys(), grid.masks()
    rg = ref.grid_from_chunks(geom.size, geom.spacing, geom.origin, pd.solver_channels(), keys, masks)
    for p in pd.solver_channels():
        rg.set_prop(p, grid.channel_data(p))
    ours = Path(a.dir) / f"vtk_ours_{os.getpid()}.vtk"
    theirs = Path(a.dir) / f"vtk_ref_{os.getpid()}.vtk"
    vtk.write_grid_vtk(grid, ours)  # warm (pool, module load)
    t0 = time.perf_counter()
    vtk.write_grid_vtk(grid, ours)
    t_ours = time.perf_counter() - t0
    t0 = time.perf_counter()
    code, msg = rg.write_vtk(theirs)
    t_ref = time.perf_counter() - t0
    assert code == 0, msg
    size = ours.stat().st_size
    same = size == theirs.stat().st_size and ours.read_bytes() == theirs.read_bytes()
    nodes = geom.node_count()
    vals = nodes * (len(pd.solver_channels()) + 1)
    print(f"{n}^3 lattice, {len(pd.solver_channels())} arrays + mask = {vals / 1e6:.1f} M values, "
          f"file {size / 1e9:.2f} GB, byte-identical: {same}")
    print(f"  device writer   {t_ours:8.2f} s  {vals / t_ours / 1e6:8.1f} M values/s  {size / t_ours / 1e9:6.2f} GB/s")
    print(f"  reference (1 thread) {t_ref:8.2f} s  {vals / t_ref / 1e6:8.1f} M values/s  {size / t_ref / 1e9:6.2f} GB/s")
    print(f"  speed-up {t_ref / t_ours:.1f}x")
    ours.unlink()
    theirs.unlink()


if __name__ == "__main__":
    main()
