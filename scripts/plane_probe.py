"""Fraction of (chunk, z-plane) pairs with no active node at the bench geometry."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2304_11165_b200 import porediff as pd, synthetic as sy
n = int(sys.argv[1])
geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
pack = sy.pack_for_porosity(0.2, 128.0 / 2048, 12345)
c, r = pack.arrays()
dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4)
keys, masks = dev.layout()
planes = masks.reshape(-1, 8)  # word w = plane z (64 bits = one 8x8 plane)
empty = planes == 0
print(f"{n}^3: {len(keys)} chunks; empty planes {empty.mean():.3f}; chunks with >=1 empty plane {empty.any(axis=1).mean():.3f}")
