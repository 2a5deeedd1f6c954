"""Fractions of chunks by D_eff structure at the bench geometry (n^3): all
active; own-uniform; uniform with the neighbours' facing layers (the
kFlagUnif criterion)."""
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
dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n))
keys, masks = dev.layout()
D = dev.download(2).view(np.uint64)
full = np.all(masks == np.uint64(0xFFFFFFFFFFFFFFFF), axis=1)
own = full & np.all(D == D[:, :1], axis=1)
cc = (n + 7) // 8
lin = (keys[:, 2].astype(np.int64) * cc + keys[:, 1]) * cc + keys[:, 0]
table = -np.ones(cc ** 3, np.int64)
table[lin] = np.arange(len(keys))
v = D[:, 0]
offs = {}
a = np.arange(8)
B, A = np.meshgrid(a, a, indexing="ij")
offs[(0, -1)] = ((B << 6) | (A << 3) | 7).ravel()
offs[(0, 1)] = ((B << 6) | (A << 3)).ravel()
offs[(1, -1)] = ((B << 6) | (7 << 3) | A).ravel()
offs[(1, 1)] = ((B << 6) | A).ravel()
offs[(2, -1)] = ((7 << 6) | (B << 3) | A).ravel()
offs[(2, 1)] = ((B << 3) | A).ravel()
ok = own.copy()
for ax, s in ((0, 1), (1, cc), (2, cc * cc)):
    for sg in (-1, 1):
        k = keys[:, ax].astype(np.int64) + sg
        inside = (k >= 0) & (k < cc)
        nb = np.where(inside, table[np.clip(lin + sg * s, 0, cc ** 3 - 1)], -1)
        idx = np.nonzero(ok & (nb >= 0))[0]
        good = np.zeros(len(keys), bool)
        face = D[nb[idx]][:, offs[(ax, sg)]]
        good[idx] = np.all(face == v[idx, None], axis=1)
        ok &= good
print(f"{n}^3: {len(keys)} chunks; all-active {full.mean():.3f}; own-uniform {own.mean():.3f}; "
      f"kFlagUnif (facing layers) {ok.mean():.3f}")
