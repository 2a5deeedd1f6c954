import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2304_11165_b200 import porediff as pd, synthetic as sy
n = int(sys.argv[1])
geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
pack = sy.pack_for_porosity(0.2, 128.0 / 2048, 12345)
c, r = pack.arrays()
dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4)
dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n))
keys, masks = dev.layout()
D = dev.download(2)
full = np.all(masks == np.uint64(0xFFFFFFFFFFFFFFFF), axis=1)
uni = full & (D.min(axis=1) == D.max(axis=1))
print(f"{n}^3: chunks {len(keys)}, all-active {full.mean():.3f}, uniform-D all-active {uni.mean():.3f}, D values of uniform chunks: {np.unique(D[uni][:,0])[:5]}")
# fully uniform: own uniform and all six face neighbours uniform with the same D
cc = (n + 7) // 8
lin = (keys[:, 2].astype(np.int64) * cc + keys[:, 1]) * cc + keys[:, 0]
table = -np.ones(cc ** 3, np.int64)
table[lin] = np.arange(len(keys))
dv = np.where(uni, D[:, 0], np.nan)
ok = uni.copy()
for a, s in ((0, 1), (1, cc), (2, cc * cc)):
    for sgn in (-1, 1):
        k = keys[:, a].astype(np.int64) + sgn
        inside = (k >= 0) & (k < cc)
        nb = np.where(inside, table[np.clip(lin + sgn * s, 0, cc ** 3 - 1)], -1)
        good = inside & (nb >= 0)
        same = np.zeros(len(keys), bool)
        same[good] = uni[nb[good]] & (dv[nb[good]] == dv[good])
        ok &= same
print(f"fully uniform (with 6 neighbours): {ok.mean():.3f}; own-uniform only: {(uni & ~ok).mean():.3f}")
