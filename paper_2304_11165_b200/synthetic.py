"""Synthetic benchmark geometries (reference synthetic.hpp:16-108), host side.

The sphere pack reproduces ``SpherePacking::random`` bit for bit: mt19937 with
the standard 32-bit seeding and libstdc++'s ``uniform_real_distribution``
(generate_canonical with two 32-bit draws). Dense fields follow
``field_from`` (axis-0-fastest flat order, positions origin + i*h).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .porediff import GridGeometry


class MT19937:
    """std::mt19937 (32-bit Mersenne twister, default seeding)."""

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 624
        self.mt[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            self.mt[i] = (1812433253 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 30)) + i) & 0xFFFFFFFF
        self.idx = 624

    def _twist(self):
        mt = self.mt
        for i in range(624):
            y = (mt[i] & 0x80000000) | (mt[(i + 1) % 624] & 0x7FFFFFFF)
            v = mt[(i + 397) % 624] ^ (y >> 1)
            if y & 1:
                v ^= 0x9908B0DF
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 624:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= y >> 11
        y ^= (y << 7) & 0x9D2C5680
        y ^= (y << 15) & 0xEFC60000
        y ^= y >> 18
        return y & 0xFFFFFFFF


def uniform_real(rng: MT19937, a: float, b: float) -> float:
    """libstdc++ uniform_real_distribution<double>: generate_canonical<double,53>
    (k = 2 draws, sum = x0 + x1*2^32 in double, / 2^64, clamp below 1), then
    gc * (b - a) + a."""
    s = 0.0
    tmp = 1.0
    for _ in range(2):
        s += float(rng()) * tmp
        tmp *= 4294967296.0
    r = s / tmp
    if r >= 1.0:
        r = math.nextafter(1.0, 0.0)
    return r * (b - a) + a


@dataclass
class SpherePacking:
    """Random union of solid spheres; the transport phase is the complement."""

    centers: List[tuple] = field(default_factory=list)
    radii: List[float] = field(default_factory=list)

    @staticmethod
    def random(lo, hi, count: int, r_min: float, r_max: float, seed: int) -> "SpherePacking":
        rng = MT19937(seed)
        p = SpherePacking()
        for _ in range(count):
            x = uniform_real(rng, lo[0], hi[0])
            y = uniform_real(rng, lo[1], hi[1])
            z = uniform_real(rng, lo[2], hi[2])
            p.centers.append((x, y, z))
            p.radii.append(uniform_real(rng, r_min, r_max))
        return p

    def arrays(self):
        return np.array(self.centers, np.float64).reshape(-1, 3), np.array(self.radii, np.float64)

    def fluid_sdf_field(self, geom: GridGeometry) -> np.ndarray:
        """field_from(geom, fluid_sdf) as a flat float64 array (host numpy;
        small grids only — the device builder handles large ones)."""
        xs = geom.positions()
        best = np.full(tuple(geom.size[::-1]), np.inf)
        for c, r in zip(self.centers, self.radii):
            d0 = xs[0] - c[0]
            d1 = xs[1] - c[1]
            d2 = xs[2] - c[2]
            r2 = d0 * d0
            r2 = r2 + d1 * d1
            r2 = r2 + d2 * d2
            v = np.sqrt(r2) - r
            best = np.where(v < best, v, best)
        return best.reshape(-1)


def ball_sdf_field(geom: GridGeometry, center, radius: float, sign: float = 1.0) -> np.ndarray:
    """field_from(geom, sign * ball_sdf(x, c, r)) (synthetic.hpp:16-22)."""
    xs = geom.positions()
    r2 = np.zeros(tuple(geom.size[::-1]))
    for a in range(geom.dims):
        d = xs[a] - center[a]
        r2 = r2 + d * d
    return (sign * (radius - np.sqrt(r2))).reshape(-1)


def pack_for_porosity(psi: float, radius: float, seed: int, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
    """Overlapping equal spheres whose complement has expected porosity psi
    (Boolean model: psi = exp(-n * 4/3 pi r^3) per unit volume)."""
    vol = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2])
    count = int(round(math.log(1.0 / psi) * vol / (4.0 / 3.0 * math.pi * radius ** 3)))
    return SpherePacking.random(lo, hi, count, radius, radius, seed)


def grf_mask(size, porosity: float, n_modes: int = 48, k_max: float = 6.0, seed: int = 0, device=None) -> np.ndarray:
    """Soil-CT-like binary volume for config C3 (not in the reference): a
    Gaussian random field sum_m cos(2 pi k_m . x / L + phi_m) with n_modes
    random wave vectors |k| <= k_max (per box length), thresholded at the
    porosity quantile (pore = 1). Returns uint8 bits, axis 0 fastest. Built
    with torch on `device` (an input generator, not the simulated path); feed
    the same mask to both sides of a comparison."""
    import torch
    dev = torch.device(device) if device is not None else torch.device("cuda" if torch.cuda.is_available() else "cpu")
    g = torch.Generator().manual_seed(int(seed))
    k = (torch.rand((n_modes, 3), generator=g, dtype=torch.float64) * 2 - 1) * k_max
    ph = torch.rand(n_modes, generator=g, dtype=torch.float64) * 2 * math.pi
    nx, ny, nz = (int(s) for s in size)
    xs = [torch.arange(s, dtype=torch.float64, device=dev) / s for s in (nx, ny, nz)]
    field_ = torch.zeros((nz, ny, nx), dtype=torch.float64, device=dev)
    for m in range(n_modes):
        a = 2 * math.pi * k[m].to(dev)
        field_ += torch.cos(a[0] * xs[0][None, None, :] + a[1] * xs[1][None, :, None] + a[2] * xs[2][:, None, None]
                            + float(ph[m]))
    flat = field_.reshape(-1)
    # pore = the `porosity` fraction of largest values
    kth = int(round((1.0 - porosity) * flat.numel()))
    kth = min(max(kth, 1), flat.numel())
    thr = torch.kthvalue(flat.cpu() if flat.numel() > (1 << 27) else flat, kth).values.to(dev)
    return (flat > thr).to(torch.uint8).cpu().numpy()
