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
