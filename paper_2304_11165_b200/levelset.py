"""Level-set geometry stage on the device — the reference's image -> SDF ->
sparse grid pipeline (north_star subsystem 2):

    mask_to_indicator   geometry.hpp:67-77
    filter_thin_features geometry.hpp:121-142 (cubic-window opening)
    sussman_redistance  levelset.hpp:115-191 (full-grid Jacobi sweeps)
    build_sparse_grid   geometry.hpp:148-176 (band activation, chunk allocation)

A ``DeviceField`` is the reference's DenseField<T, Dims> (one T array, axis 0
fastest) resident in HBM; every stage above runs as CUDA kernels through the C
ABI and is bit-identical to the reference (node values, iteration count,
stopping residual, activation masks). Host-side helpers here are the
reference's scalar building blocks (smoothed_sign, godunov_axis_sq) and its
verification norm (band_error_norms), used by tests and reports only.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib
from . import porediff as pd
from ._lib import lib
from .porediff import InputError, _check


@dataclass
class LevelSetOptions:
    """levelset.hpp:13-20."""
    max_iterations: int = 1000
    tolerance: float = 1e-3
    pseudo_time_step: float = 0.5
    band_width_for_error: float = 4.0
    residual_band_width: float = 6.0
    rescale_initial: bool = True

    def c(self) -> _lib.pd_levelset_options:
        return _lib.pd_levelset_options(self.max_iterations, self.tolerance, self.pseudo_time_step,
                                        self.band_width_for_error, self.residual_band_width,
                                        1 if self.rescale_initial else 0)


@dataclass
class RedistanceDiagnostics:
    """levelset.hpp:22-26."""
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False


@dataclass
class VoxelMask:
    """geometry.hpp:17-39: binary volume, axis 0 fastest."""
    size: Sequence[int]
    voxel_size: Sequence[float]
    bits: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))


class DeviceField:
    """DenseField<T, Dims> in HBM."""

    def __init__(self, geometry: pd.GridGeometry, dtype=np.float64, device: int = 0):
        self.geom = geometry
        self.dtype = np.dtype(dtype)
        self.device = device
        dims = geometry.dims
        size = (C.c_int64 * 3)(*(list(geometry.size) + [1] * (3 - dims)))
        spacing = (C.c_double * 3)(*(list(geometry.spacing) + [1.0] * (3 - dims)))
        origin = (C.c_double * 3)(*(list(geometry.origin) + [0.0] * (3 - dims)))
        self.h = C.c_void_p()
        _check(lib.pd_field_create(dims, self.dtype.itemsize, size, spacing, origin, device, C.byref(self.h)))

    @classmethod
    def from_host(cls, geometry: pd.GridGeometry, values, dtype=np.float64, device: int = 0) -> "DeviceField":
        f = cls(geometry, dtype, device)
        f.upload(values)
        return f

    def node_count(self) -> int:
        return self.geom.node_count()

    def upload(self, values):
        a = np.ascontiguousarray(values, self.dtype).reshape(-1)
        if a.size != self.node_count():
            raise InputError("field value count does not match the geometry")
        _check(lib.pd_field_upload(self.h, a.ctypes.data))

    def upload_device(self, ptr: int):
        """Values from device memory (nodes x itemsize bytes at ptr)."""
        _check(lib.pd_field_upload_device(self.h, C.c_void_p(ptr)))

    def download(self) -> np.ndarray:
        out = np.empty(self.node_count(), self.dtype)
        _check(lib.pd_field_download(self.h, out.ctypes.data))
        return out

    def copy(self) -> "DeviceField":
        """Device-to-device copy (same geometry and scalar type)."""
        out = DeviceField(self.geom, self.dtype, self.device)
        ptr = C.c_void_p()
        _check(lib.pd_field_device_ptr(self.h, C.byref(ptr)))
        out.upload_device(ptr.value)
        return out

    def close(self):
        if self.h is not None and self.h.value:
            lib.pd_field_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mask_to_indicator(mask: VoxelMask, dtype=np.float64, device: int = 0) -> DeviceField:
    """geometry.hpp:67-77: true -> +1, false -> -1; node 0 at the origin."""
    geom = pd.GridGeometry.make(tuple(mask.size), tuple(mask.voxel_size))
    f = DeviceField(geom, dtype, device)
    bits = np.ascontiguousarray(mask.bits, np.uint8).reshape(-1)
    _check(lib.pd_field_from_mask(f.h, bits.ctypes.data, bits.size))
    return f


def filter_thin_features(indicator: DeviceField, min_thickness_cells: int = 2) -> DeviceField:
    """geometry.hpp:121-142: returns the opened indicator (input untouched)."""
    out = indicator.copy()
    _check(lib.pd_field_filter_thin(out.h, int(min_thickness_cells)))
    return out


def sussman_redistance(phi: DeviceField, opts: LevelSetOptions = LevelSetOptions()) -> RedistanceDiagnostics:
    """levelset.hpp:115-191, in place on the device."""
    o = opts.c()
    d = _lib.pd_redistance_diag()
    _check(lib.pd_field_redistance(phi.h, C.byref(o), C.byref(d)))
    return RedistanceDiagnostics(int(d.iterations), float(d.final_residual), bool(d.converged))


def build_sparse_grid(sdf: DeviceField, band: pd.PhaseBand = pd.PhaseBand(),
                      channels: Sequence[str] = ("phi", "u", "D")) -> pd.SparseBlockGrid:
    """geometry.hpp:148-176 on the device: the grid's state stays in HBM.
    Checks in the reference's order: band, finiteness, "phi" channel, empty
    result."""
    chans = list(channels)
    has_phi = "phi" in chans
    h = C.c_void_p()
    # without "phi" a one-property build still runs the finiteness check first
    _check(lib.pd_build_grid_from_field(sdf.h, band.b_low, band.b_up, len(chans) if has_phi else 1,
                                        chans.index("phi") if has_phi else 0, C.byref(h)))
    n = C.c_int64()
    act = C.c_int64()
    lib.pd_grid_info(h, C.byref(n), C.byref(act))
    if not has_phi or act.value == 0:
        lib.pd_grid_destroy(h)
        if not has_phi:
            raise InputError('channel list must contain "phi" to receive the level set')
        raise InputError("no node lies inside the phase band: the grid would be empty")
    dev = pd.DeviceGrid(h, sdf.geom, sdf.dtype, int(n.value), len(chans))
    return pd.SparseBlockGrid.from_device(sdf.geom, chans, dev, sdf.dtype)


# ---- host scalar helpers (reference building blocks; verification) ---------

def smoothed_sign(phi: float, grad_mag: float, h: float) -> float:
    """levelset.hpp:30-34."""
    if phi == 0.0:
        return 0.0
    return phi / math.sqrt(phi * phi + grad_mag * grad_mag * h * h)


def godunov_axis_sq(d_minus: float, d_plus: float, sign: int) -> float:
    """levelset.hpp:43-53 (std::max(a, b) = a < b ? b : a)."""
    mx = lambda a, b: b if a < b else a  # noqa: E731
    mn = lambda a, b: b if b < a else a  # noqa: E731
    if sign >= 0:
        a, b = mx(d_minus, 0.0), mn(d_plus, 0.0)
    else:
        a, b = mn(d_minus, 0.0), mx(d_plus, 0.0)
    return mx(a * a, b * b)


@dataclass
class BandErrorNorms:
    l2: float = 0.0
    linf: float = 0.0
    count: int = 0


def band_error_norms(phi: np.ndarray, geom: pd.GridGeometry, exact: Callable[[tuple], float],
                     band_width: float) -> BandErrorNorms:
    """levelset.hpp:201-226 (host; verification only)."""
    band = band_width * geom.min_spacing()
    n = BandErrorNorms()
    sum_sq = 0.0
    vals = np.asarray(phi).reshape(-1)
    for f in range(geom.node_count()):
        idx = []
        r = f
        for a in range(geom.dims):
            idx.append(r % geom.size[a])
            r //= geom.size[a]
        e = exact(geom.position(idx))
        if abs(e) <= band:
            err = abs(float(vals[f]) - e)
            sum_sq += err * err
            n.linf = max(n.linf, err)
            n.count += 1
    if n.count == 0:
        raise InputError("error band is empty: no node satisfies |exact| <= band_width*h")
    n.l2 = math.sqrt(sum_sq / n.count)
    return n
