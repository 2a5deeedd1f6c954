"""Python mirror of the reference ``porediff`` hot-path API over the C ABI.

Same names, argument meaning and error behaviour as the C++ templates in
/root/reference/proj/include/porediff (solver.hpp, sparse_block_grid.hpp,
grid_geometry.hpp, geometry.hpp, errors.hpp), so parity tests read like the
reference's own gtest suites. The host ``SparseBlockGrid`` is the source of
truth between runs; ``FtcsStepper`` / ``run_simulation`` upload it once,
advance it on the B200 through ``libporediff_b200.so`` and download lazily
(only when the host touches the data), exactly the ownership rule of
SURVEY.md §8b. There is no CPU execution path for the step.
"""
from __future__ import annotations

import ctypes as C
import math
import time as _time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import lib

# ---------------------------------------------------------------------------
# errors (errors.hpp:9-41)
# ---------------------------------------------------------------------------


class PorediffError(RuntimeError):
    """porediff::error"""


class InputError(PorediffError):
    """porediff::input_error"""


class BoundsError(PorediffError):
    """porediff::bounds_error"""


class PropertyError(PorediffError):
    """porediff::property_error"""


class IoError(PorediffError):
    """porediff::io_error"""


class StabilityError(PorediffError):
    """porediff::stability_error"""


class NumericError(PorediffError):
    """porediff::numeric_error"""


class DeviceError(PorediffError):
    """CUDA / driver failure (no reference analogue)."""


_ERRORS = {
    _lib.PD_E_INPUT: InputError,
    _lib.PD_E_BOUNDS: BoundsError,
    _lib.PD_E_PROPERTY: PropertyError,
    _lib.PD_E_IO: IoError,
    _lib.PD_E_STABILITY: StabilityError,
    _lib.PD_E_NUMERIC: NumericError,
    _lib.PD_E_CUDA: DeviceError,
}


def _check(rc: int) -> None:
    if rc != _lib.PD_OK:
        raise _ERRORS.get(rc, PorediffError)(_lib.last_error())


def format_scalar(v: float, digits: int = 17) -> str:
    """scalar_text.hpp:21-28 (%.17g for double, %.9g for float; nan)."""
    if math.isnan(v):
        return "nan"
    s = "%.*g" % (digits, v)
    return s


# ---------------------------------------------------------------------------
# geometry (grid_geometry.hpp:23-112)
# ---------------------------------------------------------------------------


@dataclass
class GridGeometry:
    size: tuple
    spacing: tuple
    origin: tuple

    @property
    def dims(self) -> int:
        return len(self.size)

    @staticmethod
    def make(size, spacing, origin=None) -> "GridGeometry":
        size = tuple(int(s) for s in size)
        spacing = tuple(float(h) for h in spacing)
        if len(size) not in (2, 3) or len(spacing) != len(size):
            raise InputError("only 2-D and 3-D grids are supported")
        for a, (s, h) in enumerate(zip(size, spacing)):
            if s < 1:
                raise InputError(f"grid size must be >= 1 along every axis, got {s} on axis {a}")
            if not h > 0.0:
                raise InputError(f"grid spacing must be > 0 along every axis, got {h} on axis {a}")
        origin = tuple(float(o) for o in origin) if origin is not None else (0.0,) * len(size)
        return GridGeometry(size, spacing, origin)

    @staticmethod
    def cell_centered_box(n: int, lo: float, hi: float, dims: int = 3) -> "GridGeometry":
        h = (hi - lo) / float(n)
        return GridGeometry.make((n,) * dims, (h,) * dims, (lo + 0.5 * h,) * dims)

    def node_count(self) -> int:
        return int(np.prod(self.size))

    def flat_index(self, idx) -> int:
        f = idx[-1]
        for a in range(self.dims - 2, -1, -1):
            f = f * self.size[a] + idx[a]
        return int(f)

    def contains(self, idx) -> bool:
        return all(0 <= i < s for i, s in zip(idx, self.size))

    def coord(self, axis: int, i: int) -> float:
        return self.origin[axis] + float(i) * self.spacing[axis]

    def position(self, idx):
        return tuple(self.coord(a, i) for a, i in enumerate(idx))

    def min_spacing(self) -> float:
        h = self.spacing[0]
        for a in range(1, self.dims):
            h = h if h < self.spacing[a] else self.spacing[a]
        return h

    def cell_volume(self) -> float:
        v = 1.0
        for h in self.spacing:
            v *= h
        return v

    def positions(self) -> List[np.ndarray]:
        """Per-axis node coordinates broadcastable to the flat (axis-0 fastest)
        array of shape size[::-1]."""
        out = []
        for a in range(self.dims):
            x = self.origin[a] + np.arange(self.size[a], dtype=np.float64) * self.spacing[a]
            shape = [1] * self.dims
            shape[self.dims - 1 - a] = self.size[a]
            out.append(x.reshape(shape))
        return out


# ---------------------------------------------------------------------------
# configuration (solver.hpp:38-106, geometry.hpp:43-63)
# ---------------------------------------------------------------------------


@dataclass
class PhaseBand:
    b_low: float = 0.0
    b_up: float = math.inf


@dataclass
class DiffusionProfile:
    d_min: float = 0.0
    d_max: float = 1.0
    gamma1: float = 0.0
    gamma2: float = 1.0

    @staticmethod
    def anchored(d_min, d_max, gamma2, phi_anchor) -> "DiffusionProfile":
        return DiffusionProfile(d_min, d_max, -gamma2 * phi_anchor, gamma2)


@dataclass
class ReactionSpec:
    kind: str = "none"  # none | surface_sink | volumetric
    rate: float = 0.0
    band_half_width: float = 1.0
    source_channel: str = ""
    time_factor: Optional[Callable[[float], float]] = None

    @staticmethod
    def none() -> "ReactionSpec":
        return ReactionSpec()

    @staticmethod
    def surface_sink(k: float, w: float = 1.0) -> "ReactionSpec":
        return ReactionSpec("surface_sink", rate=k, band_half_width=w)

    @staticmethod
    def volumetric(channel: str, g: Optional[Callable[[float], float]] = None) -> "ReactionSpec":
        return ReactionSpec("volumetric", source_channel=channel, time_factor=g)


@dataclass
class FaceBc:
    type: str = "no_flux"
    value: float = 0.0

    @staticmethod
    def no_flux() -> "FaceBc":
        return FaceBc()

    @staticmethod
    def dirichlet(v: float) -> "FaceBc":
        return FaceBc("dirichlet", float(v))


@dataclass
class SimulationConfig:
    dt: float = 0.0
    n_steps: int = 1
    phase_band: PhaseBand = field(default_factory=PhaseBand)
    boundary_epsilon: float = 0.0
    reaction: ReactionSpec = field(default_factory=ReactionSpec)
    outer_bc: List[FaceBc] = field(default_factory=lambda: [FaceBc() for _ in range(6)])
    record_every: int = 1
    enforce_stability: bool = True


@dataclass
class StepDiagnostics:
    step: int = 0
    time: float = 0.0
    total_mass: float = 0.0
    min_u: float = 0.0
    max_u: float = 0.0
    wall_seconds: float = 0.0


@dataclass
class SimulationResult:
    diagnostics: List[StepDiagnostics]
    # device region-mass observer (run_frap): box sum of u per diagnostics row
    region_sums: List[float] = field(default_factory=list)


scratch_channel = "u_next"


def solver_channels() -> List[str]:
    return ["phi", "u", "D", scratch_channel]


def stability_dt(geometry: GridGeometry, d_max: float) -> float:
    """solver.hpp:111-120."""
    if not d_max > 0.0:
        raise InputError("stability bound needs D_max > 0")
    inv_sum = 0.0
    for h in geometry.spacing:
        inv_sum += 1.0 / (h * h)
    return 1.0 / (2.0 * d_max) / inv_sum


def pairwise_sum(values) -> float:
    """parallel.hpp:68-84 (host utility; the device uses the same tree)."""
    v = [float(x) for x in values]
    if not v:
        return 0.0
    n = len(v)
    while n > 1:
        half = n // 2
        for i in range(half):
            v[i] = v[2 * i] + v[2 * i + 1]
        if n % 2 == 1:
            v[half] = v[n - 1]
            n = half + 1
        else:
            n = half
    return v[0]


def hash_unit_value(seed: int, key: int) -> float:
    """config.hpp:558-564."""
    m = (1 << 64) - 1
    seed, key = int(seed), int(key)
    z = (seed + 0x9E3779B97F4A7C15 * (key + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    z ^= z >> 31
    return float(z >> 11) * 2.0 ** -53


# ---------------------------------------------------------------------------
# sparse block grid (sparse_block_grid.hpp:30-304)
# ---------------------------------------------------------------------------


class SparseBlockGrid:
    """8^Dims chunk store. Host arrays are kept in ascending chunk linear
    index (the reference traversal order); one (n_chunks, V) array per
    logical property; ``swap_channels`` swaps the arrays in O(1)."""

    chunk_edge = 8

    def __init__(self, geometry: GridGeometry, properties: Sequence[str], dtype=np.float64):
        if not properties:
            raise InputError("sparse grid needs at least one property")
        props = list(properties)
        for i in range(len(props)):
            for j in range(i + 1, len(props)):
                if props[i] == props[j]:
                    raise InputError(f"duplicate property name '{props[i]}'")
        self.geom = geometry
        self.props = props
        self.dtype = np.dtype(dtype)
        self.dims = geometry.dims
        self.V = 512 if self.dims == 3 else 64
        self.W = self.V // 64
        self.cc = tuple((s + 7) // 8 for s in geometry.size)
        self._keys = np.zeros((0, self.dims), np.int32)
        self._masks = np.zeros((0, self.W), np.uint64)
        self._data = {p: np.zeros((0, self.V), self.dtype) for p in props}
        self._lin = np.zeros(0, np.int64)
        self._pending = {}  # linear index -> chunk being built by insert()
        self._dev = None  # DeviceGrid mirror
        self._dev_newer = set()  # properties whose device copy the host has not fetched
        self._host_newer = True

    # -- construction ------------------------------------------------------
    @classmethod
    def from_layout(cls, geometry, properties, keys, masks, data=None, dtype=np.float64):
        g = cls(geometry, properties, dtype)
        keys = np.ascontiguousarray(keys, np.int32).reshape(-1, g.dims)
        masks = np.ascontiguousarray(masks, np.uint64).reshape(-1, g.W)
        lin = g._linear(keys)
        if len(lin) > 1 and not np.all(np.diff(lin) > 0):
            order = np.argsort(lin, kind="stable")
            keys, masks, lin = keys[order], masks[order], lin[order]
            if data:
                data = {k: np.asarray(v)[order] for k, v in data.items()}
        g._keys, g._masks, g._lin = keys, masks, lin
        for p in g.props:
            if data and p in data:
                g._data[p] = np.ascontiguousarray(data[p], g.dtype).reshape(-1, g.V).copy()
            else:
                g._data[p] = np.zeros((len(lin), g.V), g.dtype)
        return g

    @classmethod
    def from_device(cls, geometry, properties, dev: "DeviceGrid", dtype=np.float64):
        """A grid whose state lives on the device (host slabs fetched on first
        access)."""
        g = cls(geometry, properties, dtype)
        keys, masks = dev.layout()
        g._keys, g._masks, g._lin = keys, masks, g._linear(keys)
        g._data = {p: None for p in g.props}
        g._dev = dev
        g._dev_newer = set(g.props)
        g._host_newer = False
        return g

    def _linear(self, keys: np.ndarray) -> np.ndarray:
        keys = keys.astype(np.int64)
        lin = keys[:, self.dims - 1].copy()
        for a in range(self.dims - 2, -1, -1):
            lin = lin * self.cc[a] + keys[:, a]
        return lin

    def geometry(self) -> GridGeometry:
        return self.geom

    def property_names(self):
        return list(self.props)

    def property_index(self, name: str) -> int:
        try:
            return self.props.index(name)
        except ValueError:
            raise PropertyError(f"unknown property '{name}'") from None

    # -- device coherence ----------------------------------------------------
    def _sync_host(self):
        self._flush_pending()
        if self._dev is not None and self._dev_newer:
            for p in self.props:
                if p not in self._dev_newer:
                    continue
                cur = self._data.get(p)
                if (isinstance(cur, np.ndarray) and cur.shape == (self._dev.n_chunks, self.V)
                        and cur.dtype == self.dtype and cur.flags.c_contiguous and cur.flags.writeable):
                    self._dev.download_into(self.property_index(p), cur)  # reuse (possibly pinned) buffer
                else:
                    self._data[p] = self._dev.download(self.property_index(p))
            self._dev_newer = set()

    def _touch_host(self):
        self._sync_host()
        self._host_newer = True

    def device(self, device: int = 0) -> "DeviceGrid":
        """Device mirror, (re)uploaded if the host changed since last use."""
        self._flush_pending()
        if self._dev is None or self._dev.n_chunks != len(self._lin):
            self._sync_host()
            if self._dev is not None:
                self._dev.close()
            self._dev = DeviceGrid.create(self.geom, self.dtype, self._keys, self._masks,
                                          len(self.props), device)
            self._host_newer = True
        if self._host_newer:
            for p in self.props:
                self._dev.upload(self.property_index(p), self._data[p])
            self._host_newer = False
        return self._dev

    def _mark_device_newer(self, props=None):
        """The device advanced these properties (default: all)."""
        self._dev_newer |= set(self.props if props is None else props)

    # -- insertion (sparse_block_grid.hpp:117-132) ---------------------------
    def _check_bounds(self, idx):
        if not self.geom.contains(idx):
            raise BoundsError("node index (" + ",".join(str(int(i)) for i in idx) + ") outside grid")

    @staticmethod
    def offset_of(idx) -> int:
        off = int(idx[-1]) & 7
        for a in range(len(idx) - 2, -1, -1):
            off = (off << 3) | (int(idx[a]) & 7)
        return off

    def _chunk_lin(self, idx) -> int:
        k = [int(i) >> 3 for i in idx]
        f = k[-1]
        for a in range(self.dims - 2, -1, -1):
            f = f * self.cc[a] + k[a]
        return f

    def _find(self, lin):
        if lin in self._pending:
            return ("p", self._pending[lin])
        j = int(np.searchsorted(self._lin, lin))
        if j < len(self._lin) and self._lin[j] == lin:
            return ("o", j)
        return None

    def insert(self, idx, values=()):
        self._check_bounds(idx)
        values = list(values)
        if values and len(values) != len(self.props):
            raise InputError(f"insert expects one value per property ({len(self.props)}), got {len(values)}")
        self._touch_host()
        lin = self._chunk_lin(idx)
        off = self.offset_of(idx)
        loc = self._find(lin)
        if loc is None:
            ch = {"key": [int(i) >> 3 for i in idx], "mask": np.zeros(self.W, np.uint64),
                  "data": {p: np.zeros(self.V, self.dtype) for p in self.props}}
            self._pending[lin] = ch
            loc = ("p", ch)
        if loc[0] == "p":
            ch = loc[1]
            ch["mask"][off >> 6] |= np.uint64(1 << (off & 63))
            for p, v in zip(self.props, values):
                ch["data"][p][off] = v
        else:
            j = loc[1]
            self._masks[j, off >> 6] |= np.uint64(1 << (off & 63))
            for p, v in zip(self.props, values):
                self._data[p][j, off] = v

    def _flush_pending(self):
        if not self._pending:
            return
        lins = np.array(sorted(self._pending), np.int64)
        keys = np.array([self._pending[l]["key"] for l in lins], np.int32).reshape(-1, self.dims)
        masks = np.array([self._pending[l]["mask"] for l in lins], np.uint64).reshape(-1, self.W)
        all_lin = np.concatenate([self._lin, lins])
        order = np.argsort(all_lin, kind="stable")
        self._lin = all_lin[order]
        self._keys = np.concatenate([self._keys, keys])[order]
        self._masks = np.concatenate([self._masks, masks])[order]
        for p in self.props:
            new = np.array([self._pending[l]["data"][p] for l in lins], self.dtype).reshape(-1, self.V)
            self._data[p] = np.concatenate([self._data[p], new])[order]
        self._pending = {}

    # -- access ----------------------------------------------------------------
    def _locate(self, idx):
        self._check_bounds(idx)
        self._flush_pending()
        lin = self._chunk_lin(idx)
        j = int(np.searchsorted(self._lin, lin))
        if j < len(self._lin) and self._lin[j] == lin:
            off = self.offset_of(idx)
            if (int(self._masks[j, off >> 6]) >> (off & 63)) & 1:
                return j, off
        return None

    def is_active(self, idx) -> bool:
        return self._locate(idx) is not None

    def get(self, idx, prop: str):
        p = self.property_index(prop)
        loc = self._locate(idx)
        if loc is None:
            return None
        self._sync_host()
        return self._data[self.props[p]][loc]

    def set(self, idx, prop: str, value) -> None:
        p = self.property_index(prop)
        loc = self._locate(idx)
        if loc is None:
            raise InputError("set on inactive node; insert it first")
        self._touch_host()
        self._data[self.props[p]][loc] = value

    def swap_channels(self, a: str, b: str) -> None:
        ia, ib = self.property_index(a), self.property_index(b)
        self._sync_host()
        pa, pb = self.props[ia], self.props[ib]
        self._data[pa], self._data[pb] = self._data[pb], self._data[pa]
        self._host_newer = True

    def channel_data(self, prop: str, writable: bool = False) -> np.ndarray:
        """(n_chunks, V) slabs of one logical property in ordinal order."""
        p = self.property_index(prop)
        if writable:
            self._touch_host()
        else:
            self._sync_host()
        return self._data[self.props[p]]

    def keys(self) -> np.ndarray:
        self._flush_pending()
        return self._keys

    def masks(self) -> np.ndarray:
        self._flush_pending()
        return self._masks

    def active_bool(self) -> np.ndarray:
        """(n_chunks, V) boolean activation."""
        m = self.masks()
        bits = np.unpackbits(m.view(np.uint8).reshape(len(m), self.W, 8), axis=-1, bitorder="little")
        return bits.reshape(len(m), self.V).astype(bool)

    def chunk_count(self) -> int:
        self._flush_pending()
        return len(self._lin)

    def active_node_count(self) -> int:
        self._flush_pending()
        return int(sum(bin(int(w)).count("1") for w in self._masks.ravel())) if len(self._masks) < 4096 \
            else int(self.active_bool().sum())

    def stats(self) -> dict:
        n = self.chunk_count()
        a = self.active_node_count()
        mx = int(np.prod(self.cc))
        return {"chunk_count": n, "active_nodes": a, "dense_node_count": self.geom.node_count(),
                "max_chunks": mx, "node_fill_fraction": a / self.geom.node_count(),
                "chunk_fill_fraction": n / mx}

    def node_indices(self) -> np.ndarray:
        """Global node index of every slot, shape (n_chunks, V, Dims)."""
        keys = self.keys().astype(np.int64)
        off = np.arange(self.V)
        local = np.stack([(off >> (3 * a)) & 7 for a in range(self.dims)], axis=-1)
        return (keys[:, None, :] << 3) | local[None, :, :]

    def flat_indices(self) -> np.ndarray:
        idx = self.node_indices()
        f = idx[..., self.dims - 1]
        for a in range(self.dims - 2, -1, -1):
            f = f * self.geom.size[a] + idx[..., a]
        return f

    def for_each_active(self):
        """Yields (node_index tuple, ordinal, offset) in the reference order."""
        act = self.active_bool()
        idx = self.node_indices()
        for j in range(act.shape[0]):
            for off in np.nonzero(act[j])[0]:
                yield tuple(int(v) for v in idx[j, off]), j, int(off)

    def close(self, keep: bool = True):
        """Drop the device mirror. keep=True first pulls every property the
        device advanced, so the host grid stays the full state; keep=False
        discards them (temporary grids, e.g. the D_eff fit's free boxes)."""
        if self._dev is not None:
            if keep:
                self._sync_host()
            else:
                self._dev_newer = set()
            self._dev.close()
            self._dev = None
            self._host_newer = True

    def __del__(self):
        try:
            if self._dev is not None:
                self._dev.close()
        except Exception:
            pass


class DeviceGrid:
    """Owning handle of a pd_grid (device sparse block grid)."""

    def __init__(self, handle, geometry: GridGeometry, dtype, n_chunks: int, n_props: int):
        self.h = handle
        self.geom = geometry
        self.dtype = np.dtype(dtype)
        self.n_chunks = n_chunks
        self.n_props = n_props
        self.V = 512 if geometry.dims == 3 else 64

    @classmethod
    def create(cls, geom, dtype, keys, masks, n_props, device=0) -> "DeviceGrid":
        size = (C.c_int64 * 3)(*(list(geom.size) + [1] * (3 - geom.dims)))
        spacing = (C.c_double * 3)(*(list(geom.spacing) + [1.0] * (3 - geom.dims)))
        keys = np.ascontiguousarray(keys, np.int32)
        masks = np.ascontiguousarray(masks, np.uint64)
        h = C.c_void_p()
        _check(lib.pd_grid_create(geom.dims, np.dtype(dtype).itemsize, size, spacing, len(keys),
                                  keys.ctypes.data, masks.ctypes.data, n_props, device, C.byref(h)))
        return cls(h, geom, dtype, len(keys), n_props)

    @classmethod
    def sphere_pack(cls, geom: GridGeometry, centers, radii, band: PhaseBand = PhaseBand(),
                    n_props: int = 4, prop_phi: int = 0, dtype=np.float64, device=0) -> "DeviceGrid":
        """build_sparse_grid(field_from(pack.fluid_sdf)) on the device."""
        centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        radii = np.ascontiguousarray(radii, np.float64)
        size = (C.c_int64 * 3)(*geom.size)
        spacing = (C.c_double * 3)(*geom.spacing)
        origin = (C.c_double * 3)(*geom.origin)
        h = C.c_void_p()
        _check(lib.pd_build_sphere_pack_grid(
            np.dtype(dtype).itemsize, size, spacing, origin, len(radii),
            centers.ctypes.data_as(C.POINTER(C.c_double)), radii.ctypes.data_as(C.POINTER(C.c_double)),
            band.b_low, band.b_up, n_props, prop_phi, device, C.byref(h)))
        n = C.c_int64()
        lib.pd_grid_info(h, C.byref(n), None)
        return cls(h, geom, dtype, int(n.value), n_props)

    def info(self):
        n, a = C.c_int64(), C.c_int64()
        lib.pd_grid_info(self.h, C.byref(n), C.byref(a))
        return int(n.value), int(a.value)

    def layout(self):
        dims = self.geom.dims
        keys = np.zeros((self.n_chunks, dims), np.int32)
        masks = np.zeros((self.n_chunks, self.V // 64), np.uint64)
        _check(lib.pd_grid_download_layout(self.h, keys.ctypes.data, masks.ctypes.data))
        return keys, masks

    def upload(self, prop: int, slabs: np.ndarray):
        a = np.ascontiguousarray(slabs, self.dtype)
        assert a.size == self.n_chunks * self.V
        _check(lib.pd_grid_upload(self.h, prop, a.ctypes.data))

    def download(self, prop: int) -> np.ndarray:
        out = np.empty((self.n_chunks, self.V), self.dtype)
        _check(lib.pd_grid_download(self.h, prop, out.ctypes.data))
        return out

    def download_into(self, prop: int, out: np.ndarray) -> None:
        assert out.shape == (self.n_chunks, self.V) and out.dtype == self.dtype and out.flags.c_contiguous
        _check(lib.pd_grid_download(self.h, prop, out.ctypes.data))

    def device_ptr(self, prop: int) -> int:
        p = C.c_void_p()
        _check(lib.pd_grid_device_ptr(self.h, prop, C.byref(p)))
        return int(p.value or 0)

    def total_mass(self, prop: int) -> float:
        out = C.c_double()
        _check(lib.pd_grid_total_mass(self.h, prop, C.byref(out)))
        return out.value

    def max_active(self, prop: int) -> float:
        out = C.c_double()
        _check(lib.pd_grid_max_active(self.h, prop, C.byref(out)))
        return out.value

    def populate_diffusion(self, prop_phi: int, prop_d: int, profile: DiffusionProfile):
        _check(lib.pd_grid_populate_diffusion(self.h, prop_phi, prop_d, profile.d_min, profile.d_max,
                                              profile.gamma1, profile.gamma2))

    def fill_hash(self, prop: int, seed: int):
        _check(lib.pd_grid_fill_hash(self.h, prop, seed))

    def fill_const(self, prop: int, value: float):
        _check(lib.pd_grid_fill_const(self.h, prop, value))

    @classmethod
    def full(cls, geom: GridGeometry, n_props: int, prop_phi: int = -1, phi_value: float = 0.0,
             dtype=np.float64, device=0) -> "DeviceGrid":
        """Every node active (build_free_box_grid, analysis.hpp:147-153)."""
        size = (C.c_int64 * 3)(*(list(geom.size) + [1] * (3 - geom.dims)))
        spacing = (C.c_double * 3)(*(list(geom.spacing) + [1.0] * (3 - geom.dims)))
        h = C.c_void_p()
        _check(lib.pd_grid_create_full(geom.dims, np.dtype(dtype).itemsize, size, spacing, n_props, prop_phi,
                                       phi_value, device, C.byref(h)))
        n = C.c_int64()
        lib.pd_grid_info(h, C.byref(n), None)
        return cls(h, geom, dtype, int(n.value), n_props)

    @staticmethod
    def _box(lo, hi):
        return (C.c_int64 * 3)(*(list(lo) + [0] * (3 - len(lo)))), (C.c_int64 * 3)(*(list(hi) + [1] * (3 - len(hi))))

    def box_sum(self, prop: int, lo, hi) -> float:
        """Lexicographic sequential sum of the active values in [lo, hi)."""
        a, b = self._box(lo, hi)
        out = C.c_double()
        _check(lib.pd_grid_box_sum(self.h, prop, a, b, C.byref(out)))
        return out.value

    def frap_init(self, prop_u: int, prop_d: int, lo, hi, d_molecular: float):
        a, b = self._box(lo, hi)
        region, phase = C.c_int64(), C.c_int64()
        _check(lib.pd_grid_frap_init(self.h, prop_u, prop_d, a, b, d_molecular, C.byref(region), C.byref(phase)))
        return int(region.value), int(phase.value)

    def close(self):
        if self.h is not None and self.h.value:
            lib.pd_grid_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# stepper (solver.hpp:183-467) and orchestration (solver.hpp:469-519)
# ---------------------------------------------------------------------------


def _to_c_config(cfg: SimulationConfig, src_prop: int) -> _lib.pd_sim_config:
    c = _lib.pd_sim_config()
    c.dt = cfg.dt
    c.n_steps = cfg.n_steps
    c.b_low = cfg.phase_band.b_low
    c.b_up = cfg.phase_band.b_up
    c.boundary_epsilon = cfg.boundary_epsilon
    kind = cfg.reaction.kind
    c.reaction_kind = {"none": 0, "surface_sink": 1, "volumetric": 2}[kind]
    c.source_prop = src_prop
    c.rate = cfg.reaction.rate
    c.band_half_width = cfg.reaction.band_half_width
    for f in range(6):
        bc = cfg.outer_bc[f] if f < len(cfg.outer_bc) else FaceBc()
        c.bc_type[f] = 1 if bc.type == "dirichlet" else 0
        c.bc_value[f] = bc.value
    c.record_every = cfg.record_every
    c.enforce_stability = 1 if cfg.enforce_stability else 0
    c.has_time_factor = 1 if cfg.reaction.time_factor is not None else 0
    return c


def _validate(grid: SparseBlockGrid, cfg: SimulationConfig) -> None:
    """solver.hpp:304-331 (the C ABI repeats the numeric checks; the
    name-based ones live here, like in the reference)."""
    if not (cfg.dt > 0.0) or not math.isfinite(cfg.dt):
        raise InputError("time step must be positive and finite")
    if cfg.n_steps < 1:
        raise InputError("step count must be at least 1")
    if cfg.record_every < 1:
        raise InputError("record_every must be at least 1")
    if not (cfg.phase_band.b_low < cfg.phase_band.b_up):
        raise InputError("phase band is empty (b_low must be < b_up)")
    if cfg.boundary_epsilon < 0.0 or not math.isfinite(cfg.boundary_epsilon):
        raise InputError("boundary_epsilon must be finite and >= 0")
    if cfg.reaction.kind == "surface_sink":
        if cfg.reaction.rate < 0.0:
            raise InputError("surface sink rate must be >= 0")
        if not (cfg.reaction.band_half_width > 0.0):
            raise InputError("surface sink band half-width must be > 0")
    for ch in ("phi", "u", "D", scratch_channel):
        try:
            grid.property_index(ch)
        except PropertyError:
            raise InputError(f"grid lacks the '{ch}' channel; build simulation grids with channels "
                             "{phi, u, D, u_next}") from None
    if cfg.reaction.kind == "volumetric":
        grid.property_index(cfg.reaction.source_channel)


class FtcsStepper:
    """FtcsStepper<T,Dims> (solver.hpp:183-467) backed by the device."""

    def __init__(self, grid: SparseBlockGrid, config: SimulationConfig, device: int = 0):
        _validate(grid, config)
        self.grid = grid
        self.cfg = config
        self.dev = grid.device(device)
        src = grid.property_index(config.reaction.source_channel) if config.reaction.kind == "volumetric" else -1
        self._ccfg = _to_c_config(config, src)
        self.h = C.c_void_p()
        _check(lib.pd_stepper_create(self.dev.h, C.byref(self._ccfg), grid.property_index("phi"),
                                     grid.property_index("u"), grid.property_index("D"),
                                     grid.property_index(scratch_channel), C.byref(self.h)))

    def config(self) -> SimulationConfig:
        return self.cfg

    def stability_bound(self) -> float:
        out = C.c_double()
        _check(lib.pd_stepper_stability_bound(self.h, C.byref(out)))
        return out.value

    def snapshot_diagnostics(self) -> StepDiagnostics:
        d = _lib.pd_diag()
        _check(lib.pd_stepper_snapshot_diag(self.h, C.byref(d)))
        return StepDiagnostics(0, 0.0, d.total_mass, d.min_u, d.max_u)

    def _factors(self, step0: int, n: int):
        tf = self.cfg.reaction.time_factor
        if self.cfg.reaction.kind != "volumetric" or tf is None:
            return None
        arr = (C.c_double * n)(*[float(tf(float(step0 + k) * self.cfg.dt)) for k in range(n)])
        return arr

    def run(self, step0: int, n_steps: int, final_step: int) -> List[StepDiagnostics]:
        """Advances n_steps; returns the rows of the steps run_simulation
        records (solver.hpp:516)."""
        rows = (_lib.pd_diag * max(1, n_steps))()
        nr = C.c_int64()
        fac = self._factors(step0, n_steps)
        t0 = _time.perf_counter()
        rc = lib.pd_stepper_run(self.h, step0, n_steps, final_step, fac, rows, C.byref(nr))
        self.grid._mark_device_newer(["u", scratch_channel])
        _check(rc)
        wall = _time.perf_counter() - t0
        return [StepDiagnostics(r.step, r.time, r.total_mass, r.min_u, r.max_u, wall)
                for r in rows[: nr.value]]

    def step(self, step_index: int = 0) -> StepDiagnostics:
        """One validated step with diagnostics (solver.hpp:228-279): a
        non-finite node raises NumericError; a non-finite total mass is
        returned in the row (only run_simulation checks it)."""
        row = _lib.pd_diag()
        fac = self._factors(step_index, 1)
        t0 = _time.perf_counter()
        rc = lib.pd_stepper_step(self.h, step_index, fac[0] if fac is not None else 1.0, C.byref(row))
        self.grid._mark_device_newer(["u", scratch_channel])
        _check(rc)
        return StepDiagnostics(row.step, row.time, row.total_mass, row.min_u, row.max_u,
                               _time.perf_counter() - t0)

    def set_region(self, lo, hi):
        a, b = DeviceGrid._box(lo, hi)
        _check(lib.pd_stepper_set_region(self.h, a, b))
        self._has_region = True

    def region_sums(self) -> List[float]:
        if not getattr(self, "_has_region", False):
            return []
        n = C.c_int64()
        lib.pd_stepper_region_sums(self.h, None, 0, C.byref(n))
        buf = (C.c_double * max(1, n.value))()
        lib.pd_stepper_region_sums(self.h, buf, n.value, C.byref(n))
        return list(buf[: n.value])

    # -- steady-state observers (pd_observe.cu; no reference counterpart) ---
    def set_convergence(self, on: bool = True):
        """Every recorded row also yields max |u(step) - u(step-1)|."""
        _check(lib.pd_stepper_set_convergence(self.h, 1 if on else 0))

    def convergence_norms(self) -> List[float]:
        n = C.c_int64()
        lib.pd_stepper_convergence(self.h, None, 0, C.byref(n))
        buf = (C.c_double * max(1, n.value))()
        lib.pd_stepper_convergence(self.h, buf, n.value, C.byref(n))
        return list(buf[: n.value])

    def plane_flux(self, axis: int, layer: int) -> Tuple[float, float]:
        """(face_sum, flux) of the current u through the plane between node
        layers `layer` and `layer`+1 of `axis` (pd_stepper_plane_flux)."""
        fs, fl = C.c_double(), C.c_double()
        nf = C.c_int64()
        _check(lib.pd_stepper_plane_flux(self.h, axis, layer, C.byref(fs), C.byref(fl), C.byref(nf)))
        return fs.value, fl.value

    def last_ms(self) -> float:
        ms = C.c_double()
        lib.pd_stepper_last_ms(self.h, C.byref(ms))
        return ms.value

    def launches(self) -> int:
        n = C.c_int64()
        lib.pd_stepper_launch_count(self.h, C.byref(n))
        return int(n.value)

    def close(self):
        if self.h is not None and self.h.value:
            lib.pd_stepper_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ftcs_step(grid: SparseBlockGrid, config: SimulationConfig, step_index: int = 0) -> StepDiagnostics:
    """solver.hpp:470-475: one step, no stability gate, no record."""
    s = FtcsStepper(grid, config)
    try:
        return s.step(step_index)
    finally:
        s.close()


def max_diffusivity(grid: SparseBlockGrid, channel: str = "D") -> float:
    """solver.hpp:139-154, on the device."""
    return grid.device().max_active(grid.property_index(channel))


def total_mass(grid: SparseBlockGrid, channel: str = "u") -> float:
    """solver.hpp:158-171, on the device."""
    return grid.device().total_mass(grid.property_index(channel))


def run_simulation(grid: SparseBlockGrid, config: SimulationConfig,
                   observers: Sequence[Callable[[SparseBlockGrid, StepDiagnostics], None]] = (),
                   region: Optional[Tuple[Sequence[int], Sequence[int]]] = None) -> SimulationResult:
    """solver.hpp:489-519. ``region=(lo, hi)`` attaches the device
    region-mass observer of run_frap (analysis.hpp:211-219): the result then
    carries the box sum of u for every diagnostics row."""
    stepper = FtcsStepper(grid, config)
    sums: List[float] = []
    if region is not None:
        stepper.set_region(*region)
    try:
        if config.enforce_stability:
            bound = stepper.stability_bound()
            if not (config.dt < bound):
                dmax = max_diffusivity(grid)
                raise StabilityError(
                    f"time step {format_scalar(config.dt)} violates the explicit stability bound "
                    f"{format_scalar(bound)} (dt must be strictly below it; max D = {format_scalar(dmax)})")
        diags: List[StepDiagnostics] = []

        def record(d):
            diags.append(d)
            for obs in observers:
                obs(grid, d)

        record(stepper.snapshot_diagnostics())
        if region is not None:
            sums.append(stepper.dev.box_sum(grid.property_index("u"), *region))
        n = config.n_steps
        if not observers:
            diags.extend(stepper.run(0, n, n))
            sums.extend(stepper.region_sums())
        else:
            s = 0
            while s < n:
                # run up to and including the next recorded step
                nxt = min(n, ((s // config.record_every) + 1) * config.record_every)
                for d in stepper.run(s, nxt - s, n):
                    record(d)
                sums.extend(stepper.region_sums())
                s = nxt
        return SimulationResult(diags, sums)
    finally:
        stepper.close()


# ---------------------------------------------------------------------------
# host geometry stage (geometry.hpp:148-206; the device builder for sphere
# packs is DeviceGrid.sphere_pack)
# ---------------------------------------------------------------------------


def build_sparse_grid(sdf: np.ndarray, geometry: GridGeometry, band: PhaseBand = PhaseBand(),
                      channels: Sequence[str] = ("phi", "u", "D"), dtype=np.float64) -> SparseBlockGrid:
    """Inserts b_low+eps < phi < b_up-eps (T arithmetic, eps of T); phi copied
    into "phi", other channels zero (geometry.hpp:148-176)."""
    if not (band.b_low < band.b_up):
        raise InputError("phase band is empty: lower bound must be below upper bound")
    T = np.dtype(dtype).type
    phi = np.asarray(sdf).reshape(-1).astype(T)
    if not np.all(np.isfinite(np.asarray(sdf))):
        raise InputError("level-set field contains non-finite values")
    if "phi" not in channels:
        raise InputError('channel list must contain "phi" to receive the level set')
    eps = np.finfo(T).eps
    lo = T(T(band.b_low) + eps)
    hi = T(T(band.b_up) - eps)
    act = (phi > lo) & (phi < hi)
    flat = np.nonzero(act)[0]
    if flat.size == 0:
        raise InputError("no node lies inside the phase band: the grid would be empty")
    dims = geometry.dims
    idx = []
    rem = flat.copy()
    for a in range(dims):
        idx.append(rem % geometry.size[a])
        rem //= geometry.size[a]
    cc = [(s + 7) // 8 for s in geometry.size]
    lin = np.zeros_like(flat)
    off = np.zeros_like(flat)
    for a in range(dims - 1, -1, -1):
        lin = lin * cc[a] + (idx[a] >> 3)
        off = off | ((idx[a] & 7) << (3 * a))
    ulin, inv = np.unique(lin, return_inverse=True)
    keys = np.zeros((len(ulin), dims), np.int32)
    r = ulin.copy()
    for a in range(dims):
        keys[:, a] = r % cc[a]
        r //= cc[a]
    V = 512 if dims == 3 else 64
    W = V // 64
    masks = np.zeros((len(ulin), W), np.uint64)
    np.bitwise_or.at(masks, (inv, off >> 6), (np.uint64(1) << (off & 63).astype(np.uint64)))
    phis = np.zeros((len(ulin), V), T)
    phis[inv, off] = phi[flat]
    return SparseBlockGrid.from_layout(geometry, list(channels), keys, masks, {"phi": phis}, dtype)


def smooth_diffusion_coefficient(phi: float, profile: DiffusionProfile) -> float:
    """geometry.hpp:182-187 (libm exp, like the reference)."""
    if profile.d_min < 0.0:
        raise InputError("d_min must be non-negative")
    if not (profile.d_max > 0.0):
        raise InputError("d_max must be positive")
    return profile.d_min + profile.d_max / (1.0 + math.exp(-(profile.gamma1 + profile.gamma2 * phi)))


def populate_diffusion_channel(grid: SparseBlockGrid, profile: DiffusionProfile,
                               phi_channel: str = "phi", d_channel: str = "D") -> None:
    """geometry.hpp:191-206 on the host with libm exp (bit-identical to the
    reference); use DeviceGrid.populate_diffusion for large grids."""
    phi = grid.channel_data(phi_channel)
    d = grid.channel_data(d_channel, writable=True)
    act = grid.active_bool()
    T = grid.dtype.type
    vals = [T(smooth_diffusion_coefficient(float(p), profile)) for p in phi[act]]
    d[act] = np.array(vals, grid.dtype)
