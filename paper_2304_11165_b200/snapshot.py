"""SBGR / SBGD snapshots (reference snapshot.hpp:195-348)
streamed from / to the device: the bytes are identical to the reference's
write_sparse_snapshot / write_dense_snapshot, and a reference-written file
reads back into a device grid bit for bit (checkpoint / resume)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib
from . import porediff as pd
from ._lib import lib
from .levelset import DeviceField
from .porediff import _check


@dataclass
class SnapshotInfo:
    """snapshot.hpp:41-50."""
    magic: str = ""
    version: int = 0
    scalar_bits: int = 0
    dims: int = 0
    size: List[int] = field(default_factory=list)
    spacing: List[float] = field(default_factory=list)
    origin: List[float] = field(default_factory=list)
    properties: List[str] = field(default_factory=list)


def write_sparse_snapshot(grid: pd.SparseBlockGrid, path: str) -> None:
    """Payloads in registration order regardless of channel swaps."""
    dev = grid.device()
    names = (C.c_char_p * len(grid.props))(*[p.encode() for p in grid.props])
    geom = grid.geometry()
    origin = (C.c_double * 3)(*(list(geom.origin) + [0.0] * (3 - geom.dims)))
    _check(lib.pd_grid_write_snapshot(dev.h, str(path).encode(), names, len(grid.props), origin))


def read_sparse_snapshot(path: str, dtype=np.float64, dims: int = 3, device: int = 0) -> pd.SparseBlockGrid:
    h = C.c_void_p()
    origin = (C.c_double * 3)()
    buf = C.create_string_buffer(1 << 16)
    n = C.c_int()
    _check(lib.pd_grid_read_snapshot(str(path).encode(), dims, np.dtype(dtype).itemsize, device, C.byref(h), origin,
                                     buf, len(buf), C.byref(n)))
    names = [s.decode() for s in buf.raw.split(b"\0")[: n.value]]
    info = peek_snapshot(path)
    geom = pd.GridGeometry.make(tuple(info.size), tuple(info.spacing), tuple(origin[:dims]))
    nch = C.c_int64()
    lib.pd_grid_info(h, C.byref(nch), None)
    dev = pd.DeviceGrid(h, geom, dtype, int(nch.value), len(names))
    return pd.SparseBlockGrid.from_device(geom, names, dev, dtype)


def write_dense_snapshot(f: DeviceField, path: str) -> None:
    _check(lib.pd_field_write_snapshot(f.h, str(path).encode()))


def read_dense_snapshot(path: str, dtype=np.float64, dims: int = 3, device: int = 0) -> DeviceField:
    info = peek_snapshot(path)
    geom = pd.GridGeometry.make(tuple(info.size), tuple(info.spacing), tuple(info.origin))
    f = DeviceField.__new__(DeviceField)
    f.geom, f.dtype, f.h, f.device = geom, np.dtype(dtype), C.c_void_p(), device
    _check(lib.pd_field_read_snapshot(str(path).encode(), dims, np.dtype(dtype).itemsize, device, C.byref(f.h)))
    return f


def peek_snapshot(path: str) -> SnapshotInfo:
    i = _lib.pd_snapshot_info()
    buf = C.create_string_buffer(1 << 16)
    _check(lib.pd_peek_snapshot(str(path).encode(), C.byref(i), buf, len(buf)))
    d = i.dims
    props = [s.decode() for s in buf.raw.split(b"\0")[: i.n_properties]]
    return SnapshotInfo(i.magic.decode(), i.version, i.scalar_bits, d, list(i.size[:d]), list(i.spacing[:d]),
                        list(i.origin[:d]), props)
