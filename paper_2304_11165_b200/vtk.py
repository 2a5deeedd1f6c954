"""Legacy ASCII VTK export (reference vtk.hpp:25-250, scalar_text.hpp:20-55;
SURVEY.md §8f row 4) with every node's text produced on the device.

    write_vtk(ds, path)            vtk.hpp:57-111   dataset of host arrays
    vtk_from_sparse(grid, ...)     vtk.hpp:115-143  densified on the device
    write_grid_vtk(grid, path,...) write_vtk(vtk_from_sparse(...)) fused: the
                                   lattice is formatted straight from the
                                   device grid, nothing dense touches the host
    write_field_vtk(field, path)   a DeviceField (level set) as one array
    read_vtk(path)                 vtk.hpp:181-248 (host parser; verification)
    format_scalar(v)               scalar_text.hpp:20-28 (the device formatter)

Files are byte-identical to the reference writer's: "%.17g" ("%.9g" for
float) exactly rounded like glibc, "nan" for every NaN, the same header lines
and array order (tests/test_vtk.py compares whole files with oracle/_ref).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import porediff as pd
from ._lib import lib
from .porediff import InputError, IoError, _check

DEFAULT_TITLE = "porediff field export"


def format_scalar(v: float, dtype=np.float64) -> str:
    """scalar_text.hpp:20-28, evaluated by the same routine the device runs."""
    buf = C.create_string_buffer(32)
    n = C.c_int()
    _check(lib.pd_format_scalar(float(v), np.dtype(dtype).itemsize, buf, len(buf), C.byref(n)))
    return buf.value.decode()


def parse_scalar(token: str, dtype=np.float64):
    """scalar_text.hpp:33-46 (float tokens parse straight to float32)."""
    try:
        if token.strip() != token or not token:
            raise ValueError
        v = float(token)
    except ValueError:
        raise InputError(f"malformed numeric token '{token}'") from None
    return np.float32(np.float64(v)) if np.dtype(dtype).itemsize == 4 else v


@dataclass
class VtkDataset:
    """vtk.hpp:28-37: a dense lattice plus named point-data arrays."""
    geometry: pd.GridGeometry
    scalars: List[Tuple[str, np.ndarray]] = field(default_factory=list)
    mask: Optional[np.ndarray] = None  # int32, None = no mask array
    dtype: np.dtype = np.dtype(np.float64)

    def add_scalar(self, name: str, values) -> None:
        self.scalars.append((name, np.ascontiguousarray(values, self.dtype).reshape(-1)))


def _check_name(name: str) -> None:
    """vtk.hpp:46-51."""
    if not name:
        raise InputError("VTK array name must not be empty")
    if any(c in name for c in " \t\n\r"):
        raise InputError(f"VTK array name '{name}' contains whitespace")


def _lattice(geom: pd.GridGeometry):
    d = geom.dims
    size = (C.c_int64 * 3)(*(list(geom.size) + [1] * (3 - d)))
    spacing = (C.c_double * 3)(*(list(geom.spacing) + [1.0] * (3 - d)))
    origin = (C.c_double * 3)(*(list(geom.origin) + [0.0] * (3 - d)))
    return size, spacing, origin


def write_vtk(ds: VtkDataset, path: str, title: str = DEFAULT_TITLE, device: int = 0) -> None:
    """vtk.hpp:57-111: checks in the reference's order, then the node texts
    are formatted on the device and streamed to `path`."""
    n = ds.geometry.node_count()
    if not ds.scalars and (ds.mask is None or len(ds.mask) == 0):
        raise InputError("VTK dataset has no arrays to write")
    for name, values in ds.scalars:
        _check_name(name)
        if len(values) != n:
            raise InputError(f"VTK array '{name}' holds {len(values)} values, lattice has {n} nodes")
    for i in range(len(ds.scalars)):
        for k in range(i + 1, len(ds.scalars)):
            if ds.scalars[i][0] == ds.scalars[k][0]:
                raise InputError(f"duplicate VTK array name '{ds.scalars[i][0]}'")
    mask = None
    if ds.mask is not None and len(ds.mask) > 0:
        if len(ds.mask) != n:
            raise InputError("VTK mask array size mismatch")
        mask = np.ascontiguousarray(ds.mask, np.int32)
    tb = np.dtype(ds.dtype).itemsize
    arrays = [np.ascontiguousarray(v, ds.dtype) for _, v in ds.scalars]
    names = (C.c_char_p * max(1, len(arrays)))(*[nm.encode() for nm, _ in ds.scalars])
    vals = (C.c_void_p * max(1, len(arrays)))(*[a.ctypes.data for a in arrays])
    size, spacing, origin = _lattice(ds.geometry)
    _check(lib.pd_write_vtk(str(path).encode(), title.encode(), ds.geometry.dims, size, spacing, origin, tb,
                            len(arrays), names, vals, 0, mask.ctypes.data if mask is not None else None, device))


def _channels(grid: pd.SparseBlockGrid, channels: Optional[Sequence[str]]):
    chans = list(channels) if channels else grid.property_names()
    return chans, [grid.property_index(c) for c in chans]  # PropertyError on unknown names


def vtk_from_sparse(grid: pd.SparseBlockGrid, channels: Optional[Sequence[str]] = None,
                    blank: float = math.nan) -> VtkDataset:
    """vtk.hpp:115-143: the chosen channels (default all) on the full
    lattice, inactive nodes = blank, mask 1 = active; densified on the device."""
    chans, idx = _channels(grid, channels)
    dev = grid.device()
    n = grid.geometry().node_count()
    ds = VtkDataset(grid.geometry(), dtype=grid.dtype)
    for name, p in zip(chans, idx):
        v = np.empty(n, grid.dtype)
        _check(lib.pd_grid_densify(dev.h, p, float(blank), v.ctypes.data, None))
        ds.scalars.append((name, v))
    ds.mask = np.empty(n, np.int32)
    _check(lib.pd_grid_densify(dev.h, 0, float(blank), None, ds.mask.ctypes.data))
    return ds


def write_grid_vtk(grid: pd.SparseBlockGrid, path: str, channels: Optional[Sequence[str]] = None,
                   blank: float = math.nan, title: str = DEFAULT_TITLE) -> None:
    """write_vtk(vtk_from_sparse(grid, channels, blank), path, title) with the
    lattice formatted directly from the device grid."""
    chans, idx = _channels(grid, channels)
    for c in chans:
        _check_name(c)
    for i in range(len(chans)):
        for k in range(i + 1, len(chans)):
            if chans[i] == chans[k]:
                raise InputError(f"duplicate VTK array name '{chans[i]}'")
    dev = grid.device()
    geom = grid.geometry()
    names = (C.c_char_p * max(1, len(chans)))(*[c.encode() for c in chans])
    props = (C.c_int * max(1, len(idx)))(*idx)
    _, _, origin = _lattice(geom)
    _check(lib.pd_grid_write_vtk(dev.h, str(path).encode(), title.encode(), props, names, len(chans), float(blank),
                                 origin))


def write_field_vtk(f, path: str, name: str = "phi", title: str = DEFAULT_TITLE) -> None:
    """A DeviceField (levelset.DeviceField) as a one-array dataset, formatted
    from device memory."""
    _check_name(name)
    ptr = C.c_void_p()
    _check(lib.pd_field_device_ptr(f.h, C.byref(ptr)))
    size, spacing, origin = _lattice(f.geom)
    names = (C.c_char_p * 1)(name.encode())
    vals = (C.c_void_p * 1)(ptr.value)
    _check(lib.pd_write_vtk(str(path).encode(), title.encode(), f.geom.dims, size, spacing, origin, f.dtype.itemsize,
                            1, names, vals, 1, None, getattr(f, "device", 0)))


# ---- reader (vtk.hpp:145-248; host, verification) -------------------------

@dataclass
class VtkScalarArray:
    name: str
    type: str
    tokens: List[str]

    def as_(self, dtype):
        dt = np.dtype(dtype)
        if dt.kind in "iu":
            out = []
            for t in self.tokens:
                try:
                    out.append(int(t))
                except ValueError:
                    raise InputError(f"malformed integer token '{t}'") from None
            return np.array(out, dt)
        return np.array([parse_scalar(t, dt) for t in self.tokens], dt)


@dataclass
class VtkFile:
    dimensions: List[int] = field(default_factory=lambda: [1, 1, 1])
    origin: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    spacing: List[float] = field(default_factory=lambda: [1.0, 1.0, 1.0])
    point_count: int = 0
    arrays: List[VtkScalarArray] = field(default_factory=list)

    def array(self, name: str) -> VtkScalarArray:
        for a in self.arrays:
            if a.name == name:
                return a
        raise InputError(f"VTK file has no array named '{name}'")


def read_vtk(path: str) -> VtkFile:
    """vtk.hpp:183-248: the STRUCTURED_POINTS / SCALARS subset write_vtk emits."""
    try:
        fh = open(path, "r", newline="\n")
    except OSError:
        raise IoError(f"cannot open '{path}' for reading") from None
    where = f"VTK file '{path}'"
    with fh:
        first = fh.readline()
        if not first.startswith("# vtk DataFile"):
            raise InputError(f"{where}: missing '# vtk DataFile' header")
        if not fh.readline():
            raise InputError(f"{where}: missing title line")
        toks = fh.read().split()
    pos = 0

    def nxt(what):
        nonlocal pos
        if pos >= len(toks):
            raise InputError(f"{where}: unexpected end of file, wanted {what}")
        pos += 1
        return toks[pos - 1]

    def integer(t):
        try:
            return int(t)
        except ValueError:
            raise InputError(f"malformed integer token '{t}'") from None

    if nxt("format") != "ASCII":
        raise InputError(f"{where}: only ASCII format is supported")
    if nxt("DATASET") != "DATASET" or nxt("dataset type") != "STRUCTURED_POINTS":
        raise InputError(f"{where}: only DATASET STRUCTURED_POINTS is supported")
    f = VtkFile()
    while True:
        kw = nxt("geometry keyword or POINT_DATA")
        if kw == "POINT_DATA":
            break
        if kw == "DIMENSIONS":
            f.dimensions = [integer(nxt("dimension")) for _ in range(3)]
        elif kw == "ORIGIN":
            f.origin = [parse_scalar(nxt("origin component")) for _ in range(3)]
        elif kw in ("SPACING", "ASPECT_RATIO"):
            f.spacing = [parse_scalar(nxt("spacing component")) for _ in range(3)]
        else:
            raise InputError(f"{where}: unsupported keyword '{kw}'")
    f.point_count = integer(nxt("point count"))
    if f.point_count != f.dimensions[0] * f.dimensions[1] * f.dimensions[2]:
        raise InputError(f"{where}: POINT_DATA count does not match DIMENSIONS")
    while pos < len(toks):
        tok = nxt("SCALARS")
        if tok != "SCALARS":
            raise InputError(f"{where}: unsupported point-data section '{tok}'")
        name = nxt("array name")
        typ = nxt("array type")
        ct = nxt("component count or LOOKUP_TABLE")
        comps = 1
        if ct != "LOOKUP_TABLE":
            comps = integer(ct)
            if comps < 1 or comps > 9:
                raise InputError(f"{where}: bad component count for array '{name}'")
            if nxt("LOOKUP_TABLE") != "LOOKUP_TABLE":
                raise InputError(f"{where}: expected LOOKUP_TABLE after SCALARS line")
        nxt("lookup table name")
        want = f.point_count * comps
        if pos + want > len(toks):
            pos = len(toks)
            nxt("array value")
        f.arrays.append(VtkScalarArray(name, typ, toks[pos:pos + want]))
        pos += want
    return f
