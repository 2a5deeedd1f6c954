"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Ref``  -> oracle/_ref/libporediff_ref.so: the UNMODIFIED reference headers
  compiled in place (oracle/Makefile). Its outputs are the ground truth.
* ``Port`` -> oracle/build/libftcs_oracle.so: the plain-C restatement
  (oracle/ftcs_oracle.c), itself pinned against Ref and tests/golden.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
--impl reference) may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libporediff_ref.so"
PORT_SO = HERE / "build" / "libftcs_oracle.so"


class pd_sim_config(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("n_steps", C.c_int64), ("b_low", C.c_double), ("b_up", C.c_double),
        ("boundary_epsilon", C.c_double), ("reaction_kind", C.c_int32), ("source_prop", C.c_int32),
        ("rate", C.c_double), ("band_half_width", C.c_double), ("bc_type", C.c_int32 * 6),
        ("bc_value", C.c_double * 6), ("record_every", C.c_int64), ("enforce_stability", C.c_int32),
        ("has_time_factor", C.c_int32),
    ]


class pd_diag(C.Structure):
    _fields_ = [("step", C.c_int64), ("time", C.c_double), ("total_mass", C.c_double),
                ("min_u", C.c_double), ("max_u", C.c_double)]


TF = C.CFUNCTYPE(C.c_double, C.c_double)


def make_config(dt, n_steps, *, b_low=0.0, b_up=float("inf"), boundary_epsilon=0.0, reaction="none",
                rate=0.0, band_half_width=1.0, source_prop=-1, bc=None, record_every=1,
                enforce_stability=True) -> pd_sim_config:
    c = pd_sim_config()
    c.dt, c.n_steps, c.b_low, c.b_up = dt, n_steps, b_low, b_up
    c.boundary_epsilon = boundary_epsilon
    c.reaction_kind = {"none": 0, "surface_sink": 1, "volumetric": 2}[reaction]
    c.rate, c.band_half_width, c.source_prop = rate, band_half_width, source_prop
    for f in range(6):
        t, v = (bc or {}).get(f, ("no_flux", 0.0))
        c.bc_type[f] = 1 if t == "dirichlet" else 0
        c.bc_value[f] = v
    c.record_every = record_every
    c.enforce_stability = 1 if enforce_stability else 0
    return c


def _arr(x, dt):
    return np.ascontiguousarray(x, dt)


import collections

_KEEP = collections.deque(maxlen=64)  # arrays whose pointers are in flight


def _p(x, dt):
    """Pointer to a contiguous copy that stays alive until the next _release()."""
    a = np.ascontiguousarray(x, dt)
    _KEEP.append(a)
    return a.ctypes.data


def _release():
    _KEEP.clear()


class Ref:
    """The reference itself (header-only C++ compiled unmodified)."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref with /root/reference present)")
        L = self.L = C.CDLL(str(REF_SO))
        P = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_hash_unit_value.restype = C.c_double
        L.ref_hash_unit_value.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_pairwise_sum.restype = C.c_double
        L.ref_pairwise_sum.argtypes = [P, C.c_int64]
        L.ref_stability_dt.restype = C.c_double
        L.ref_stability_dt.argtypes = [C.c_int, P, C.c_double, C.POINTER(C.c_int)]
        L.ref_sphere_packing.argtypes = [P, P, C.c_int, C.c_double, C.c_double, C.c_uint32, P, P]
        L.ref_field_sphere_pack.argtypes = [P, P, P, C.c_int, P, P, P]
        L.ref_field_ball.argtypes = [C.c_int, P, P, P, P, C.c_double, C.c_double, P]
        L.ref_grid_from_sdf.restype = P
        L.ref_grid_from_sdf.argtypes = [C.c_int, C.c_int, P, P, P, P, C.c_double, C.c_double, C.c_int, P, C.POINTER(C.c_int)]
        L.ref_grid_from_chunks.restype = P
        L.ref_grid_from_chunks.argtypes = [C.c_int, C.c_int, P, P, P, C.c_int, P, C.c_int64, P, P, C.POINTER(C.c_int)]
        L.ref_grid_free.argtypes = [P]
        L.ref_grid_chunk_count.restype = C.c_int64
        L.ref_grid_chunk_count.argtypes = [P]
        L.ref_grid_active_count.restype = C.c_int64
        L.ref_grid_active_count.argtypes = [P]
        L.ref_grid_export_layout.argtypes = [P, P, P]
        L.ref_grid_export_prop.argtypes = [P, C.c_int, P]
        L.ref_grid_import_prop.argtypes = [P, C.c_int, P]
        L.ref_grid_populate_diffusion.argtypes = [P, C.c_double, C.c_double, C.c_double, C.c_double]
        L.ref_grid_fill_hash.argtypes = [P, C.c_int, C.c_uint64]
        L.ref_grid_total_mass.restype = C.c_double
        L.ref_grid_total_mass.argtypes = [P, C.c_int]
        L.ref_grid_max_diffusivity.restype = C.c_double
        L.ref_grid_max_diffusivity.argtypes = [P, C.c_int]
        L.ref_run_simulation.argtypes = [P, C.POINTER(pd_sim_config), P, P, C.POINTER(C.c_int64)]
        L.ref_set_worker_count.argtypes = [C.c_int]
        L.ref_worker_count.restype = C.c_int
        L.ref_frap_fit.argtypes = [P, C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_double, P, P, P, P, P, P]
        L.ref_field_redistance.argtypes = [C.c_int, C.c_int, P, P, P, P, P]
        L.ref_field_filter_thin.argtypes = [C.c_int, C.c_int, P, P, P, C.c_int]
        L.ref_grid_write_snapshot.argtypes = [P, C.c_char_p]
        L.ref_grid_read_snapshot.restype = P
        L.ref_grid_read_snapshot.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_field_write_snapshot.argtypes = [C.c_int, C.c_int, P, P, P, P, C.c_char_p]
        L.ref_grid_write_vtk.argtypes = [P, C.c_char_p, C.c_char_p, C.c_double, P]
        L.ref_write_vtk.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, P, P, P, C.c_int, C.c_char_p, P, P,
                                    C.c_int64]

    def field_redistance(self, size, spacing, values, opts):
        """sussman_redistance on a dense field (axis 0 fastest); returns
        (code, message, field, (iterations, final_residual, converged))."""
        from paper_2304_11165_b200._lib import pd_levelset_options, pd_redistance_diag
        v = np.ascontiguousarray(values).copy()
        o = pd_levelset_options(*opts)
        d = pd_redistance_diag()
        code = self.L.ref_field_redistance(len(size), v.dtype.itemsize, _p(size, np.int64),
                                           _p(list(spacing), np.float64), v.ctypes.data, C.byref(o), C.byref(d))
        return code, self.last_error(), v, (d.iterations, d.final_residual, bool(d.converged))

    def write_dense_snapshot(self, size, spacing, origin, values, path):
        v = np.ascontiguousarray(values)
        code = self.L.ref_field_write_snapshot(len(size), v.dtype.itemsize, _p(size, np.int64), _p(list(spacing), np.float64),
                                               _p(list(origin), np.float64), v.ctypes.data, str(path).encode())
        return code, self.last_error()

    def write_vtk(self, path, size, spacing, origin, arrays, mask=None, title="porediff field export"):
        """write_vtk (vtk.hpp:57-111) of a dense dataset: arrays = [(name, values)]
        (one dtype), mask = int32 values or None."""
        vals = [np.ascontiguousarray(v) for _, v in arrays]
        tb = vals[0].dtype.itemsize if vals else 8
        ptrs = (C.c_void_p * max(1, len(vals)))(*[v.ctypes.data for v in vals])
        m = None if mask is None else np.ascontiguousarray(mask, np.int32)
        code = self.L.ref_write_vtk(str(path).encode(), title.encode(), len(size), tb, _p(size, np.int64),
                                    _p(list(spacing), np.float64), _p(list(origin), np.float64), len(vals),
                                    "\n".join(nm for nm, _ in arrays).encode(), ptrs,
                                    None if m is None else m.ctypes.data, 0 if m is None else len(m))
        return code, self.last_error()

    def read_sparse_snapshot(self, path):
        code = C.c_int()
        h = self.L.ref_grid_read_snapshot(str(path).encode(), C.byref(code))
        if code.value:
            return code.value, self.last_error(), None
        return 0, "", RefGrid(self, h, 3, 8, ["phi", "u", "D", "u_next"])

    def field_filter_thin(self, size, spacing, values, w):
        v = np.ascontiguousarray(values).copy()
        code = self.L.ref_field_filter_thin(len(size), v.dtype.itemsize, _p(size, np.int64),
                                            _p(list(spacing), np.float64), v.ctypes.data, w)
        return code, self.last_error(), v

    def last_error(self):
        return (self.L.ref_last_error() or b"").decode()

    def hash_unit_value(self, seed, key):
        return self.L.ref_hash_unit_value(seed, key)

    def pairwise_sum(self, v):
        v = _arr(v, np.float64)
        return self.L.ref_pairwise_sum(v.ctypes.data, len(v))

    def sphere_packing(self, lo, hi, count, r_min, r_max, seed):
        c = np.zeros((count, 3))
        r = np.zeros(count)
        self.L.ref_sphere_packing(_p(lo, np.float64), _p(hi, np.float64),
                                  count, r_min, r_max, seed, c.ctypes.data, r.ctypes.data)
        return c, r

    def field_sphere_pack(self, size, spacing, origin, centers, radii):
        out = np.zeros(int(np.prod(size)))
        centers = _arr(centers, np.float64)
        radii = _arr(radii, np.float64)
        self.L.ref_field_sphere_pack(_p(size, np.int64), _p(spacing, np.float64),
                                     _p(origin, np.float64), len(radii), centers.ctypes.data,
                                     radii.ctypes.data, out.ctypes.data)
        return out

    def field_ball(self, size, spacing, origin, center, radius, sign=1.0):
        out = np.zeros(int(np.prod(size)))
        self.L.ref_field_ball(len(size), _p(size, np.int64), _p(spacing, np.float64),
                              _p(origin, np.float64), _p(center, np.float64),
                              radius, sign, out.ctypes.data)
        return out

    def grid_from_sdf(self, size, spacing, origin, sdf, b_low=0.0, b_up=float("inf"),
                      channels=("phi", "u", "D", "u_next"), tbytes=8):
        names = (C.c_char_p * len(channels))(*[c.encode() for c in channels])
        code = C.c_int()
        h = self.L.ref_grid_from_sdf(len(size), tbytes, _p(size, np.int64),
                                     _p(spacing, np.float64), _p(origin, np.float64),
                                     _p(sdf, np.float64), b_low, b_up, len(channels), names,
                                     C.byref(code))
        if code.value:
            raise RuntimeError(f"ref_grid_from_sdf: {code.value} {self.last_error()}")
        return RefGrid(self, h, len(size), tbytes, list(channels))

    def grid_from_chunks(self, size, spacing, origin, channels, keys, masks, tbytes=8):
        names = (C.c_char_p * len(channels))(*[c.encode() for c in channels])
        code = C.c_int()
        keys = _arr(keys, np.int32)
        masks = _arr(masks, np.uint64)
        h = self.L.ref_grid_from_chunks(len(size), tbytes, _p(size, np.int64),
                                        _p(spacing, np.float64), _p(origin, np.float64),
                                        len(channels), names, len(keys), keys.ctypes.data, masks.ctypes.data,
                                        C.byref(code))
        if code.value:
            raise RuntimeError(f"ref_grid_from_chunks: {code.value} {self.last_error()}")
        return RefGrid(self, h, len(size), tbytes, list(channels))


class RefGrid:
    def __init__(self, ref: Ref, h, dims, tbytes, channels):
        self.ref, self.h, self.dims, self.tbytes, self.channels = ref, h, dims, tbytes, channels
        self.V = 512 if dims == 3 else 64
        self.dtype = np.float64 if tbytes == 8 else np.float32

    def __del__(self):
        try:
            self.ref.L.ref_grid_free(self.h)
        except Exception:
            pass

    def write_snapshot(self, path):
        return self.ref.L.ref_grid_write_snapshot(self.h, str(path).encode()), self.ref.last_error()

    def write_vtk(self, path, channels=(), blank=float("nan"), origin=None):
        """write_vtk(vtk_from_sparse(grid, channels, blank))."""
        o = None if origin is None else _p(list(origin), np.float64)
        code = self.ref.L.ref_grid_write_vtk(self.h, str(path).encode(), "\n".join(channels).encode(), blank, o)
        return code, self.ref.last_error()

    def chunk_count(self):
        return self.ref.L.ref_grid_chunk_count(self.h)

    def active_count(self):
        return self.ref.L.ref_grid_active_count(self.h)

    def layout(self):
        n = self.chunk_count()
        keys = np.zeros((n, self.dims), np.int32)
        masks = np.zeros((n, self.V // 64), np.uint64)
        self.ref.L.ref_grid_export_layout(self.h, keys.ctypes.data, masks.ctypes.data)
        return keys, masks

    def prop(self, name):
        out = np.zeros((self.chunk_count(), self.V), self.dtype)
        self.ref.L.ref_grid_export_prop(self.h, self.channels.index(name), out.ctypes.data)
        return out

    def set_prop(self, name, slabs):
        a = _arr(slabs, self.dtype)
        self.ref.L.ref_grid_import_prop(self.h, self.channels.index(name), a.ctypes.data)

    def populate_diffusion(self, dmin, dmax, g1, g2):
        rc = self.ref.L.ref_grid_populate_diffusion(self.h, dmin, dmax, g1, g2)
        if rc:
            raise RuntimeError(self.ref.last_error())

    def fill_hash(self, name, seed):
        rc = self.ref.L.ref_grid_fill_hash(self.h, self.channels.index(name), seed)
        if rc:
            raise RuntimeError(self.ref.last_error())

    def total_mass(self, name="u"):
        return self.ref.L.ref_grid_total_mass(self.h, self.channels.index(name))

    def max_diffusivity(self, name="D"):
        return self.ref.L.ref_grid_max_diffusivity(self.h, self.channels.index(name))

    def run(self, cfg: pd_sim_config, time_factor=None):
        """Returns (code, message, rows[list of tuples])."""
        rows = (pd_diag * (cfg.n_steps // max(1, cfg.record_every) + 3))()
        n = C.c_int64()
        tf = TF(time_factor) if time_factor else None
        code = self.ref.L.ref_run_simulation(self.h, C.byref(cfg), C.cast(tf, C.c_void_p) if tf else None,
                                             rows, C.byref(n))
        out = [(r.step, r.time, r.total_mass, r.min_u, r.max_u) for r in rows[: n.value]]
        return code, self.ref.last_error(), out

    def frap_fit(self, bleach_fraction, d_molecular, t_final, n_samples, dt, d_lo, d_hi, rel_tol):
        d_eff, tau, res = C.c_double(), C.c_double(), C.c_double()
        ct = np.zeros(n_samples * 4 + 16)
        cr = np.zeros_like(ct)
        cn = C.c_int64()
        rc = self.ref.L.ref_frap_fit(self.h, bleach_fraction, d_molecular, t_final, n_samples, dt, d_lo, d_hi,
                                     rel_tol, C.byref(d_eff), C.byref(tau), C.byref(res), ct.ctypes.data,
                                     cr.ctypes.data, C.byref(cn))
        if rc:
            raise RuntimeError(self.ref.last_error())
        return d_eff.value, tau.value, res.value, ct[: cn.value], cr[: cn.value]


class Port:
    """The plain-C restatement (oracle/ftcs_oracle.c)."""

    def __init__(self):
        if not PORT_SO.exists():
            raise FileNotFoundError(f"{PORT_SO} not built (make -C oracle port)")
        L = self.L = C.CDLL(str(PORT_SO))
        P = C.c_void_p
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_run_simulation.restype = C.c_int
        L.oracle_run_simulation.argtypes = [C.c_int, C.c_int, P, P, C.c_int64, P, P, P, P, P, P, P,
                                            C.POINTER(pd_sim_config), P, P, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int)]
        L.oracle_total_mass.restype = C.c_double
        L.oracle_total_mass.argtypes = [C.c_int, C.c_int, P, C.c_int64, P, P]
        L.oracle_hash_unit_value.restype = C.c_double
        L.oracle_hash_unit_value.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_pairwise_sum.restype = C.c_double
        L.oracle_pairwise_sum.argtypes = [P, C.c_int64, P]

    def run(self, size, spacing, keys, masks, phi, u, d, u_next, cfg, src=None, factors=None):
        """Runs in place on copies; returns (code, message, rows, u_final, u_next_final)."""
        dims = len(size)
        dtype = np.asarray(u).dtype
        u = np.array(u, dtype, copy=True)
        un = np.array(u_next, dtype, copy=True)
        phi = _arr(phi, dtype)
        d = _arr(d, dtype)
        keys = _arr(keys, np.int32)
        masks = _arr(masks, np.uint64)
        src_p = _p(src, dtype) if src is not None else None
        fac = _p(factors, np.float64) if factors is not None else None
        rows = (pd_diag * (cfg.n_steps // max(1, cfg.record_every) + 3))()
        n = C.c_int64()
        sw = C.c_int()
        code = self.L.oracle_run_simulation(dims, dtype.itemsize, _p(size, np.int64),
                                            _p(spacing, np.float64), len(keys), keys.ctypes.data,
                                            masks.ctypes.data, phi.ctypes.data, u.ctypes.data, d.ctypes.data,
                                            un.ctypes.data, src_p, C.byref(cfg), fac, rows, C.byref(n),
                                            C.byref(sw))
        msg = (self.L.oracle_last_error() or b"").decode()
        out = [(r.step, r.time, r.total_mass, r.min_u, r.max_u) for r in rows[: n.value]]
        if sw.value:
            u, un = un, u
        return code, msg, out, u, un
