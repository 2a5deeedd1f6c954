"""ctypes binding of the in-tree CUDA library ``lib/libporediff_b200.so``.

This is the reference-side binding a maintainer would add for a Python caller
(the C++ caller uses include/porediff/*.hpp). Every function here is a 1:1
declaration of include/porediff_b200.h. There is deliberately NO fallback:
if the shared library is missing the import fails loudly, and compute entry
points fail with a CUDA error on a host without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libporediff_b200.so"
# kernel A/B experiments load an alternative in-tree build (scripts/gpu_ab_lib.sh)
if os.environ.get("PD_LIB_VARIANT"):
    LIB_PATH = Path(__file__).resolve().parent / "lib" / "variants" / f"{os.environ['PD_LIB_VARIANT']}.so"

PD_OK = 0
PD_E_INPUT = 1
PD_E_BOUNDS = 2
PD_E_PROPERTY = 3
PD_E_IO = 4
PD_E_STABILITY = 5
PD_E_NUMERIC = 6
PD_E_CUDA = 7

PD_REACTION_NONE = 0
PD_REACTION_SURFACE_SINK = 1
PD_REACTION_VOLUMETRIC = 2
PD_BC_NO_FLUX = 0
PD_BC_DIRICHLET = 1


class pd_sim_config(C.Structure):
    _fields_ = [
        ("dt", C.c_double),
        ("n_steps", C.c_int64),
        ("b_low", C.c_double),
        ("b_up", C.c_double),
        ("boundary_epsilon", C.c_double),
        ("reaction_kind", C.c_int32),
        ("source_prop", C.c_int32),
        ("rate", C.c_double),
        ("band_half_width", C.c_double),
        ("bc_type", C.c_int32 * 6),
        ("bc_value", C.c_double * 6),
        ("record_every", C.c_int64),
        ("enforce_stability", C.c_int32),
        ("has_time_factor", C.c_int32),
    ]


class pd_diag(C.Structure):
    _fields_ = [
        ("step", C.c_int64),
        ("time", C.c_double),
        ("total_mass", C.c_double),
        ("min_u", C.c_double),
        ("max_u", C.c_double),
    ]


class pd_levelset_options(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_int32),
        ("tolerance", C.c_double),
        ("pseudo_time_step", C.c_double),
        ("band_width_for_error", C.c_double),
        ("residual_band_width", C.c_double),
        ("rescale_initial", C.c_int32),
    ]


class pd_redistance_diag(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("final_residual", C.c_double), ("converged", C.c_int32)]


class pd_snapshot_info(C.Structure):
    _fields_ = [
        ("magic", C.c_char * 5),
        ("version", C.c_uint32),
        ("scalar_bits", C.c_uint32),
        ("dims", C.c_uint32),
        ("size", C.c_uint64 * 3),
        ("spacing", C.c_double * 3),
        ("origin", C.c_double * 3),
        ("n_properties", C.c_uint32),
    ]


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_DP = C.POINTER(C.c_double)

# (name, restype, argtypes)
_SIGNATURES = [
    ("pd_last_error", C.c_char_p, []),
    ("pd_device_count", C.c_int, []),
    ("pd_version", C.c_char_p, []),
    ("pd_grid_create", C.c_int, [C.c_int, C.c_int, _I64P, _DP, C.c_int64, _P, _P, C.c_int, C.c_int, C.POINTER(_P)]),
    ("pd_grid_destroy", C.c_int, [_P]),
    ("pd_grid_upload", C.c_int, [_P, C.c_int, _P]),
    ("pd_grid_download", C.c_int, [_P, C.c_int, _P]),
    ("pd_grid_upload_device", C.c_int, [_P, C.c_int, _P]),
    ("pd_grid_set_stream", C.c_int, [_P, _P]),
    ("pd_grid_pack_face", C.c_int, [_P, C.c_int, _P, C.c_int64, C.c_int, _P]),
    ("pd_grid_unpack_face", C.c_int, [_P, C.c_int, _P, C.c_int64, C.c_int, _P]),
    ("pd_grid_swap", C.c_int, [_P, C.c_int, C.c_int]),
    ("pd_grid_column_of", C.c_int, [_P, C.c_int, C.POINTER(C.c_int)]),
    ("pd_grid_device_ptr", C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    ("pd_grid_info", C.c_int, [_P, _I64P, _I64P]),
    ("pd_grid_download_layout", C.c_int, [_P, _P, _P]),
    ("pd_grid_total_mass", C.c_int, [_P, C.c_int, _DP]),
    ("pd_grid_max_active", C.c_int, [_P, C.c_int, _DP]),
    ("pd_grid_minmax_active", C.c_int, [_P, C.c_int, _DP, _DP]),
    ("pd_stepper_create", C.c_int, [_P, C.POINTER(pd_sim_config), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("pd_stepper_destroy", C.c_int, [_P]),
    ("pd_stepper_set_range", C.c_int, [_P, C.c_int64, C.c_int64]),
    ("pd_stepper_stability_bound", C.c_int, [_P, _DP]),
    ("pd_stepper_snapshot_diag", C.c_int, [_P, C.POINTER(pd_diag)]),
    ("pd_stepper_run", C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, _DP, C.POINTER(pd_diag), _I64P]),
    ("pd_stepper_step", C.c_int, [_P, C.c_int64, C.c_double, C.POINTER(pd_diag)]),
    ("pd_stepper_last_ms", C.c_int, [_P, _DP]),
    ("pd_stepper_launch_count", C.c_int, [_P, _I64P]),
    ("pd_build_sphere_pack_grid", C.c_int, [C.c_int, _I64P, _DP, _DP, C.c_int64, _DP, _DP, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("pd_build_sphere_pack_region", C.c_int, [C.c_int, _I64P, _DP, _DP, C.c_int64, _DP, _DP, C.c_double, C.c_double, _I64P, _I64P, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("pd_grid_populate_diffusion", C.c_int, [_P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]),
    ("pd_grid_fill_hash", C.c_int, [_P, C.c_int, C.c_uint64]),
    ("pd_grid_fill_const", C.c_int, [_P, C.c_int, C.c_double]),
    ("pd_smooth_diffusion_coefficients", C.c_int, [_P, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                                   _P, C.c_int]),
    ("pd_grid_create_full", C.c_int, [C.c_int, C.c_int, _I64P, _DP, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(_P)]),
    ("pd_grid_frap_init", C.c_int, [_P, C.c_int, C.c_int, _I64P, _I64P, C.c_double, _I64P, _I64P]),
    ("pd_grid_box_sum", C.c_int, [_P, C.c_int, _I64P, _I64P, _DP]),
    ("pd_stepper_set_region", C.c_int, [_P, _I64P, _I64P]),
    ("pd_stepper_region_sums", C.c_int, [_P, _DP, C.c_int64, _I64P]),
    ("pd_stepper_enqueue", C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_double]),
    ("pd_stepper_swap", C.c_int, [_P]),
    ("pd_stepper_status", C.c_int, [_P, C.c_int64]),
    ("pd_stepper_partials", C.c_int, [_P, _P, _P, _P]),
    ("pd_reduce_partials", C.c_int, [_P, _P, _P, _P, C.c_int64, _DP]),
    ("pd_field_create", C.c_int, [C.c_int, C.c_int, _I64P, _DP, _DP, C.c_int, C.POINTER(_P)]),
    ("pd_field_destroy", C.c_int, [_P]),
    ("pd_field_upload", C.c_int, [_P, _P]),
    ("pd_field_upload_device", C.c_int, [_P, _P]),
    ("pd_field_download", C.c_int, [_P, _P]),
    ("pd_field_device_ptr", C.c_int, [_P, C.POINTER(_P)]),
    ("pd_field_from_mask", C.c_int, [_P, _P, C.c_int64]),
    ("pd_field_filter_thin", C.c_int, [_P, C.c_int]),
    ("pd_field_redistance", C.c_int, [_P, C.POINTER(pd_levelset_options), C.POINTER(pd_redistance_diag)]),
    ("pd_build_grid_from_field", C.c_int, [_P, C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(_P)]),
    ("pd_grid_write_snapshot", C.c_int, [_P, C.c_char_p, C.POINTER(C.c_char_p), C.c_int, _DP]),
    ("pd_grid_read_snapshot", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_P), _DP, C.c_char_p,
                                        C.c_size_t, C.POINTER(C.c_int)]),
    ("pd_field_write_snapshot", C.c_int, [_P, C.c_char_p]),
    ("pd_field_read_snapshot", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("pd_peek_snapshot", C.c_int, [C.c_char_p, C.POINTER(pd_snapshot_info), C.c_char_p, C.c_size_t]),
    ("pd_sphere_pack_layer_work", C.c_int, [C.c_int, C.POINTER(C.c_int64), _DP, _DP, C.c_int64, _DP, _DP, C.c_double,
                                            C.c_double, C.c_int, _P, _P]),
    ("pd_sphere_pack_layer_cost", C.c_int, [C.c_int, C.POINTER(C.c_int64), _DP, _DP, C.c_int64, _DP, _DP, C.c_double,
                                            C.c_double, C.c_int, _P, _P, _P]),
    ("pd_grid_make_shareable", C.c_int, [_P]),
    ("pd_grid_ipc_handles", C.c_int, [_P, _P]),
    ("pd_grid_column_ptrs", C.c_int, [_P, C.POINTER(C.c_void_p)]),
    ("pd_ipc_handle_size", C.c_int, []),
    ("pd_ipc_open", C.c_int, [_P, C.c_int, C.POINTER(C.c_void_p)]),
    ("pd_ipc_close", C.c_int, [_P, C.c_int]),
    ("pd_stepper_sync_words", C.c_int, [_P, C.POINTER(C.c_void_p)]),
    ("pd_stepper_sync_ipc_handle", C.c_int, [_P, _P]),
    ("pd_stepper_set_peer", C.c_int, [_P, C.c_int, C.POINTER(C.c_void_p), C.c_int, _P, _P, _P, C.c_int64]),
    ("pd_stepper_set_convergence", C.c_int, [_P, C.c_int]),
    ("pd_stepper_convergence", C.c_int, [_P, _DP, C.c_int64, _I64P]),
    ("pd_stepper_plane_flux", C.c_int, [_P, C.c_int, C.c_int64, _DP, _DP, _I64P]),
    ("pd_stepper_peer_stats", C.c_int, [_P, C.POINTER(C.c_uint64), _I64P]),
    ("pd_stepper_peer_reset", C.c_int, [_P]),
    ("pd_format_scalar", C.c_int, [C.c_double, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_int)]),
    ("pd_write_vtk", C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int64), _DP, _DP, C.c_int, C.c_int,
                               C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), C.c_int, _P, C.c_int]),
    ("pd_grid_write_vtk", C.c_int, [_P, C.c_char_p, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_char_p), C.c_int,
                                    C.c_double, _DP]),
    ("pd_grid_densify", C.c_int, [_P, C.c_int, C.c_double, _P, _P]),
]

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGNATURES]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"porediff_b200 CUDA library missing at {LIB_PATH}; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH))
    for name, res, args in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    return (lib.pd_last_error() or b"").decode()


def device_count() -> int:
    return int(lib.pd_device_count())
