"""ctypes binding of libfdwave_cuda.so (include/fdwave_cuda.h).

This is the Python side of the C-ABI boundary.  There is no fallback: if the
shared library is missing the import of the solver fails loudly with the build
command to run.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDW_LIB") or os.path.join(_HERE, "libfdwave_cuda.so")  # FDW_LIB: A/B builds

FDW_ABI_VERSION = 3
FDW_OK, FDW_EINVAL, FDW_ECUDA, FDW_EPEER, FDW_EINSTABLE, FDW_ENOMEM, FDW_ESTATE = range(7)
FDW_KERNEL_AUTO, FDW_KERNEL_SIMPLE, FDW_KERNEL_ZMARCH, FDW_KERNEL_TMA, FDW_KERNEL_FUSED2D = 0, 1, 2, 3, 4
FDW_MATH_EXACT, FDW_MATH_FMA = 0, 1
FDW_ADVANCE_RECORD = 1
FDW_ADVANCE_ASYNC = 2


class fdw_desc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32),
        ("ndim", C.c_int32),
        ("space_order", C.c_int32),
        ("dtype_bytes", C.c_int32),
        ("extended", C.c_uint64 * 3),
        ("spacing", C.c_double * 3),
        ("coeffs", C.c_double * 11),
        ("bc", (C.c_int32 * 2) * 3),
        ("dt", C.c_double),
        ("n_steps", C.c_uint64),
        ("check_interval", C.c_uint64),
        ("device", C.c_int32),
        ("variant", C.c_int32),
        ("math", C.c_int32),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("z_segments", C.c_int32),
        ("z_begin", C.c_uint64),
        ("z_end", C.c_uint64),
        ("coeffs1", C.c_double * 10),
    ]


_P = C.c_void_p
_U64P = C.POINTER(C.c_uint64)
_DP = C.POINTER(C.c_double)

# name -> (restype, argtypes)
_SIGS = {
    "fdw_desc_init": (None, [C.POINTER(fdw_desc)]),
    "fdw_create": (C.c_int, [C.POINTER(fdw_desc), C.POINTER(_P)]),
    "fdw_destroy": (C.c_int, [_P]),
    "fdw_last_error": (C.c_char_p, [_P]),
    "fdw_status_string": (C.c_char_p, [C.c_int]),
    "fdw_set_stream": (C.c_int, [_P, _P]),
    "fdw_set_medium": (C.c_int, [_P, _P, _P, C.c_int]),
    "fdw_set_density": (C.c_int, [_P, _P, C.c_int]),
    "fdw_wait": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
    "fdw_snapshot_async": (C.c_int, [_P, _P]),
    "fdw_add_volume_source": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int]),
    "fdw_set_sources": (C.c_int, [_P, C.c_uint64, _P, _P, _P, _P, C.c_uint64]),
    "fdw_set_receivers": (C.c_int, [_P, C.c_uint64, _P, _P, _P]),
    "fdw_set_levels": (C.c_int, [_P, _P, _P]),
    "fdw_get_levels": (C.c_int, [_P, _P, _P]),
    "fdw_zero_levels": (C.c_int, [_P]),
    "fdw_get_extended": (C.c_int, [_P, _P]),
    "fdw_refresh_boundary": (C.c_int, [_P]),
    "fdw_record": (C.c_int, [_P]),
    "fdw_advance": (C.c_int, [_P, C.c_uint64, C.c_uint32, _U64P, _DP]),
    "fdw_step_index": (C.c_int, [_P, _U64P]),
    "fdw_set_step_index": (C.c_int, [_P, C.c_uint64]),
    "fdw_max_abs": (C.c_int, [_P, _DP]),
    "fdw_download_seismogram": (C.c_int, [_P, _P, C.c_uint64]),
    "fdw_download_seismogram_f64": (C.c_int, [_P, _P, C.c_uint64]),
    "fdw_synchronize": (C.c_int, [_P]),
    "fdw_profile_steps": (C.c_int, [_P, C.c_uint64, _DP]),
    "fdw_launch_count": (C.c_int, [_P, _U64P]),
    "fdw_layout": (C.c_int, [_P, _U64P, _U64P, _U64P, _U64P, C.POINTER(C.c_int32)]),
    "fdw_slab_range": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, _U64P, _U64P]),
    "fdw_owner_of": (C.c_int32, [C.c_uint64, _U64P, C.c_int32, C.c_int32]),
    "fdw_peer_export": (C.c_int, [_P, _P]),
    "fdw_peer_import": (C.c_int, [_P, _P, C.c_int32]),
    "fdw_peer_link": (C.c_int, [_P, _P, C.c_int32]),
    "fdw_peer_loopback": (C.c_int, [_P]),
    "fdw_debug_check_guards": (C.c_int, [_P, _U64P]),
    "fdw_receiver_split_info": (C.c_int, [_P, _U64P, _U64P, _U64P]),
    "fdw_download_receiver_products": (C.c_int, [_P, _P, C.c_uint64]),
}

FDW_PEER_BLOB_BYTES = 512

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Loads libfdwave_cuda.so once; raises if it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("FDW_LIB") and not hasattr(L, name):
                continue  # an older A/B build may predate some entry points
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    """Raw data pointer of a numpy array (or None)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)
