"""ctypes binding of librsh.so, the sm_100a C ABI declared in include/rsh.h.

There is no fallback: if the library is missing, was built for another architecture, or no
CUDA device is present, every entry point raises.  Status codes map to the reference's error
types (include/rsh.h): 1 -> ValueError, 2 -> FormatError, 3 -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librsh.so")

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double
_sz = ctypes.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "rsh_last_error": (ctypes.c_char_p, []),
    "rsh_abi_version": (ctypes.c_int, []),
    "rsh_launch_count": (ctypes.c_ulonglong, []),
    "rsh_device_info": (ctypes.c_int, [_vp, _vp, _vp]),
    "rsh_partition_workspace": (_sz, [_i64]),
    "rsh_partition": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rsh_plan_workspace": (_sz, [_i64, _i64, _i64]),
    "rsh_plan_windows": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i32, _vp, _vp, _i64, _i64, _i32, _f64, _vp,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rsh_fill_workspace": (_sz, [_i64, _i64]),
    "rsh_build_fill": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _i64,
                                      _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rsh_residual_workspace": (_sz, [_i64]),
    "rsh_residual_offsets": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "rsh_residual_gather": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "rsh_permute_workspace": (_sz, [_i64]),
    "rsh_permute_rows": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rsh_transpose_workspace": (_sz, [_i64, _i64, _i64]),
    "rsh_transpose_csr": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rsh_reorder_workspace": (_sz, [_i64, _i64]),
    "rsh_column_weights": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _f64, _vp, _vp, _vp, _sz, _vp]),
    "rsh_knn": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp]),
    "rsh_pair_dis": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "rsh_two_opt_sweep": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i64, _vp, _vp]),
    "rsh_mst_order": (ctypes.c_int, [_i64, _i32, _vp, _vp, _vp, _vp]),
    "rsh_sum_sequential": (_f64, [_vp, _i64]),
    "rsh_isolation_adjust": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _f64, _i64, _vp, _vp]),
    "rsh_schedule_bytes": (_sz, [_i64, _i64, _i64, _i64]),
    "rsh_schedule": (ctypes.c_int, [_i64, _i32, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _vp, _sz, _vp, _vp]),
    "rsh_partials_bytes": (_sz, [_i64, _i64, _i64, _i32]),
    "rsh_rowmajor_bytes": (_sz, [_i64, _i64, _i64, _i64, _i64]),
    "rsh_schedule_rowmajor": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp, _sz, _vp]),
    "rsh_spmm_cc": (ctypes.c_int, [_i64, _i32, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64,
                                   _i32, _i64, _vp, _i64, _i32, _vp, _sz, _vp, _sz, _vp]),
    "rsh_tc_fragment_bytes": (_sz, [_i64, _i32]),
    "rsh_tc_fragments": (ctypes.c_int, [_i64, _i64, _vp, _vp, _i64, _i64, _i32, _vp, _sz, _vp, _sz, _vp]),
    "rsh_spmm_tc": (ctypes.c_int, [_i64, _i32, _i64, _vp, _vp, _vp, _sz, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64,
                                   _i64, _i32, _i64, _vp, _i64, _i32, _vp, _sz, _vp, _sz, _vp]),
    "rsh_candidates": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp]),
    "rsh_csr_spmm_f64": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _i64, _vp]),
    "rsh_tile_density": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "rsh_window_nnz": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp]),
    "rsh_report_slots": (ctypes.c_int, []),
    "rsh_validate_workspace": (_sz, [_i64, _i64, _i64]),
    "rsh_validate": (ctypes.c_int, [_i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64,
                                    _vp, _i64, _i32, _i32, _vp, _vp, _sz, _vp]),
    "rsh_decode_workspace": (_sz, [_i64, _i64, _i64]),
    "rsh_decode": (ctypes.c_int, [_i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp,
                                  _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rsh_max_relative_error": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
}

_lib = None


class FormatError(ValueError):
    """A tile format violated one of its structural invariants (tile.py:39-40)."""


def lib() -> ctypes.CDLL:
    """Load librsh.so; raise loudly if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2603_08734_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = lib().rsh_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == 1:
        raise ValueError(text)
    if status == 2:
        raise FormatError(text)
    raise RuntimeError(text)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
