"""ctypes binding of the C ABI in include/sparsh_b200.h (libsparsh_b200.so).

The library is built in-tree by ``make -C paper_2007_00056_b200/csrc`` (see
``__graft_entry__.build``). There is no fallback: if the shared object is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SB_LIB") or os.path.join(_HERE, "_lib", "libsparsh_b200.so")  # SB_LIB: tools/ variant builds
CSRC = os.path.join(_HERE, "csrc")

SB_OK, SB_EINVAL, SB_ERUNTIME, SB_ECUDA = 0, 1, 2, 3


class sb_csr(C.Structure):
    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("row_ptr32", C.POINTER(C.c_int32)),
        ("row_ptr64", C.POINTER(C.c_int64)),
        ("col_idx", C.POINTER(C.c_int32)),
        ("values", C.POINTER(C.c_double)),
    ]


class sb_setup_opts(C.Structure):
    _fields_ = [
        ("coarsening", C.c_int),
        ("coarse_target", C.c_int64),
        ("max_levels", C.c_int),
        ("coarse_solver", C.c_int),
        ("threads", C.c_int),
        ("galerkin_gpu", C.c_int),
        ("gpu_device", C.c_int),
    ]


class sb_cycle(C.Structure):
    _fields_ = [
        ("pre_sweeps", C.c_int),
        ("post_sweeps", C.c_int),
        ("smoother", C.c_int),
        ("omega", C.c_double),
    ]


class sb_report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("termination", C.c_int),
        ("wall_time", C.c_double),
        ("true_residual", C.c_double),
        ("hist_len", C.c_int),
        ("hist_cap", C.c_int),
        ("residual_history", C.POINTER(C.c_double)),
        ("time_history", C.POINTER(C.c_double)),
    ]


class sb_device_opts(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("use_graphs", C.c_int),
        ("host_levels_from", C.c_int64),
        ("coarse_exact", C.c_int),
    ]


# every symbol include/sparsh_b200.h declares (tests/test_abi.py checks them)
EXPORTS = [
    "sb_last_error", "sb_version", "sb_setup", "sb_hier_from_levels", "sb_hier_free",
    "sb_hier_nlevels", "sb_hier_stalled", "sb_hier_level", "sb_hier_coarse_counts",
    "sb_create", "sb_destroy", "sb_device_bytes", "sb_stream", "sb_vcycle", "sb_vcycle_dev",
    "sb_pcg", "sb_pbicgstab", "sb_amg_solve", "sb_pcg_dev", "sb_pbicgstab_dev", "sb_spmv",
    "sb_smooth", "sb_residual", "sb_restrict", "sb_prolong", "sb_coarse_solve",
    "sb_gen_convdiff2d", "sb_gen_stencil7", "sb_gen_convdiff3d", "sb_gen_stencil27",
    "sb_free_csr", "sb_gen_rhs_random", "sb_last_solve_ms", "sb_last_solve_launches", "sb_time_kernel", "sb_time_kernel_cold", "sb_vcycle_launches", "sb_tail_trace",
    "sb_tail_info", "sb_level_format", "sb_level_march", "sb_level_sweep_kernel", "sb_level_fused_sweeps", "sb_build_flags", "sb_level_residency", "sb_partition", "sb_partition_free", "sb_partition_info",
    "sb_partition_level", "sb_partition_exchange", "sb_nccl_unique_id", "sb_dist_create",
    "sb_dist_create_local", "sb_dist_create_local_p2p", "sb_dist_create_p2p", "sb_dist_p2p_export",
    "sb_dist_p2p_connect", "sb_dist_destroy", "sb_dist_rows", "sb_dist_pcg", "sb_dist_pbicgstab",
    "sb_dist_vcycle", "sb_dist_last_solve_ms", "sb_dist_last_launches", "sb_galerkin_gpu", "sb_host_bytes", "sb_setup_stencil27",
    "sb_read_matrix_market", "sb_write_matrix_market",
]

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_SIGS = {
    "sb_last_error": (C.c_char_p, []),
    "sb_version": (C.c_char_p, []),
    "sb_setup": (C.c_int, [C.POINTER(sb_csr), C.POINTER(sb_setup_opts), C.POINTER(_P)]),
    "sb_hier_from_levels": (C.c_int, [C.c_int, C.POINTER(sb_csr), C.POINTER(C.POINTER(C.c_int32)), C.POINTER(_P)]),
    "sb_hier_free": (None, [_P]),
    "sb_hier_nlevels": (C.c_int, [_P]),
    "sb_hier_stalled": (C.c_int, [_P]),
    "sb_hier_level": (C.c_int, [_P, C.c_int, C.POINTER(sb_csr), C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int64)]),
    "sb_hier_coarse_counts": (C.c_int, [_P, C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    "sb_create": (C.c_int, [_P, C.POINTER(sb_device_opts), C.POINTER(_P)]),
    "sb_destroy": (None, [_P]),
    "sb_device_bytes": (C.c_int64, [_P]),
    "sb_host_bytes": (C.c_int64, [_P]),
    "sb_stream": (_P, [_P]),
    "sb_vcycle": (C.c_int, [_P, C.POINTER(sb_cycle), C.c_int, _D, _D]),
    "sb_vcycle_dev": (C.c_int, [_P, C.POINTER(sb_cycle), C.c_int, _P, _P, C.c_int]),
    "sb_pcg": (C.c_int, [_P, C.POINTER(sb_cycle), _D, _D, C.c_double, C.c_int, C.POINTER(sb_report)]),
    "sb_pbicgstab": (C.c_int, [_P, C.POINTER(sb_cycle), _D, _D, C.c_double, C.c_int, C.POINTER(sb_report)]),
    "sb_amg_solve": (C.c_int, [_P, C.POINTER(sb_cycle), _D, _D, C.c_double, C.c_int, C.POINTER(sb_report)]),
    "sb_pcg_dev": (C.c_int, [_P, C.POINTER(sb_cycle), _P, _P, C.c_double, C.c_int, C.POINTER(sb_report)]),
    "sb_pbicgstab_dev": (C.c_int, [_P, C.POINTER(sb_cycle), _P, _P, C.c_double, C.c_int, C.POINTER(sb_report)]),
    "sb_spmv": (C.c_int, [_P, C.c_int, _D, _D]),
    "sb_smooth": (C.c_int, [_P, C.c_int, C.POINTER(sb_cycle), _D, _D, C.c_int]),
    "sb_residual": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "sb_restrict": (C.c_int, [_P, C.c_int, _D, _D]),
    "sb_prolong": (C.c_int, [_P, C.c_int, _D, _D]),
    "sb_coarse_solve": (C.c_int, [_P, _D, _D]),
    "sb_gen_convdiff2d": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double, C.POINTER(sb_csr)]),
    "sb_gen_stencil7": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_double, _D, C.POINTER(sb_csr)]),
    "sb_gen_convdiff3d": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(sb_csr)]),
    "sb_gen_stencil27": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.POINTER(sb_csr)]),
    "sb_setup_stencil27": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                     C.POINTER(sb_setup_opts), C.POINTER(_P)]),
    "sb_free_csr": (None, [C.POINTER(sb_csr)]),
    "sb_read_matrix_market": (C.c_int, [C.c_char_p, C.POINTER(sb_csr)]),
    "sb_write_matrix_market": (C.c_int, [C.c_char_p, C.POINTER(sb_csr)]),
    "sb_galerkin_gpu": (C.c_int, [C.POINTER(sb_csr), C.POINTER(C.c_int32), C.c_int64, C.c_int, C.POINTER(sb_csr)]),
    "sb_gen_rhs_random": (C.c_int, [C.c_int64, C.c_uint, _D]),
    "sb_last_solve_ms": (C.c_double, [_P]),
    "sb_last_solve_launches": (C.c_int64, [_P]),
    "sb_time_kernel": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(sb_cycle), C.c_int, _D, C.POINTER(C.c_int)]),
    "sb_time_kernel_cold": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(sb_cycle), C.c_int, C.c_int64, _D,
                                      C.POINTER(C.c_int)]),
    "sb_vcycle_launches": (C.c_int, [_P, C.POINTER(sb_cycle)]),
    "sb_tail_trace": (C.c_int, [_P, C.POINTER(C.c_ulonglong), C.c_int]),
    "sb_tail_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sb_level_format": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "sb_level_march": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sb_level_sweep_kernel": (C.c_int, [_P, C.c_int, C.c_char_p, C.c_int]),
    "sb_level_fused_sweeps": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int)]),
    "sb_build_flags": (C.c_int, []),
    "sb_level_residency": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "sb_partition": (C.c_int, [_P, C.c_int, C.c_int, C.c_int64, C.POINTER(_P)]),
    "sb_partition_free": (None, [_P]),
    "sb_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "sb_dist_create": (C.c_int, [_P, C.c_int, C.c_int, C.c_char_p, C.c_int64, C.POINTER(sb_device_opts), C.POINTER(_P)]),
    "sb_dist_create_local": (C.c_int, [_P, C.c_int, C.c_int64, C.POINTER(sb_device_opts), C.POINTER(_P)]),
    "sb_dist_create_local_p2p": (C.c_int, [_P, C.c_int, C.c_int64, C.POINTER(sb_device_opts), C.POINTER(_P)]),
    "sb_dist_create_p2p": (C.c_int, [_P, C.c_int, C.c_int, C.c_int64, C.POINTER(sb_device_opts), C.POINTER(_P)]),
    "sb_dist_p2p_export": (C.c_int, [_P, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]),
    "sb_dist_p2p_connect": (C.c_int, [_P, C.c_char_p, C.c_int64]),
    "sb_dist_destroy": (None, [_P]),
    "sb_dist_rows": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "sb_dist_pcg": (C.c_int, [_P, C.POINTER(sb_cycle), _P, _P, C.c_double, C.c_int, C.POINTER(sb_report), C.c_int]),
    "sb_dist_pbicgstab": (C.c_int, [_P, C.POINTER(sb_cycle), _P, _P, C.c_double, C.c_int, C.POINTER(sb_report), C.c_int]),
    "sb_dist_vcycle": (C.c_int, [_P, C.POINTER(sb_cycle), _D, _D]),
    "sb_dist_last_solve_ms": (C.c_double, [_P]),
    "sb_dist_last_launches": (C.c_int, [_P]),
    "sb_partition_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sb_partition_level": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int64), C.POINTER(sb_csr),
                                     C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int64)),
                                     C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int32)),
                                     C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.POINTER(C.c_int32))]),
    "sb_partition_exchange": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.POINTER(C.c_int)),
                                        C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int32)),
                                        C.POINTER(C.POINTER(C.c_int)), C.POINTER(C.POINTER(C.c_int64)),
                                        C.POINTER(C.POINTER(C.c_int64))]),
}


class InvalidArgument(ValueError):
    """The reference would throw std::invalid_argument (SB_EINVAL)."""


class CudaError(RuntimeError):
    """CUDA failure inside the library (SB_ECUDA); there is no CPU fallback."""


_lib = None


def lib() -> C.CDLL:
    """Loads libsparsh_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == SB_OK:
        return
    msg = lib().sb_last_error().decode()
    if rc == SB_EINVAL:
        raise InvalidArgument(msg)
    if rc == SB_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def lptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int64))
