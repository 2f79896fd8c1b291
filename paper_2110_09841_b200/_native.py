"""ctypes binding of libcvpb200.so (include/cvpb200.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_2110_09841_b200/csrc``). There is no CPU fallback: if the
library is missing or no CUDA device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CVPB_LIB: developer override (kernel-variant experiments); defaults to the in-tree build
LIB_PATH = os.environ.get("CVPB_LIB") or os.path.join(HERE, "libcvpb200.so")


class cvpb_volume_geometry(C.Structure):
    _fields_ = [("counts", C.c_int * 3), ("voxel_size", C.c_double * 3)]


class cvpb_detector_geometry(C.Structure):
    _fields_ = [("rows", C.c_int), ("cols", C.c_int), ("pixel_width", C.c_double),
                ("pixel_height", C.c_double)]


class cvpb_view(C.Structure):
    _fields_ = [("source", C.c_double * 3), ("frame", C.c_double * 9),
                ("focal_length", C.c_double), ("principal_point", C.c_double * 2),
                ("pixel_size", C.c_double * 2)]


class cvpb_cvp_options(C.Structure):
    _fields_ = [("scaling", C.c_int), ("elevation_correction", C.c_int), ("precision", C.c_int),
                ("r_estimate", C.c_int)]


class cvpb_exec_policy(C.Structure):
    _fields_ = [("threads", C.c_int), ("deterministic", C.c_int), ("allow_expensive", C.c_int)]


class cvpb_slab_targets(C.Structure):
    _fields_ = [("n", C.c_int), ("plane_begin", C.c_int * 17), ("slab", C.c_void_p * 16),
                ("store", C.c_int)]


class cvpb_pixel_roi(C.Structure):
    _fields_ = [("row_begin", C.c_int), ("row_end", C.c_int), ("col_begin", C.c_int),
                ("col_end", C.c_int)]


class cvpb_tt_options(C.Structure):
    _fields_ = [("amplitude", C.c_int)]


_P = C.POINTER
_vp = C.c_void_p
_dp = _P(C.c_double)
_ip = _P(C.c_int)

# name -> (restype, argtypes); every symbol include/cvpb200.h declares.
SIGNATURES = {
    "cvpb_abi_version": (C.c_int, []),
    "cvpb_last_error": (C.c_char_p, []),
    "cvpb_device_count": (C.c_int, [_ip]),
    "cvpb_context_create": (C.c_int, [C.c_int, _P(_vp)]),
    "cvpb_context_destroy": (None, [_vp]),
    "cvpb_set_geometry": (C.c_int, [_vp, _P(cvpb_volume_geometry), _P(cvpb_detector_geometry),
                                    C.c_int, _P(cvpb_view)]),
    "cvpb_get_counts": (C.c_int, [_vp, _ip, _P(C.c_size_t), _P(C.c_size_t)]),
    "cvpb_view_make": (C.c_int, [_dp, _dp, C.c_double, _dp, _dp, _P(cvpb_view)]),
    "cvpb_make_circular_trajectory": (C.c_int, [C.c_double, C.c_double, C.c_int, C.c_double,
                                                _P(cvpb_detector_geometry), _P(cvpb_view)]),
    "cvpb_view_standard_matrix": (C.c_int, [_P(cvpb_view), _dp]),
    "cvpb_view_from_standard_matrix": (C.c_int, [_dp, _dp, _P(cvpb_view)]),
    "cvpb_view_project_point": (C.c_int, [_P(cvpb_view), _dp, _dp]),
    "cvpb_pixel_scale": (C.c_int, [_P(cvpb_view), _P(cvpb_detector_geometry), C.c_int, C.c_int,
                                   C.c_int, _dp]),
    "cvpb_fill_uniform01": (C.c_int, [_dp, C.c_size_t, C.c_uint64]),
    "cvpb_project_cvp": (C.c_int, [_vp, _P(cvpb_cvp_options), _P(cvpb_exec_policy), _vp, _vp,
                                   C.c_int, C.c_int, _vp]),
    "cvpb_backproject_cvp": (C.c_int, [_vp, _P(cvpb_cvp_options), _P(cvpb_exec_policy), _vp, _vp,
                                       C.c_int, C.c_int, C.c_int, _vp]),
    "cvpb_project_cvp_host": (C.c_int, [_vp, _P(cvpb_cvp_options), _P(cvpb_exec_policy), _vp,
                                        _vp, _vp]),
    "cvpb_backproject_cvp_host": (C.c_int, [_vp, _P(cvpb_cvp_options), _P(cvpb_exec_policy), _vp,
                                            _vp, _vp]),
    "cvpb_sync": (C.c_int, [_vp, _vp]),
    "cvpb_sum_slabs": (C.c_int, [_vp, _P(C.c_void_p), C.c_int, C.c_size_t, _vp, _vp, _vp]),
    "cvpb_ipc_alloc": (C.c_int, [_vp, C.c_size_t, _P(C.c_void_p), _vp]),
    "cvpb_ipc_open": (C.c_int, [_vp, _vp, _P(C.c_void_p)]),
    "cvpb_ipc_close": (C.c_int, [_vp, _vp]),
    "cvpb_ipc_free": (C.c_int, [_vp, _vp]),
    "cvpb_backproject_cvp_scatter": (C.c_int, [_vp, _P(cvpb_cvp_options), _P(cvpb_exec_policy), _vp,
                                               C.c_int, C.c_int, _P(cvpb_slab_targets), _vp]),
    "cvpb_cvp_view_weights": (C.c_int, [_vp, _P(cvpb_cvp_options), C.c_int, C.c_int, _dp]),
    "cvpb_collect_cut_records": (C.c_int, [_vp, _P(cvpb_cvp_options), C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, _ip]),
    "cvpb_scale_image": (C.c_int, [_vp, C.c_int, C.c_int, _dp]),
    "cvpb_project_siddon": (C.c_int, [_vp, C.c_int, _P(cvpb_pixel_roi), _P(cvpb_exec_policy),
                                      _vp, _vp, C.c_int, C.c_int, _vp]),
    "cvpb_backproject_siddon": (C.c_int, [_vp, C.c_int, _P(cvpb_exec_policy), _vp, _vp, C.c_int,
                                          C.c_int, C.c_int, _vp]),
    "cvpb_trace_ray": (C.c_int, [_vp, _P(cvpb_volume_geometry), _dp, _dp, C.c_int, _ip, _dp, _ip]),
    "cvpb_project_tt": (C.c_int, [_vp, _P(cvpb_tt_options), _vp, _vp, C.c_int, C.c_int, _vp]),
    "cvpb_backproject_tt": (C.c_int, [_vp, _P(cvpb_tt_options), _vp, _vp, C.c_int, C.c_int,
                                      C.c_int, _vp]),
    "cvpb_project_siddon_host": (C.c_int, [_vp, C.c_int, _P(cvpb_pixel_roi), _P(cvpb_exec_policy),
                                           _vp, _vp]),
    "cvpb_backproject_siddon_host": (C.c_int, [_vp, C.c_int, _P(cvpb_exec_policy), _vp, _vp]),
    "cvpb_project_tt_host": (C.c_int, [_vp, _P(cvpb_tt_options), _vp, _vp]),
    "cvpb_backproject_tt_host": (C.c_int, [_vp, _P(cvpb_tt_options), _vp, _vp]),
    "cvpb_cgls_host": (C.c_int, [_vp, C.c_int, _P(cvpb_cvp_options), _P(cvpb_tt_options),
                                 _P(cvpb_exec_policy), C.c_int, _vp, _vp, C.c_int, _dp]),
    "cvpb_backproject_cvp_host_partial": (C.c_int, [_vp, _P(cvpb_cvp_options),
                                                    _P(cvpb_exec_policy), _vp, _vp, _vp]),
    "cvpb_vec_to_host64": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp]),
    "cvpb_vec_dot": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _dp, _vp]),
    "cvpb_vec_axpy": (C.c_int, [_vp, C.c_double, _vp, _vp, C.c_size_t, _vp]),
    "cvpb_vec_xpby": (C.c_int, [_vp, _vp, C.c_double, _vp, C.c_size_t, _vp]),
    "cvpb_vec_all_finite": (C.c_int, [_vp, _vp, C.c_size_t, _ip, _vp]),
    "cvpb_vec_sart_residual": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
    "cvpb_vec_sart_update": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_int, C.c_size_t, _vp]),
    "cvpb_cgls": (C.c_int, [_vp, C.c_int, _P(cvpb_cvp_options), _P(cvpb_tt_options),
                            _P(cvpb_exec_policy), C.c_int, _vp, _vp, C.c_int, _dp, _vp]),
    # multi-device scenes
    "cvpb_group_create": (C.c_int, [_ip, C.c_int, _P(_vp)]),
    "cvpb_group_destroy": (None, [_vp]),
    "cvpb_group_size": (C.c_int, [_vp, _ip]),
    "cvpb_group_member": (C.c_int, [_vp, C.c_int, _ip, _ip, _ip, _P(C.c_size_t), _P(C.c_size_t)]),
    "cvpb_group_context": (C.c_int, [_vp, C.c_int, _P(_vp)]),
    "cvpb_group_set_geometry": (C.c_int, [_vp, _P(cvpb_volume_geometry),
                                          _P(cvpb_detector_geometry), C.c_int, _P(cvpb_view)]),
    "cvpb_group_project_cvp_host": (C.c_int, [_vp, _P(cvpb_cvp_options), _P(cvpb_exec_policy),
                                              _vp, _vp, _vp]),
    "cvpb_group_backproject_cvp_host": (C.c_int, [_vp, _P(cvpb_cvp_options),
                                                  _P(cvpb_exec_policy), _vp, _vp, _vp]),
    "cvpb_group_project_tt_host": (C.c_int, [_vp, _P(cvpb_tt_options), _vp, _vp]),
    "cvpb_group_backproject_tt_host": (C.c_int, [_vp, _P(cvpb_tt_options), _vp, _vp]),
    "cvpb_group_cgls_host": (C.c_int, [_vp, C.c_int, _P(cvpb_cvp_options), _P(cvpb_tt_options),
                                       _P(cvpb_exec_policy), C.c_int, _vp, _vp, C.c_int, _dp]),
}

# status code -> exception type the reference throws for the same condition
OK, INVALID_ARGUMENT, RUNTIME_ERROR, OUT_OF_RANGE, DOMAIN_ERROR, CUDA_ERROR, NO_DEVICE = range(7)


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ArithmeticError):
    """std::domain_error"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class CvpbRuntimeError(RuntimeError):
    """std::runtime_error (and device failures)"""


class NoDevice(RuntimeError):
    """No CUDA device: the product path has no CPU fallback."""


_EXC = {INVALID_ARGUMENT: InvalidArgument, RUNTIME_ERROR: CvpbRuntimeError,
        OUT_OF_RANGE: OutOfRange, DOMAIN_ERROR: DomainError, CUDA_ERROR: CvpbRuntimeError,
        NO_DEVICE: NoDevice}

_lib = None


def lib():
    """Load libcvpb200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2110_09841_b200/csrc). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc != OK:
        msg = lib().cvpb_last_error().decode()
        raise _EXC.get(rc, CvpbRuntimeError)(msg)
    return rc
