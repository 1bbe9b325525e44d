"""ctypes binding of libck.so (include/ck/ck.h).

The library is the product: there is no Python or CPU fallback.  Importing a
block without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libck.so")

CK_OK, CK_ERR_SHAPE, CK_ERR_DATA, CK_ERR_NUMERIC, CK_ERR_CUDA, CK_ERR_ARG = range(6)
CK_MATH_TF32, CK_MATH_FP32 = 0, 1
CK_POOL_MAX, CK_POOL_AVG = 0, 1


class ck_shape(C.Structure):
    _fields_ = [("h", C.c_int64), ("w", C.c_int64), ("c", C.c_int64), ("n", C.c_int64)]


class ck_tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("shape", ck_shape)]


class ck_conv_geom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("stride_h", "stride_w", "pad_top", "pad_bottom", "pad_left", "pad_right", "groups")]


class ck_convt_geom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("up_h", "up_w", "crop_top", "crop_bottom", "crop_left", "crop_right")]


class ck_pool_geom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("window_h", "window_w", "stride_h", "stride_w", "pad_top", "pad_bottom",
                 "pad_left", "pad_right", "mode")]


class ck_spnorm_params(C.Structure):
    _fields_ = [("window_h", C.c_int64), ("window_w", C.c_int64), ("alpha", C.c_double),
                ("beta", C.c_double)]


class ck_loss_options(C.Structure):
    _fields_ = [("top_k", C.c_int64), ("threshold", C.c_double), ("random_ties", C.c_int64),
                ("tie_seed", C.c_uint64)]


class ck_lrn_params(C.Structure):
    _fields_ = [("group_size", C.c_int64), ("kappa", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double)]


P = C.c_void_p
T = C.POINTER(ck_tensor)
S = C.c_int

# name -> (restype, argtypes); every symbol ck.h declares.
SIGNATURES = {
    "ck_create": (S, [C.POINTER(P), C.c_int]),
    "ck_destroy": (None, [P]),
    "ck_last_error": (C.c_char_p, [P]),
    "ck_version": (C.c_char_p, []),
    "ck_launch_count": (C.c_int64, [P]),
    "ck_tc_launch_count": (C.c_int64, [P]),
    "ck_trainer_set_graph": (C.c_int, [P, C.c_int]),
    "ck_set_kernel_profiling": (C.c_int, [P, C.c_int]),
    "ck_kernel_profile_count": (C.c_int, [P]),
    "ck_kernel_profile_get": (C.c_int, [P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_float),
                                        C.POINTER(C.c_double)]),
    "ck_kernel_profile_clear": (C.c_int, [P]),
    "ck_memcpy": (S, [P, P, P, C.c_int64, P]),
    "ck_conv_output_shape": (S, [P, ck_shape, ck_shape, C.POINTER(ck_conv_geom), C.POINTER(ck_shape)]),
    "ck_convt_output_shape": (S, [P, ck_shape, ck_shape, C.POINTER(ck_convt_geom), C.POINTER(ck_shape)]),
    "ck_pool_output_shape": (S, [P, ck_shape, C.POINTER(ck_pool_geom), C.POINTER(ck_shape)]),
    "ck_conv_forward": (S, [P, T, T, T, C.POINTER(ck_conv_geom), T, C.c_int, P]),
    "ck_conv_backward": (S, [P, T, T, C.POINTER(ck_conv_geom), T, T, T, T, C.c_int, C.c_int, P]),
    "ck_convt_forward": (S, [P, T, T, C.POINTER(ck_convt_geom), T, C.c_int, P]),
    "ck_convt_backward": (S, [P, T, T, C.POINTER(ck_convt_geom), T, T, T, C.c_int, C.c_int, P]),
    "ck_pool_forward": (S, [P, T, C.POINTER(ck_pool_geom), T, P]),
    "ck_pool_backward": (S, [P, T, C.POINTER(ck_pool_geom), T, T, C.c_int, P]),
    "ck_relu_forward": (S, [P, T, T, P]),
    "ck_relu_backward": (S, [P, T, T, T, C.c_int, P]),
    "ck_lrn_forward": (S, [P, T, C.POINTER(ck_lrn_params), T, P]),
    "ck_lrn_backward": (S, [P, T, C.POINTER(ck_lrn_params), T, T, C.c_int, P]),
    "ck_bnorm_forward": (S, [P, T, T, T, C.c_double, T, T, P]),
    "ck_bnorm_infer": (S, [P, T, T, T, C.c_double, T, T, P]),
    "ck_bnorm_backward": (S, [P, T, T, T, C.c_double, T, T, T, T, C.c_int, P]),
    "ck_softmaxlog_forward": (S, [P, T, T, T, P, C.c_int, P]),
    "ck_softmaxlog_backward": (S, [P, T, T, T, C.c_float, T, C.c_int, P]),
    "ck_loss_metrics": (S, [P, T, T, T, C.c_int64, P, P, P]),
    "ck_check_labels": (S, [P, P]),
    "ck_sgd_step": (S, [P, P, P, P, C.c_int64, C.c_float, C.c_float, C.c_float, P]),
    "ck_sigmoid_forward": (S, [P, T, T, P]),
    "ck_sigmoid_backward": (S, [P, T, T, T, C.c_int, P]),
    "ck_softmax_forward": (S, [P, T, T, P]),
    "ck_softmax_backward": (S, [P, T, T, T, C.c_int, P]),
    "ck_spnorm_forward": (S, [P, T, C.POINTER(ck_spnorm_params), T, P]),
    "ck_spnorm_backward": (S, [P, T, C.POINTER(ck_spnorm_params), T, T, C.c_int, P]),
    "ck_bilinear_output_shape": (S, [P, ck_shape, ck_shape, C.POINTER(ck_shape)]),
    "ck_bilinear_forward": (S, [P, T, T, T, P]),
    "ck_bilinear_backward": (S, [P, T, T, T, T, T, C.c_int, P]),
    "ck_pdist_forward": (S, [P, T, T, C.c_double, C.c_int, T, P]),
    "ck_pdist_backward": (S, [P, T, T, C.c_double, C.c_int, T, T, T, C.c_int, P]),
    "ck_loss_forward": (S, [P, T, T, T, C.c_int, C.POINTER(ck_loss_options), P, C.c_int, P]),
    "ck_loss_backward": (S, [P, T, T, T, C.c_int, C.POINTER(ck_loss_options), C.c_float, T,
                             C.c_int, P]),
    "ck_graph_create": (S, [P, C.POINTER(P)]),
    "ck_graph_destroy": (None, [P]),
    "ck_graph_add_input": (S, [P, C.c_char_p, ck_shape]),
    "ck_graph_add_param": (S, [P, C.c_char_p, ck_shape]),
    "ck_graph_add_layer": (S, [P, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                               C.POINTER(C.c_double), C.c_int]),
    "ck_graph_finalize": (S, [P, C.c_int]),
    "ck_graph_var": (S, [P, C.c_char_p, C.c_int, T]),
    "ck_graph_bind_input": (S, [P, C.c_char_p, C.c_void_p]),
    "ck_graph_forward": (S, [P, P]),
    "ck_graph_backward": (S, [P, C.c_char_p, P]),
    "ck_graph_last_launches": (C.c_int64, [P]),
    "ck_graph_set_profiling": (S, [P, C.c_int]),
    "ck_graph_layer_count": (C.c_int, [P]),
    "ck_graph_layer_name": (C.c_char_p, [P, C.c_int]),
    "ck_graph_layer_ms": (S, [P, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "ck_graph_set_option": (S, [P, C.c_char_p, C.c_int64]),
    "ck_nccl_unique_id": (S, [C.c_char_p]),
    "ck_trainer_create": (S, [P, C.c_char_p, C.c_float, C.c_float, C.c_float, C.POINTER(P)]),
    "ck_trainer_destroy": (None, [P]),
    "ck_trainer_init_dp": (S, [P, C.c_char_p, C.c_int, C.c_int]),
    "ck_trainer_step": (S, [P, C.POINTER(C.c_float), P]),
    "ck_trainer_set_update_stream": (S, [P, C.c_int]),
    "ck_trainer_last_timing": (S, [P, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                   C.POINTER(C.c_float)]),
    "ck_trainer_allreduce_count": (C.c_int64, [P]),
    "ck_rng_create": (P, [C.c_uint64]),
    "ck_rng_destroy": (None, [P]),
    "ck_rng_uniform": (None, [P, P, C.c_int64, C.c_float, C.c_float]),
    "ck_rng_normal": (None, [P, P, C.c_int64, C.c_float]),
    "ck_rng_labels": (None, [P, P, C.c_int64, C.c_uint64]),
    "ck_rng_permutation": (None, [P, C.c_int64, P]),
    "ck_rng_get_state": (None, [P, P]),
    "ck_rng_set_state": (None, [P, P]),
    "ck_io_last_error": (C.c_char_p, []),
    "ck_blob_write": (S, [C.c_char_p, P, ck_shape]),
    "ck_blob_read_shape": (S, [C.c_char_p, C.POINTER(ck_shape)]),
    "ck_blob_read": (S, [C.c_char_p, P, ck_shape]),
    "ck_idx_read": (S, [C.c_char_p, P, P]),
    "ck_graph_save": (S, [P, C.c_char_p]),
    "ck_graph_load": (S, [P, C.c_char_p, C.c_int, C.POINTER(P)]),
    "ck_graph_set_meta": (S, [P, C.c_char_p, C.c_char_p]),
    "ck_graph_get_meta": (C.c_char_p, [P, C.c_char_p]),
    "ck_trainer_save": (S, [P, C.c_char_p, P, C.c_int64]),
    "ck_trainer_load": (S, [P, C.c_char_p, P, P]),
}


class CkError(RuntimeError):
    """A non-OK ck_status; .code mirrors convkit's exception classes."""

    NAMES = {CK_ERR_SHAPE: "ShapeError", CK_ERR_DATA: "DataError", CK_ERR_NUMERIC: "NumericError",
             CK_ERR_CUDA: "CudaError", CK_ERR_ARG: "ArgumentError"}

    def __init__(self, code, msg):
        super().__init__(f"{self.NAMES.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class ShapeError(CkError):
    pass


class DataError(CkError):
    pass


_lib = None


def lib():
    """Load libck.so; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback for the block library)")
        lb = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lb, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lb
    return _lib


def exported_symbols():
    return list(SIGNATURES)


class NumericError(CkError):
    pass


def raise_io(code):
    """Status of a host file function (errors in ck_io_last_error)."""
    if code == CK_OK:
        return
    raise DataError(code, lib().ck_io_last_error().decode(errors="replace"))


def raise_for(code, handle):
    if code == CK_OK:
        return
    msg = lib().ck_last_error(handle).decode(errors="replace") if handle else "error"
    cls = {CK_ERR_SHAPE: ShapeError, CK_ERR_DATA: DataError,
           CK_ERR_NUMERIC: NumericError}.get(code, CkError)
    raise cls(code, msg)
