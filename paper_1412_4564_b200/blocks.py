"""The convkit block API over CUDA tensors, through the C ABI (libck.so).

Same names, argument meaning and error behaviour as the reference's C++
templates (include/convkit/{conv,pool,activation,normalize,loss}.hpp); the
differences are a device library's: tensors live on the GPU and exceptions
come from ck_status codes (``ShapeError`` / ``DataError``).

Layout: an HWCN tensor of shape (H, W, C, N) (tensor.hpp:70-72, H fastest) is
a contiguous torch tensor of torch-shape (N, C, W, H) -- the identical bytes.
``from_hwcn`` / ``hwcn_shape`` convert between the two views.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (CK_MATH_FP32, CK_MATH_TF32, CkError, DataError, ShapeError,  # noqa: F401
                   ck_conv_geom, ck_convt_geom, ck_loss_options, ck_lrn_params, ck_pool_geom,
                   ck_shape, ck_spnorm_params, ck_tensor, lib, raise_for)


# ---- hyper-parameters (field names as in the reference headers) -------------

@dataclass
class ConvGeom:  # conv.hpp:9-17
    stride_h: int = 1
    stride_w: int = 1
    pad_top: int = 0
    pad_bottom: int = 0
    pad_left: int = 0
    pad_right: int = 0
    groups: int = 1

    def c(self):
        return ck_conv_geom(self.stride_h, self.stride_w, self.pad_top, self.pad_bottom,
                            self.pad_left, self.pad_right, self.groups)

    def params(self):
        return [self.stride_h, self.stride_w, self.pad_top, self.pad_bottom, self.pad_left,
                self.pad_right, self.groups]


@dataclass
class ConvTransposeGeom:  # conv.hpp:21-28
    up_h: int = 1
    up_w: int = 1
    crop_top: int = 0
    crop_bottom: int = 0
    crop_left: int = 0
    crop_right: int = 0

    def c(self):
        return ck_convt_geom(self.up_h, self.up_w, self.crop_top, self.crop_bottom,
                             self.crop_left, self.crop_right)

    def params(self):
        return [self.up_h, self.up_w, self.crop_top, self.crop_bottom, self.crop_left,
                self.crop_right]


MAX, AVG = "max", "avg"


@dataclass
class PoolGeom:  # pool.hpp:13-23
    window_h: int = 1
    window_w: int = 1
    stride_h: int = 1
    stride_w: int = 1
    pad_top: int = 0
    pad_bottom: int = 0
    pad_left: int = 0
    pad_right: int = 0
    mode: str = MAX

    def c(self):
        return ck_pool_geom(self.window_h, self.window_w, self.stride_h, self.stride_w,
                            self.pad_top, self.pad_bottom, self.pad_left, self.pad_right,
                            0 if self.mode == MAX else 1)

    def params(self):
        return [self.window_h, self.window_w, self.stride_h, self.stride_w, self.pad_top,
                self.pad_bottom, self.pad_left, self.pad_right, 0 if self.mode == MAX else 1]


@dataclass
class LrnParams:  # normalize.hpp:11-16
    group_size: int = 5
    kappa: float = 2.0
    alpha: float = 1e-4
    beta: float = 0.75

    def c(self):
        return ck_lrn_params(self.group_size, self.kappa, self.alpha, self.beta)

    def params(self):
        return [self.group_size, self.kappa, self.alpha, self.beta]


MATH = {"tf32": CK_MATH_TF32, "fp32": CK_MATH_FP32}


# ---- handle / tensor plumbing ---------------------------------------------------

_tls = threading.local()


class Handle:
    """One ck_handle bound to a device (one per host thread)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        raise_for(lib().ck_create(C.byref(h), device), None)
        self.h = h
        self.device = device

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.ck_destroy(self.h)
            self.h = None

    def check(self, code):
        raise_for(code, self.h)

    @property
    def launches(self) -> int:
        return lib().ck_launch_count(self.h)

    @property
    def tc_launches(self) -> int:
        """tcgen05 GEMM launches (ck_tc_launch_count)."""
        return lib().ck_tc_launch_count(self.h)

    def kernel_profiling(self, on: bool):
        """Time every tensor-core GEMM launch (ck_set_kernel_profiling)."""
        self.check(lib().ck_kernel_profile_clear(self.h))
        self.check(lib().ck_set_kernel_profiling(self.h, int(on)))

    def kernel_profile(self):
        """[(label, ms, algorithmic flops)] of the GEMM launches recorded so far."""
        out = []
        for i in range(lib().ck_kernel_profile_count(self.h)):
            lab, ms, fl = C.c_char_p(), C.c_float(), C.c_double()
            self.check(lib().ck_kernel_profile_get(self.h, i, C.byref(lab), C.byref(ms),
                                                   C.byref(fl)))
            out.append((lab.value.decode(), ms.value, fl.value))
        return out


def handle(device: int | None = None) -> Handle:
    device = torch.cuda.current_device() if device is None else device
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    if device not in hs:
        hs[device] = Handle(device)
    return hs[device]


def hwcn_shape(t: torch.Tensor):
    """(H, W, C, N) of a torch tensor stored as (N, C, W, H)."""
    assert t.dim() == 4, "HWCN tensors are 4-D torch tensors shaped (N, C, W, H)"
    n, c, w, h = t.shape
    return (h, w, c, n)


def from_hwcn(shape, device="cuda", dtype=torch.float32, fill=None):
    h, w, c, n = shape
    if fill is None:
        return torch.empty((n, c, w, h), device=device, dtype=dtype)
    return torch.full((n, c, w, h), fill, device=device, dtype=dtype)


def as_hwcn(flat: torch.Tensor, shape):
    h, w, c, n = shape
    return flat.reshape(n, c, w, h)


def _t(x: torch.Tensor | None):
    if x is None:
        return None
    if not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError("block tensors must be contiguous float32 CUDA tensors")
    return C.byref(ck_tensor(x.data_ptr(), ck_shape(*hwcn_shape(x))))


def _vec(x: torch.Tensor | None, shape=None):
    """A parameter vector (bias, bnorm w/b) as a 1x1xKx1 tensor view."""
    if x is None:
        return None
    if not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError("block tensors must be contiguous float32 CUDA tensors")
    s = shape or (1, 1, x.numel(), 1)
    return C.byref(ck_tensor(x.data_ptr(), ck_shape(*s)))


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


# ---- shape laws -------------------------------------------------------------------

def conv_output_shape(xs, fs, g: ConvGeom):
    out = ck_shape()
    hd = handle()
    hd.check(lib().ck_conv_output_shape(hd.h, ck_shape(*xs), ck_shape(*fs), C.byref(g.c()),
                                        C.byref(out)))
    return (out.h, out.w, out.c, out.n)


def convt_output_shape(xs, fs, g: ConvTransposeGeom):
    out = ck_shape()
    hd = handle()
    hd.check(lib().ck_convt_output_shape(hd.h, ck_shape(*xs), ck_shape(*fs), C.byref(g.c()),
                                         C.byref(out)))
    return (out.h, out.w, out.c, out.n)


def pool_output_shape(xs, g: PoolGeom):
    out = ck_shape()
    hd = handle()
    hd.check(lib().ck_pool_output_shape(hd.h, ck_shape(*xs), C.byref(g.c()), C.byref(out)))
    return (out.h, out.w, out.c, out.n)


# ---- blocks --------------------------------------------------------------------------

def conv_forward(x, f, bias, g: ConvGeom, math="tf32"):
    """vl_nnconv forward (conv.hpp:60-62)."""
    ys = conv_output_shape(hwcn_shape(x), hwcn_shape(f), g)
    y = from_hwcn(ys, x.device)
    hd = handle()
    hd.check(lib().ck_conv_forward(hd.h, _t(x), _t(f), _vec(bias), C.byref(g.c()), _t(y),
                                   MATH[math], _stream()))
    return y


def conv_backward(x, f, g: ConvGeom, dy, want_dx=True, want_df=True, want_db=True, math="tf32",
                  out=None, accumulate=False):
    """vl_nnconv backward (conv.hpp:64-69): returns (dx, df, db), None where skipped."""
    dx, df, db = out if out is not None else (
        torch.zeros_like(x) if want_dx else None,
        torch.zeros_like(f) if want_df else None,
        torch.zeros(f.shape[0], device=x.device) if want_db else None)
    hd = handle()
    hd.check(lib().ck_conv_backward(hd.h, _t(x), _t(f), C.byref(g.c()), _t(dy), _t(dx), _t(df),
                                    _vec(db), int(accumulate), MATH[math], _stream()))
    return dx, df, db


def convt_forward(x, f, g: ConvTransposeGeom, math="tf32"):
    ys = convt_output_shape(hwcn_shape(x), hwcn_shape(f), g)
    y = from_hwcn(ys, x.device)
    hd = handle()
    hd.check(lib().ck_convt_forward(hd.h, _t(x), _t(f), C.byref(g.c()), _t(y), MATH[math],
                                    _stream()))
    return y


def convt_backward(x, f, g: ConvTransposeGeom, dy, math="tf32"):
    dx, df = torch.zeros_like(x), torch.zeros_like(f)
    hd = handle()
    hd.check(lib().ck_convt_backward(hd.h, _t(x), _t(f), C.byref(g.c()), _t(dy), _t(dx), _t(df),
                                     0, MATH[math], _stream()))
    return dx, df


def pool_forward(x, g: PoolGeom):
    ys = pool_output_shape(hwcn_shape(x), g)
    y = from_hwcn(ys, x.device)
    hd = handle()
    hd.check(lib().ck_pool_forward(hd.h, _t(x), C.byref(g.c()), _t(y), _stream()))
    return y


def pool_backward(x, g: PoolGeom, dy):
    dx = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_pool_backward(hd.h, _t(x), C.byref(g.c()), _t(dy), _t(dx), 0, _stream()))
    return dx


def relu_forward(x):
    y = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_relu_forward(hd.h, _t(x), _t(y), _stream()))
    return y


def relu_backward(x, dy):
    dx = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_relu_backward(hd.h, _t(x), _t(dy), _t(dx), 0, _stream()))
    return dx


def lrn_forward(x, p: LrnParams):
    y = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_lrn_forward(hd.h, _t(x), C.byref(p.c()), _t(y), _stream()))
    return y


def lrn_backward(x, p: LrnParams, dy):
    dx = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_lrn_backward(hd.h, _t(x), C.byref(p.c()), _t(dy), _t(dx), 0, _stream()))
    return dx


def bnorm_forward(x, w, b, epsilon=1e-5):
    """Returns (y, moments) with moments the K x 2 (mean, var) tensor."""
    y = torch.empty_like(x)
    K = hwcn_shape(x)[2]
    mom = torch.empty(2 * K, device=x.device)
    hd = handle()
    hd.check(lib().ck_bnorm_forward(hd.h, _t(x), _vec(w), _vec(b), epsilon, _t(y),
                                    _vec(mom, (K, 2, 1, 1)), _stream()))
    return y, mom


def bnorm_infer(x, w, b, epsilon, moments):
    y = torch.empty_like(x)
    K = hwcn_shape(x)[2]
    hd = handle()
    hd.check(lib().ck_bnorm_infer(hd.h, _t(x), _vec(w), _vec(b), epsilon,
                                  _vec(moments, (K, 2, 1, 1)), _t(y), _stream()))
    return y


def bnorm_backward(x, w, b, epsilon, dy):
    dx, dw, db = torch.empty_like(x), torch.empty_like(w), torch.empty_like(b)
    hd = handle()
    hd.check(lib().ck_bnorm_backward(hd.h, _t(x), _vec(w), _vec(b), epsilon, _t(dy), _t(dx),
                                     _vec(dw), _vec(db), 0, _stream()))
    return dx, dw, db


def loss_forward(x, labels, weights=None, check_labels=True):
    """vl_nnsoftmaxloss forward, kind softmaxlog: the weighted SUM over sites."""
    out = torch.empty(1, device=x.device)
    hd = handle()
    hd.check(lib().ck_softmaxlog_forward(hd.h, _t(x), _t(labels), _t(weights), out.data_ptr(),
                                         int(check_labels), _stream()))
    return out


def loss_backward(x, labels, weights=None, p=1.0):
    dx = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_softmaxlog_backward(hd.h, _t(x), _t(labels), _t(weights), float(p), _t(dx),
                                          0, _stream()))
    return dx


def loss_metrics(x, labels, weights=None, top_k=5):
    """(top-1 error, top-k error) weighted sums: classerror and topk kinds."""
    out = torch.empty(2, device=x.device)
    hd = handle()
    hd.check(lib().ck_loss_metrics(hd.h, _t(x), _t(labels), _t(weights), top_k, out.data_ptr(),
                                   out.data_ptr() + 4, _stream()))
    return out


def sgd_step(w, v, g, lr, momentum, weight_decay):
    hd = handle()
    hd.check(lib().ck_sgd_step(hd.h, w.data_ptr(), v.data_ptr(), g.data_ptr(), w.numel(), lr,
                               momentum, weight_decay, _stream()))


# ---- the rest of the reference block set (blocks_ext.cu) ---------------------------

LOSS_KINDS = ["classerror", "topk", "log", "softmaxlog", "mhinge", "mshinge", "binaryerror",
              "binarylog", "logistic", "hinge"]  # loss.hpp:13-24


def sigmoid_forward(x):
    """activation.cpp:25-38."""
    y = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_sigmoid_forward(hd.h, _t(x), _t(y), _stream()))
    return y


def sigmoid_backward(y, dy):
    """activation.cpp:41-48 (from the forward OUTPUT y)."""
    dx = torch.empty_like(y)
    hd = handle()
    hd.check(lib().ck_sigmoid_backward(hd.h, _t(y), _t(dy), _t(dx), 0, _stream()))
    return dx


def softmax_forward(x):
    """normalize.cpp:309-328 (channel softmax per site)."""
    y = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_softmax_forward(hd.h, _t(x), _t(y), _stream()))
    return y


def softmax_backward(y, dy):
    dx = torch.empty_like(y)
    hd = handle()
    hd.check(lib().ck_softmax_backward(hd.h, _t(y), _t(dy), _t(dx), 0, _stream()))
    return dx


@dataclass
class SpnormParams:
    """convkit::SpnormParams (normalize.hpp:59-64)."""
    window_h: int = 1
    window_w: int = 1
    alpha: float = 1.0
    beta: float = 0.5

    def c(self):
        return ck_spnorm_params(self.window_h, self.window_w, self.alpha, self.beta)


def spnorm_forward(x, p: SpnormParams):
    y = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_spnorm_forward(hd.h, _t(x), C.byref(p.c()), _t(y), _stream()))
    return y


def spnorm_backward(x, p: SpnormParams, dy):
    dx = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_spnorm_backward(hd.h, _t(x), C.byref(p.c()), _t(dy), _t(dx), 0, _stream()))
    return dx


def bilinear_output_shape(xs, gs):
    out = ck_shape()
    hd = handle()
    hd.check(lib().ck_bilinear_output_shape(hd.h, ck_shape(*xs), ck_shape(*gs), C.byref(out)))
    return (out.h, out.w, out.c, out.n)


def bilinear_forward(x, grid):
    """bilinear.cpp:58-89: grid is 2 x outH x outW x N."""
    y = from_hwcn(bilinear_output_shape(hwcn_shape(x), hwcn_shape(grid)), x.device)
    hd = handle()
    hd.check(lib().ck_bilinear_forward(hd.h, _t(x), _t(grid), _t(y), _stream()))
    return y


def bilinear_backward(x, grid, dy):
    dx, dg = torch.empty_like(x), torch.empty_like(grid)
    hd = handle()
    hd.check(lib().ck_bilinear_backward(hd.h, _t(x), _t(grid), _t(dy), _t(dx), _t(dg), 0,
                                        _stream()))
    return dx, dg


def pdist_forward(x, target, p=2.0, no_root=False):
    """loss.cpp:346-371: H x W x 1 x N distances."""
    h, w, c, n = hwcn_shape(x)
    y = from_hwcn((h, w, 1, n), x.device)
    hd = handle()
    hd.check(lib().ck_pdist_forward(hd.h, _t(x), _t(target), float(p), int(no_root), _t(y),
                                    _stream()))
    return y


def pdist_backward(x, target, dy, p=2.0, no_root=False):
    dx, dt = torch.empty_like(x), torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_pdist_backward(hd.h, _t(x), _t(target), float(p), int(no_root), _t(dy),
                                     _t(dx), _t(dt), 0, _stream()))
    return dx, dt


def _kind(kind):
    return LOSS_KINDS.index(kind) if isinstance(kind, str) else int(kind)


def _opts(top_k=5, threshold=0.0, random_ties=False, tie_seed=0):
    return ck_loss_options(int(top_k), float(threshold), int(random_ties), int(tie_seed))


def loss_kind_forward(x, labels, kind="softmaxlog", weights=None, check_labels=True, **opts):
    """loss.cpp:86-228, any LossKind: the weighted SUM of per-sample penalties."""
    out = torch.empty(1, device=x.device)
    hd = handle()
    hd.check(lib().ck_loss_forward(hd.h, _t(x), _t(labels), _t(weights), _kind(kind),
                                   C.byref(_opts(**opts)), out.data_ptr(), int(check_labels),
                                   _stream()))
    return out


def loss_kind_backward(x, labels, kind="softmaxlog", weights=None, p=1.0):
    """loss.cpp:231-343, any LossKind (error kinds: exact zeros)."""
    dx = torch.empty_like(x)
    hd = handle()
    hd.check(lib().ck_loss_backward(hd.h, _t(x), _t(labels), _t(weights), _kind(kind), None,
                                    float(p), _t(dx), 0, _stream()))
    return dx

