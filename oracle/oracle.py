"""ctypes front-end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``libck_oracle.so`` -- the plain-C restatement (``ck_oracle.c``); always
  available, the checker every ``-m gpu`` parity test compares against.
* ``_ref/libconvkit_ref.so`` -- the reference convkit sources compiled verbatim
  (plus an Eigen subset shim); used to pin the restatement and as the timed
  CPU baseline.  Absent when the reference was never built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module.  The product path never does.

All arrays are numpy, HWCN, Fortran-free flat order i + H*(j + W*(c + C*n));
shapes are 4-tuples (h, w, c, n).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = os.path.join(HERE, "libck_oracle.so")
_REF = os.path.join(HERE, "_ref", "libconvkit_ref.so")

D = C.POINTER(C.c_double)
F = C.POINTER(C.c_float)
I64 = C.POINTER(C.c_int64)


class Shape(C.Structure):
    _fields_ = [("h", C.c_int64), ("w", C.c_int64), ("c", C.c_int64), ("n", C.c_int64)]


class OracleError(Exception):
    """ShapeError (code 1) / DataError (code 2) raised by the oracle."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE):
            build()
        _lib = C.CDLL(_ORACLE)
        _lib.cko_last_error.restype = C.c_char_p
        _lib.cko_rng_new.restype = C.c_void_p
        _lib.cko_rng_new.argtypes = [C.c_uint64]
        _lib.cko_rng_free.argtypes = [C.c_void_p]
        _lib.cko_rng_next.restype = C.c_uint64
        _lib.cko_rng_next.argtypes = [C.c_void_p]
        _lib.cko_rng_fill_uniform_f.argtypes = [C.c_void_p, F, C.c_int64, C.c_float, C.c_float]
        _lib.cko_rng_fill_normal_f.argtypes = [C.c_void_p, F, C.c_int64, C.c_float]
        _lib.cko_rng_fill_labels_f.argtypes = [C.c_void_p, F, C.c_int64, C.c_uint64]
        _lib.cko_lrn_forward.argtypes = [D, Shape, C.c_int64, C.c_double, C.c_double, C.c_double, D]
        _lib.cko_lrn_backward.argtypes = [D, Shape, C.c_int64, C.c_double, C.c_double,
                                          C.c_double, D, D]
        _lib.cko_bnorm_forward.argtypes = [D, Shape, D, D, C.c_double, D, D, D]
        _lib.cko_bnorm_infer.argtypes = [D, Shape, D, D, C.c_double, D, D, D]
        _lib.cko_bnorm_backward.argtypes = [D, Shape, D, D, C.c_double, D, D, D, D]
        _lib.cko_loss_forward.argtypes = [D, Shape, D, Shape, D, C.c_int, C.c_int64, D]
        _lib.cko_softmaxlog_backward.argtypes = [D, Shape, D, Shape, D, C.c_double, D]
        _lib.cko_sgd_step_f.argtypes = [F, F, F, C.c_int64, C.c_float, C.c_float, C.c_float]
        _lib.cko_relu_forward_f.argtypes = [F, C.c_int64, F]
        _lib.cko_relu_backward_f.argtypes = [F, F, C.c_int64, F]
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF)


def ref():
    """The verbatim reference build (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{_REF} not built (reference sources absent)")
        _ref = C.CDLL(_REF)
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_graph_new.restype = C.c_void_p
        for fn in ("ref_graph_free", "ref_graph_add_input", "ref_graph_add_param",
                   "ref_graph_add_layer", "ref_graph_finalize", "ref_graph_bind",
                   "ref_graph_forward_backward", "ref_graph_get"):
            getattr(_ref, fn).argtypes = None
        _ref.ref_graph_free.argtypes = [C.c_void_p]
        _ref.ref_graph_add_input.argtypes = [C.c_void_p, C.c_char_p]
        _ref.ref_graph_add_param.argtypes = [C.c_void_p, C.c_char_p]
        _ref.ref_graph_add_layer.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                             C.c_char_p, D, C.c_int]
        _ref.ref_graph_finalize.argtypes = [C.c_void_p]
        _ref.ref_graph_bind.argtypes = [C.c_void_p, C.c_char_p, F, I64]
        _ref.ref_graph_forward_backward.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        _ref.ref_graph_get.argtypes = [C.c_void_p, C.c_char_p, C.c_int, F, I64]
        _ref.ref_lrn_forward.argtypes = [F, I64, C.c_int64, C.c_double, C.c_double, C.c_double, F]
        _ref.ref_lrn_backward.argtypes = [F, I64, C.c_int64, C.c_double, C.c_double, C.c_double,
                                          F, F]
        _ref.ref_bnorm_forward.argtypes = [F, I64, F, F, C.c_double, F, F]
        _ref.ref_bnorm_backward.argtypes = [F, I64, F, F, C.c_double, F, F, F, F]
        _ref.ref_loss_forward.argtypes = [F, I64, F, I64, F, C.c_char_p, C.c_int64, F]
        _ref.ref_loss_backward.argtypes = [F, I64, F, I64, F, C.c_char_p, C.c_float, F]
        _ref.ref_loss_forward2.argtypes = [F, I64, F, I64, F, C.c_int, C.c_int64, C.c_double,
                                           C.c_int, C.c_uint64, F]
        _ref.ref_loss_backward2.argtypes = [F, I64, F, I64, F, C.c_int, C.c_float, F]
        _ref.ref_spnorm_forward.argtypes = [F, I64, C.c_int64, C.c_int64, C.c_double, C.c_double, F]
        _ref.ref_spnorm_backward.argtypes = [F, I64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                             F, F]
        _ref.ref_pdist_forward.argtypes = [F, F, I64, C.c_double, C.c_int, F]
        _ref.ref_pdist_backward.argtypes = [F, F, I64, C.c_double, C.c_int, F, I64, F, F]
        _ref.ref_write_blob.argtypes = [C.c_char_p, F, I64]
        _ref.ref_read_blob.argtypes = [C.c_char_p, F, I64]
        _ref.ref_rng_permutation.argtypes = [C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p]
    return _ref


# ---- helpers ---------------------------------------------------------------

def _d(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _f(a):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=np.float32)


def _pd(a):
    return None if a is None else a.ctypes.data_as(D)


def _pf(a):
    return None if a is None else a.ctypes.data_as(F)


def _g(g, n):
    arr = (C.c_int64 * n)(*[int(v) for v in g])
    return arr


def _check(code):
    if code:
        raise OracleError(code, lib().cko_last_error().decode())


def _check_ref(code):
    if code:
        raise OracleError(code, ref().ref_last_error().decode())


def size(s):
    return int(s[0] * s[1] * s[2] * s[3])


# ---- geometry ----------------------------------------------------------------

def conv_output_shape(xs, fs, geom):
    out = Shape()
    _check(lib().cko_conv_output_shape(Shape(*xs), Shape(*fs), _g(geom, 7), C.byref(out)))
    return (out.h, out.w, out.c, out.n)


def convt_output_shape(xs, fs, cg):
    out = Shape()
    _check(lib().cko_convt_output_shape(Shape(*xs), Shape(*fs), _g(cg, 6), C.byref(out)))
    return (out.h, out.w, out.c, out.n)


def pool_output_shape(xs, pg):
    out = Shape()
    _check(lib().cko_pool_output_shape(Shape(*xs), _g(pg, 9), C.byref(out)))
    return (out.h, out.w, out.c, out.n)


# ---- blocks (double restatement) -------------------------------------------

def im2row(x, xs, fh, fw, geom):
    rows, cols = C.c_int64(), C.c_int64()
    x = _d(x)
    _check(lib().cko_im2row(_pd(x), Shape(*xs), C.c_int64(fh), C.c_int64(fw), _g(geom, 7), None,
                            C.byref(rows), C.byref(cols)))
    A = np.zeros(rows.value * cols.value)
    _check(lib().cko_im2row(_pd(x), Shape(*xs), C.c_int64(fh), C.c_int64(fw), _g(geom, 7),
                            _pd(A), C.byref(rows), C.byref(cols)))
    return A, rows.value, cols.value


def row2im(A, target, fh, fw, geom):
    x = np.zeros(size(target))
    A = _d(A)
    _check(lib().cko_row2im(_pd(A), Shape(*target), C.c_int64(fh), C.c_int64(fw), _g(geom, 7),
                            _pd(x)))
    return x


def conv_forward(x, xs, f, fs, bias, geom):
    ys = conv_output_shape(xs, fs, geom)
    x, f, bias = _d(x), _d(f), _d(bias)
    y = np.zeros(size(ys))
    _check(lib().cko_conv_forward(_pd(x), Shape(*xs), _pd(f), Shape(*fs), _pd(bias),
                                  _g(geom, 7), _pd(y)))
    return y, ys


def conv_backward(x, xs, f, fs, geom, dy, want=(True, True, True)):
    x, f, dy = _d(x), _d(f), _d(dy)
    dx = np.zeros(size(xs)) if want[0] else None
    df = np.zeros(size(fs)) if want[1] else None
    db = np.zeros(fs[3]) if want[2] else None
    _check(lib().cko_conv_backward(_pd(x), Shape(*xs), _pd(f), Shape(*fs), _g(geom, 7), _pd(dy),
                                   _pd(dx), _pd(df), _pd(db)))
    return dx, df, db


def convt_forward(x, xs, f, fs, cg):
    ys = convt_output_shape(xs, fs, cg)
    x, f = _d(x), _d(f)
    y = np.zeros(size(ys))
    _check(lib().cko_convt_forward(_pd(x), Shape(*xs), _pd(f), Shape(*fs), _g(cg, 6), _pd(y)))
    return y, ys


def convt_backward(x, xs, f, fs, cg, dy):
    x, f, dy = _d(x), _d(f), _d(dy)
    dx = np.zeros(size(xs))
    df = np.zeros(size(fs))
    _check(lib().cko_convt_backward(_pd(x), Shape(*xs), _pd(f), Shape(*fs), _g(cg, 6), _pd(dy),
                                    _pd(dx), _pd(df)))
    return dx, df


def pool_forward(x, xs, pg):
    ys = pool_output_shape(xs, pg)
    x = _f(x)
    y = np.zeros(size(ys), np.float32)
    _check(lib().cko_pool_forward_f(_pf(x), Shape(*xs), _g(pg, 9), _pf(y)))
    return y, ys


def pool_backward(x, xs, pg, dy):
    x, dy = _f(x), _f(dy)
    dx = np.zeros(size(xs), np.float32)
    _check(lib().cko_pool_backward_f(_pf(x), Shape(*xs), _g(pg, 9), _pf(dy), _pf(dx)))
    return dx


def relu_forward(x):
    x = _f(x)
    y = np.empty_like(x)
    lib().cko_relu_forward_f(_pf(x), x.size, _pf(y))
    return y


def relu_backward(x, dy):
    x, dy = _f(x), _f(dy)
    dx = np.empty_like(x)
    lib().cko_relu_backward_f(_pf(x), _pf(dy), x.size, _pf(dx))
    return dx


def lrn_forward(x, xs, n, kappa, alpha, beta):
    x = _d(x)
    y = np.zeros(size(xs))
    _check(lib().cko_lrn_forward(_pd(x), Shape(*xs), n, kappa, alpha, beta, _pd(y)))
    return y


def lrn_backward(x, xs, n, kappa, alpha, beta, dy):
    x, dy = _d(x), _d(dy)
    dx = np.zeros(size(xs))
    _check(lib().cko_lrn_backward(_pd(x), Shape(*xs), n, kappa, alpha, beta, _pd(dy), _pd(dx)))
    return dx


def bnorm_forward(x, xs, w, b, eps):
    x, w, b = _d(x), _d(w), _d(b)
    y = np.zeros(size(xs))
    mean = np.zeros(xs[2])
    var = np.zeros(xs[2])
    _check(lib().cko_bnorm_forward(_pd(x), Shape(*xs), _pd(w), _pd(b), eps, _pd(y), _pd(mean),
                                   _pd(var)))
    return y, mean, var


def bnorm_infer(x, xs, w, b, eps, mean, var):
    x, w, b, mean, var = _d(x), _d(w), _d(b), _d(mean), _d(var)
    y = np.zeros(size(xs))
    _check(lib().cko_bnorm_infer(_pd(x), Shape(*xs), _pd(w), _pd(b), eps, _pd(mean), _pd(var),
                                 _pd(y)))
    return y


def bnorm_backward(x, xs, w, b, eps, dy):
    x, w, b, dy = _d(x), _d(w), _d(b), _d(dy)
    dx = np.zeros(size(xs))
    dw = np.zeros(xs[2])
    db = np.zeros(xs[2])
    _check(lib().cko_bnorm_backward(_pd(x), Shape(*xs), _pd(w), _pd(b), eps, _pd(dy), _pd(dx),
                                    _pd(dw), _pd(db)))
    return dx, dw, db


LOSS_KINDS = {"softmaxlog": 0, "classerror": 1, "topk": 2}


def loss_forward(x, xs, labels, cs, weights=None, kind="softmaxlog", top_k=5):
    x, labels, weights = _d(x), _d(labels), _d(weights)
    out = C.c_double()
    _check(lib().cko_loss_forward(_pd(x), Shape(*xs), _pd(labels), Shape(*cs), _pd(weights),
                                  LOSS_KINDS[kind], top_k, C.byref(out)))
    return out.value


def softmaxlog_backward(x, xs, labels, cs, weights=None, p=1.0):
    x, labels, weights = _d(x), _d(labels), _d(weights)
    dx = np.zeros(size(xs))
    _check(lib().cko_softmaxlog_backward(_pd(x), Shape(*xs), _pd(labels), Shape(*cs),
                                         _pd(weights), p, _pd(dx)))
    return dx


def sgd_step(w, v, g, lr, momentum, wd):
    w, v, g = _f(w).copy(), _f(v).copy(), _f(g)
    lib().cko_sgd_step_f(_pf(w), _pf(v), _pf(g), w.size, lr, momentum, wd)
    return w, v


# ---- synthetic inputs (xoshiro256**, identical on host for oracle and GPU) ----

class Rng:
    """The reference Xoshiro256 stream (rng.cpp:21-59)."""

    def __init__(self, seed: int):
        self._h = C.c_void_p(lib().cko_rng_new(seed))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cko_rng_free(self._h)
            self._h = None

    def next(self) -> int:
        return lib().cko_rng_next(self._h)

    def uniform(self, n, lo=-1.0, hi=1.0):
        out = np.empty(int(n), np.float32)
        lib().cko_rng_fill_uniform_f(self._h, _pf(out), out.size, lo, hi)
        return out

    def normal(self, n, scale=1.0):
        out = np.empty(int(n), np.float32)
        lib().cko_rng_fill_normal_f(self._h, _pf(out), out.size, scale)
        return out

    def labels(self, n, classes):
        out = np.empty(int(n), np.float32)
        lib().cko_rng_fill_labels_f(self._h, _pf(out), out.size, classes)
        return out


# ---- the verbatim reference (oracle/_ref) --------------------------------------

def _s(s):
    return (C.c_int64 * 4)(*[int(v) for v in s])


def ref_conv_forward(x, xs, f, fs, bias, geom):
    ys = conv_output_shape(xs, fs, geom)
    x, f, bias = _f(x), _f(f), _f(bias)
    y = np.zeros(size(ys), np.float32)
    _check_ref(ref().ref_conv_forward(_pf(x), _s(xs), _pf(f), _s(fs), _pf(bias), _g(geom, 7),
                                      _pf(y)))
    return y, ys


def ref_conv_backward(x, xs, f, fs, geom, dy, want=(True, True, True)):
    ys = conv_output_shape(xs, fs, geom)
    x, f, dy = _f(x), _f(f), _f(dy)
    dx = np.zeros(size(xs), np.float32) if want[0] else None
    df = np.zeros(size(fs), np.float32) if want[1] else None
    db = np.zeros(fs[3], np.float32) if want[2] else None
    _check_ref(ref().ref_conv_backward(_pf(x), _s(xs), _pf(f), _s(fs), _g(geom, 7), _pf(dy),
                                       _s(ys), _pf(dx), _pf(df), _pf(db)))
    return dx, df, db


def ref_convt_forward(x, xs, f, fs, cg):
    ys = convt_output_shape(xs, fs, cg)
    x, f = _f(x), _f(f)
    y = np.zeros(size(ys), np.float32)
    _check_ref(ref().ref_convt_forward(_pf(x), _s(xs), _pf(f), _s(fs), _g(cg, 6), _pf(y)))
    return y, ys


def ref_convt_backward(x, xs, f, fs, cg, dy):
    ys = convt_output_shape(xs, fs, cg)
    x, f, dy = _f(x), _f(f), _f(dy)
    dx = np.zeros(size(xs), np.float32)
    df = np.zeros(size(fs), np.float32)
    _check_ref(ref().ref_convt_backward(_pf(x), _s(xs), _pf(f), _s(fs), _g(cg, 6), _pf(dy),
                                        _s(ys), _pf(dx), _pf(df)))
    return dx, df


def ref_pool_forward(x, xs, pg):
    ys = pool_output_shape(xs, pg)
    x = _f(x)
    y = np.zeros(size(ys), np.float32)
    _check_ref(ref().ref_pool_forward(_pf(x), _s(xs), _g(pg, 9), _pf(y)))
    return y, ys


def ref_pool_backward(x, xs, pg, dy):
    ys = pool_output_shape(xs, pg)
    x, dy = _f(x), _f(dy)
    dx = np.zeros(size(xs), np.float32)
    _check_ref(ref().ref_pool_backward(_pf(x), _s(xs), _g(pg, 9), _pf(dy), _s(ys), _pf(dx)))
    return dx


def ref_relu(x, dy=None):
    x = _f(x)
    out = np.zeros_like(x)
    s = _s((x.size, 1, 1, 1))
    if dy is None:
        _check_ref(ref().ref_relu_forward(_pf(x), s, _pf(out)))
    else:
        dy = _f(dy)
        _check_ref(ref().ref_relu_backward(_pf(x), s, _pf(dy), _pf(out)))
    return out


def ref_lrn_forward(x, xs, n, kappa, alpha, beta):
    x = _f(x)
    y = np.zeros(size(xs), np.float32)
    _check_ref(ref().ref_lrn_forward(_pf(x), _s(xs), n, kappa, alpha, beta, _pf(y)))
    return y


def ref_lrn_backward(x, xs, n, kappa, alpha, beta, dy):
    x, dy = _f(x), _f(dy)
    dx = np.zeros(size(xs), np.float32)
    _check_ref(ref().ref_lrn_backward(_pf(x), _s(xs), n, kappa, alpha, beta, _pf(dy), _pf(dx)))
    return dx


def ref_bnorm_forward(x, xs, w, b, eps):
    x, w, b = _f(x), _f(w), _f(b)
    y = np.zeros(size(xs), np.float32)
    m = np.zeros(2 * xs[2], np.float32)
    _check_ref(ref().ref_bnorm_forward(_pf(x), _s(xs), _pf(w), _pf(b), eps, _pf(y), _pf(m)))
    return y, m[: xs[2]], m[xs[2]:]


def ref_bnorm_backward(x, xs, w, b, eps, dy):
    x, w, b, dy = _f(x), _f(w), _f(b), _f(dy)
    dx = np.zeros(size(xs), np.float32)
    dw = np.zeros(xs[2], np.float32)
    db = np.zeros(xs[2], np.float32)
    _check_ref(ref().ref_bnorm_backward(_pf(x), _s(xs), _pf(w), _pf(b), eps, _pf(dy), _pf(dx),
                                        _pf(dw), _pf(db)))
    return dx, dw, db


def ref_loss_forward(x, xs, labels, cs, weights=None, kind="softmaxlog", top_k=5):
    x, labels, weights = _f(x), _f(labels), _f(weights)
    out = C.c_float()
    _check_ref(ref().ref_loss_forward(_pf(x), _s(xs), _pf(labels), _s(cs), _pf(weights),
                                      kind.encode(), top_k, C.byref(out)))
    return out.value


def ref_loss_backward(x, xs, labels, cs, weights=None, kind="softmaxlog", p=1.0):
    x, labels, weights = _f(x), _f(labels), _f(weights)
    dx = np.zeros(size(xs), np.float32)
    _check_ref(ref().ref_loss_backward(_pf(x), _s(xs), _pf(labels), _s(cs), _pf(weights),
                                       kind.encode(), p, _pf(dx)))
    return dx


def ref_loss(x, xs, labels, cs, weights=None, kind=3, top_k=5, threshold=0.0, random_ties=0,
             tie_seed=0):
    """loss.cpp:86 with the full LossOptions (kind: LossKind index)."""
    x, labels, weights = _f(x), _f(labels), _f(weights)
    out = C.c_float()
    _check_ref(ref().ref_loss_forward2(_pf(x), _s(xs), _pf(labels), _s(cs), _pf(weights), kind,
                                       top_k, threshold, random_ties, tie_seed, C.byref(out)))
    return out.value


def ref_loss_grad(x, xs, labels, cs, weights=None, kind=3, p=1.0):
    x, labels, weights = _f(x), _f(labels), _f(weights)
    dx = np.zeros(size(xs), np.float32)
    _check_ref(ref().ref_loss_backward2(_pf(x), _s(xs), _pf(labels), _s(cs), _pf(weights), kind,
                                        p, _pf(dx)))
    return dx


def ref_sigmoid(x, dy=None, y=None):
    """activation.cpp:25 forward (dy None) or :41 backward from the OUTPUT y."""
    if dy is None:
        x = _f(x)
        out = np.zeros_like(x)
        _check_ref(ref().ref_sigmoid_forward(_pf(x), _s((x.size, 1, 1, 1)), _pf(out)))
        return out
    y, dy = _f(y), _f(dy)
    out = np.zeros_like(y)
    _check_ref(ref().ref_sigmoid_backward(_pf(y), _s((y.size, 1, 1, 1)), _pf(dy), _pf(out)))
    return out


def ref_softmax(x, xs, dy=None, y=None):
    """normalize.cpp:309 forward or :330 backward from the OUTPUT y."""
    if dy is None:
        x = _f(x)
        out = np.zeros_like(x)
        _check_ref(ref().ref_softmax_forward(_pf(x), _s(xs), _pf(out)))
        return out
    y, dy = _f(y), _f(dy)
    out = np.zeros_like(y)
    _check_ref(ref().ref_softmax_backward(_pf(y), _s(xs), _pf(dy), _pf(out)))
    return out


def ref_spnorm(x, xs, wh, ww, alpha, beta, dy=None):
    x = _f(x)
    out = np.zeros_like(x)
    if dy is None:
        _check_ref(ref().ref_spnorm_forward(_pf(x), _s(xs), wh, ww, alpha, beta, _pf(out)))
    else:
        dy = _f(dy)
        _check_ref(ref().ref_spnorm_backward(_pf(x), _s(xs), wh, ww, alpha, beta, _pf(dy),
                                             _pf(out)))
    return out


def ref_bilinear(x, xs, g, gs, dy=None):
    ys = (gs[1], gs[2], xs[2], xs[3])
    x, g = _f(x), _f(g)
    if dy is None:
        y = np.zeros(size(ys), np.float32)
        _check_ref(ref().ref_bilinear_forward(_pf(x), _s(xs), _pf(g), _s(gs), _pf(y)))
        return y
    dy = _f(dy)
    dx = np.zeros(size(xs), np.float32)
    dg = np.zeros(size(gs), np.float32)
    _check_ref(ref().ref_bilinear_backward(_pf(x), _s(xs), _pf(g), _s(gs), _pf(dy), _s(ys),
                                           _pf(dx), _pf(dg)))
    return dx, dg


def ref_pdist(x, t, xs, p, no_root, dy=None):
    ys = (xs[0], xs[1], 1, xs[3])
    x, t = _f(x), _f(t)
    if dy is None:
        y = np.zeros(size(ys), np.float32)
        _check_ref(ref().ref_pdist_forward(_pf(x), _pf(t), _s(xs), p, int(no_root), _pf(y)))
        return y
    dy = _f(dy)
    dx = np.zeros(size(xs), np.float32)
    dt = np.zeros(size(xs), np.float32)
    _check_ref(ref().ref_pdist_backward(_pf(x), _pf(t), _s(xs), p, int(no_root), _pf(dy), _s(ys),
                                        _pf(dx), _pf(dt)))
    return dx, dt


def ref_write_blob(path, data, shape):
    _check_ref(ref().ref_write_blob(str(path).encode(), _pf(_f(data)), _s(shape)))


def ref_read_blob(path):
    s = (C.c_int64 * 4)()
    _check_ref(ref().ref_read_blob(str(path).encode(), None, s))
    out = np.zeros(size(tuple(s)), np.float32)
    _check_ref(ref().ref_read_blob(str(path).encode(), _pf(out), s))
    return out, tuple(s)


def ref_permutation(seed, n):
    """rng.cpp:51-59 Xoshiro256(seed).permutation(n) and the generator state after it."""
    out = np.zeros(n, np.int64)
    st = np.zeros(4, np.uint64)
    _check_ref(ref().ref_rng_permutation(seed, n, out.ctypes.data, st.ctypes.data))
    return out, st


class RefGraph:
    """The reference DAG engine (graph.hpp) driven through oracle/_ref."""

    def __init__(self):
        self.h = C.c_void_p(ref().ref_graph_new())

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_graph_free(self.h)
            self.h = None

    def add_input(self, name):
        _check_ref(ref().ref_graph_add_input(self.h, name.encode()))

    def add_param(self, name):
        _check_ref(ref().ref_graph_add_param(self.h, name.encode()))

    def add_layer(self, kind, name, inputs, outputs, params=()):
        p = (C.c_double * max(1, len(params)))(*[float(v) for v in params])
        _check_ref(ref().ref_graph_add_layer(self.h, kind.encode(), name.encode(),
                                             ",".join(inputs).encode(), ",".join(outputs).encode(),
                                             p, len(params)))

    def finalize(self):
        _check_ref(ref().ref_graph_finalize(self.h))

    def bind(self, name, data, shape):
        data = _f(data)
        assert data.size == size(shape)
        _check_ref(ref().ref_graph_bind(self.h, name.encode(), _pf(data), _s(shape)))

    def run(self, objective="objective", backward=True):
        _check_ref(ref().ref_graph_forward_backward(self.h, objective.encode(), int(backward)))

    def get(self, name, deriv=False):
        s = (C.c_int64 * 4)()
        _check_ref(ref().ref_graph_get(self.h, name.encode(), int(deriv), None, s))
        out = np.zeros(size(tuple(s)), np.float32)
        _check_ref(ref().ref_graph_get(self.h, name.encode(), int(deriv), _pf(out), s))
        return out, tuple(s)
