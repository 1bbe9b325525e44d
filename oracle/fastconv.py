"""Full-size double-precision convolution oracle -- TEST INFRASTRUCTURE ONLY.

The same algorithm as ck_oracle.c's conv (conv.cpp:193-280: per-image
im2row, one product per group, bias after the product; dF += A_n^T P_n;
M = P_n F^T then row2im), with the per-image patch matrices built by the C
restatement (cko_im2row / cko_row2im, conv.cpp:35-84) and the products done
by numpy's float64 GEMM over chunks of images, so the BASELINE batch sizes
(AlexNet b=256: 1.11 TFLOP per fwd+bwd) finish in seconds.  Accumulation is
double throughout, so this is a reference for both the FP32 and the TF32
device paths (with `q` = chain.tf32_operand for the latter's operand
rounding).
"""
from __future__ import annotations

import numpy as np

import oracle as O


def _geom(xs, fs, geom):
    ys = O.conv_output_shape(xs, fs, geom)
    rows = ys[0] * ys[1]
    groups = int(geom[6])
    gcols = fs[0] * fs[1] * fs[2]
    gfil = fs[3] // groups
    return ys, rows, groups, gcols, gfil


def _patches(x, xs, fs, geom, n0, n1):
    """Stacked im2row of images n0..n1-1: (B, rows, patch), column-major rows."""
    per = xs[0] * xs[1] * xs[2]
    one = (xs[0], xs[1], xs[2], 1)
    mats = []
    for n in range(n0, n1):
        A, rows, cols = O.im2row(x[n * per:(n + 1) * per], one, fs[0], fs[1], geom)
        mats.append(A.reshape(cols, rows).T)
    return np.stack(mats)


def _fmat(f, fs):
    """Filter bank as the (fh*fw*Cg) x K matrix (conv.cpp:11-16)."""
    return np.asarray(f, np.float64).reshape(fs[3], fs[0] * fs[1] * fs[2]).T


def conv_forward(x, xs, f, fs, bias, geom, q=None, chunk=16):
    q = q or (lambda a: np.asarray(a, np.float64))
    x, F = q(x).ravel(), _fmat(q(f), fs)
    ys, rows, groups, gcols, gfil = _geom(xs, fs, geom)
    y = np.empty((xs[3], ys[2], rows))
    for n0 in range(0, xs[3], chunk):
        n1 = min(xs[3], n0 + chunk)
        A = _patches(x, xs, fs, geom, n0, n1)
        for t in range(groups):
            Yt = A[:, :, t * gcols:(t + 1) * gcols] @ F[:, t * gfil:(t + 1) * gfil]
            y[n0:n1, t * gfil:(t + 1) * gfil, :] = Yt.transpose(0, 2, 1)
    if bias is not None:
        y += np.asarray(bias, np.float64).reshape(1, -1, 1)
    return y.ravel(), ys


def conv_backward(x, xs, f, fs, geom, dy, want=(True, True, True), q=None, chunk=16):
    """(dx, df, db); q rounds the operands of the data and filter gradients
    (dy, f for dx; x, dy for df); db is the plain sum of dy."""
    q = q or (lambda a: np.asarray(a, np.float64))
    ys, rows, groups, gcols, gfil = _geom(xs, fs, geom)
    D = np.asarray(dy, np.float64).reshape(xs[3], ys[2], rows)
    Dq = q(dy).reshape(xs[3], ys[2], rows)
    F = _fmat(q(f), fs)
    xq = q(x).ravel()
    per = xs[0] * xs[1] * xs[2]
    one = (xs[0], xs[1], xs[2], 1)
    dx = np.zeros(xs[3] * per) if want[0] else None
    df = np.zeros((gcols, fs[3])) if want[1] else None
    for n0 in range(0, xs[3], chunk):
        n1 = min(xs[3], n0 + chunk)
        P = Dq[n0:n1].transpose(0, 2, 1)  # (B, rows, K)
        if want[1]:
            A = _patches(xq, xs, fs, geom, n0, n1)
            for t in range(groups):
                At = A[:, :, t * gcols:(t + 1) * gcols].reshape(-1, gcols)
                Pt = P[:, :, t * gfil:(t + 1) * gfil].reshape(-1, gfil)
                df[:, t * gfil:(t + 1) * gfil] += At.T @ Pt
        if want[0]:
            for b, n in enumerate(range(n0, n1)):
                M = np.empty((rows, gcols * groups))
                for t in range(groups):
                    M[:, t * gcols:(t + 1) * gcols] = (P[b, :, t * gfil:(t + 1) * gfil] @
                                                       F[:, t * gfil:(t + 1) * gfil].T)
                dx[n * per:(n + 1) * per] = O.row2im(M.T.ravel(), one, fs[0], fs[1], geom)
    db = D.sum(axis=(0, 2)) if want[2] else None
    return dx, (df.T.ravel() if want[1] else None), db
