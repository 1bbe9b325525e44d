"""Restatement of the rest of the reference block set -- TEST INFRASTRUCTURE ONLY.

numpy (float64) restatements of sigmoid, channel softmax, spnorm, the
bilinear sampler, pdist and every loss kind, each citing the reference
function it follows (/root/reference/proj/src).  Used by tests/ as the
checker of the CUDA kernels (blocks_ext.cu); pinned against the reference
compiled verbatim (oracle/_ref) by tests/test_oracle_ext.py.

Tensors are flat HWCN (tensor.hpp:70-72): element (i, j, c, n) at
i + H*(j + W*(c + C*n)), i.e. a numpy array of shape (N, C, W, H).
"""
from __future__ import annotations

import numpy as np

KINDS = ["classerror", "topk", "log", "softmaxlog", "mhinge", "mshinge", "binaryerror",
         "binarylog", "logistic", "hinge"]  # loss.hpp:13-24 order


class DataError(ValueError):
    pass


def _v(a, s):
    """flat HWCN -> (N, C, W, H) float64 view."""
    return np.asarray(a, np.float64).reshape(s[3], s[2], s[1], s[0])


# activation.cpp:25-38
def sigmoid_forward(x):
    x = np.asarray(x, np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


# activation.cpp:41-48 (consumes the forward output)
def sigmoid_backward(y, dy):
    y, dy = np.asarray(y, np.float64), np.asarray(dy, np.float64)
    return dy * y * (1.0 - y)


# normalize.cpp:309-328
def softmax_forward(x, xs):
    v = _v(x, xs)
    e = np.exp(v - v.max(axis=1, keepdims=True))
    return (e / e.sum(axis=1, keepdims=True)).ravel()


# normalize.cpp:330-347
def softmax_backward(y, xs, dy):
    yv, g = _v(y, xs), _v(dy, xs)
    dot = (g * yv).sum(axis=1, keepdims=True)
    return (yv * (g - dot)).ravel()


# normalize.cpp:29-42 spnorm_pool_geom + pool.cpp:20-33 window_at, avg mode
def _box_mean(sq, wh, ww):
    """Clipped centred window mean of a (N, C, W, H) array (stride 1)."""
    H, W = sq.shape[3], sq.shape[2]
    pt, pl = (wh - 1) // 2, (ww - 1) // 2
    out = np.zeros_like(sq)
    area = np.zeros((W, H))
    for j in range(W):
        j0, j1 = max(0, j - pl), min(W, j - pl + ww)
        for i in range(H):
            i0, i1 = max(0, i - pt), min(H, i - pt + wh)
            out[:, :, j, i] = sq[:, :, j0:j1, i0:i1].sum(axis=(2, 3))
            area[j, i] = (i1 - i0) * (j1 - j0)
    return out / area, area


def _box_adjoint(eta, area, wh, ww):
    """pool_backward avg (pool.cpp:113-118): spread share = eta / area over each window."""
    H, W = eta.shape[3], eta.shape[2]
    pt, pl = (wh - 1) // 2, (ww - 1) // 2
    share = eta / area
    out = np.zeros_like(eta)
    for j in range(W):
        j0, j1 = max(0, j - pl), min(W, j - pl + ww)
        for i in range(H):
            i0, i1 = max(0, i - pt), min(H, i - pt + wh)
            out[:, :, j0:j1, i0:i1] += share[:, :, j, i][:, :, None, None]
    return out


# normalize.cpp:268-281
def spnorm_forward(x, xs, wh, ww, alpha, beta):
    v = _v(x, xs)
    energy, _ = _box_mean(v * v, wh, ww)
    return (v * (1.0 + alpha * energy) ** (-beta)).ravel()


# normalize.cpp:284-306
def spnorm_backward(x, xs, wh, ww, alpha, beta, dy):
    v, g = _v(x, xs), _v(dy, xs)
    energy, area = _box_mean(v * v, wh, ww)
    base = 1.0 + alpha * energy
    eta = g * base ** (-beta - 1.0) * v
    spread = _box_adjoint(eta, area, wh, ww)
    return (g * base ** (-beta) - 2.0 * alpha * beta * v * spread).ravel()


# bilinear.cpp:17-37 tent_at
def _tent(v, extent):
    i0 = np.floor(v).astype(np.int64)
    out = []
    for i in (i0, i0 + 1):
        t = v - i
        a = np.abs(t)
        inside = (i >= 0) & (i < extent)
        w = np.where(inside & (a < 1), 1 - a, 0.0)
        d = np.where(inside & (a < 1) & (t != 0), np.where(t > 0, -1.0, 1.0), 0.0)
        out.append((i, w, d))
    return out


def bilinear_output_shape(xs, gs):
    if gs[0] != 2:
        raise ValueError("sampling grid must have two coordinate channels")
    if gs[3] != xs[3]:
        raise ValueError("sampling grid batch does not match input batch")
    return (gs[1], gs[2], xs[2], xs[3])


# bilinear.cpp:58-89
def bilinear_forward(x, xs, grid, gs):
    H, W, C, N = xs
    ys = bilinear_output_shape(xs, gs)
    OH, OW = ys[0], ys[1]
    X = _v(x, xs)                                   # (N, C, W, H)
    G = np.asarray(grid, np.float64).reshape(N, OW, OH, 2)
    v = (H - 1) / 2.0 * (G[..., 0] + 1)             # (N, OW, OH)
    u = (W - 1) / 2.0 * (G[..., 1] + 1)
    Y = np.zeros((N, C, OW, OH))
    nn = np.arange(N)[:, None, None]
    for (iv, wv, _) in _tent(v, H):
        for (iu, wu, _) in _tent(u, W):
            w = wv * wu
            ok = w != 0
            ii, jj = np.clip(iv, 0, H - 1), np.clip(iu, 0, W - 1)
            vals = X[nn, :, jj, ii]                 # (N, OW, OH, C)
            Y += np.moveaxis(vals * (w * ok)[..., None], 3, 1)
    return Y.ravel(), ys


# bilinear.cpp:92-132
def bilinear_backward(x, xs, grid, gs, dy):
    H, W, C, N = xs
    ys = bilinear_output_shape(xs, gs)
    OH, OW = ys[0], ys[1]
    X = _v(x, xs)
    G = np.asarray(grid, np.float64).reshape(N, OW, OH, 2)
    D = np.asarray(dy, np.float64).reshape(N, C, OW, OH)
    av, au = (H - 1) / 2.0, (W - 1) / 2.0
    v, u = av * (G[..., 0] + 1), au * (G[..., 1] + 1)
    dX = np.zeros_like(X)
    g1 = np.zeros((N, OW, OH))
    g2 = np.zeros((N, OW, OH))
    nn = np.broadcast_to(np.arange(N)[:, None, None], v.shape)
    Dm = np.moveaxis(D, 1, 3)                       # (N, OW, OH, C)
    for (iv, wv, dv) in _tent(v, H):
        for (iu, wu, du) in _tent(u, W):
            ok = (iv >= 0) & (iv < H) & (iu >= 0) & (iu < W)
            ii, jj = np.clip(iv, 0, H - 1), np.clip(iu, 0, W - 1)
            xv = X[nn, :, jj, ii]                   # (N, OW, OH, C)
            pxv = (Dm * xv).sum(axis=3) * ok
            g1 += pxv * dv * wu
            g2 += pxv * wv * du
            contrib = Dm * (wv * wu * ok)[..., None]
            for c in range(C):
                np.add.at(dX[:, c], (nn[ok], jj[ok], ii[ok]), contrib[..., c][ok])
    dG = np.stack([av * g1, au * g2], axis=-1)
    return dX.ravel(), dG.ravel()


# loss.cpp:346-371
def pdist_forward(x, t, xs, p, no_root):
    d = np.abs(_v(x, xs) - _v(t, xs))
    acc = (d ** p).sum(axis=1)                      # (N, W, H)
    return (acc if no_root else acc ** (1.0 / p)).ravel()


# loss.cpp:374-428
def pdist_backward(x, t, xs, p, no_root, dy):
    diff = _v(x, xs) - _v(t, xs)
    sgn, a = np.sign(diff), np.abs(diff)
    g = np.asarray(dy, np.float64).reshape(xs[3], 1, xs[1], xs[0])
    y = pdist_forward(x, t, xs, p, no_root).reshape(xs[3], 1, xs[1], xs[0])
    if no_root:
        v = sgn if p == 1 else (2 * diff if p == 2 else p * a ** (p - 1) * sgn)
    else:
        with np.errstate(divide="ignore", invalid="ignore"):
            if p == 1:
                v = sgn
            elif p == 2:
                v = diff / y
            else:
                v = a ** (p - 1) * sgn / y ** (p - 1)
        v = np.where(y == 0, 0.0, v)
    grad = (g * v).ravel()
    return grad, -grad


def _label(v, what):
    r = np.rint(v)
    if r != v:
        raise DataError(f"{what} label is not an integer")
    return int(r)


# loss.cpp:86-228
def loss_forward(x, xs, labels, cs, weights=None, kind="softmaxlog", top_k=5, threshold=0.0):
    kind = KINDS[kind] if isinstance(kind, int) else kind
    X = np.asarray(x, np.float64)
    L = np.asarray(labels, np.float64)
    Wt = None if weights is None else np.asarray(weights, np.float64)
    total = 0.0
    if kind in ("binaryerror", "binarylog", "logistic", "hinge"):
        for k in range(X.size):
            c = _label(L[k], "attribute")
            if c == 0:
                continue
            if c not in (1, -1):
                raise DataError("attribute label must be -1, 0 or +1")
            w = 1.0 if Wt is None else Wt[k]
            v = X[k]
            if kind == "binaryerror":
                l = 0.0 if (1 if v - threshold >= 0 else -1) == c else 1.0
            elif kind == "binarylog":
                if v < 0 or v > 1:
                    raise DataError("binary log loss input must lie in [0,1]")
                l = -np.log(c * (v - 0.5) + 0.5)
            elif kind == "logistic":
                l = np.logaddexp(0.0, -c * v)
            else:
                l = max(0.0, 1 - c * v)
            total += w * l
        return total
    H, W, C, N = xs
    V = X.reshape(N, C, W, H)
    for n in range(N):
        for j in range(W):
            for i in range(H):
                s = i + H * (j + W * n)
                c = _label(L[s], "class")
                if c == 0:
                    continue
                if c < 1 or c > C:
                    raise DataError(f"class label {c} out of range 1..{C}")
                col = V[n, :, j, i]
                xc = col[c - 1]
                if kind == "classerror":
                    l = 0.0 if int(np.argmax(col)) == c - 1 else 1.0
                elif kind == "topk":
                    l = 0.0 if int((col >= xc).sum()) <= top_k else 1.0
                elif kind == "log":
                    if not xc > 0:
                        raise DataError("log loss needs a positive ground-truth score")
                    l = -np.log(xc)
                elif kind == "softmaxlog":
                    m = col.max()
                    l = -xc + m + np.log(np.exp(col - m).sum())
                elif kind == "mhinge":
                    l = max(0.0, 1 - xc)
                elif kind == "mshinge":
                    other = np.delete(col, c - 1).max() if C > 1 else 0.0
                    l = max(0.0, 1 - xc + other)
                total += (1.0 if Wt is None else Wt[s]) * l
    return total


# loss.cpp:231-343
def loss_backward(x, xs, labels, cs, weights=None, kind="softmaxlog", p=1.0):
    kind = KINDS[kind] if isinstance(kind, int) else kind
    X = np.asarray(x, np.float64)
    L = np.asarray(labels, np.float64)
    Wt = None if weights is None else np.asarray(weights, np.float64)
    dx = np.zeros_like(X)
    if kind in ("classerror", "topk", "binaryerror"):
        return dx
    if kind in ("binarylog", "logistic", "hinge"):
        for k in range(X.size):
            c = _label(L[k], "attribute")
            if c == 0:
                continue
            if c not in (1, -1):
                raise DataError("attribute label must be -1, 0 or +1")
            sc = p * (1.0 if Wt is None else Wt[k])
            v = X[k]
            if kind == "binarylog":
                if v < 0 or v > 1:
                    raise DataError("binary log loss input must lie in [0,1]")
                dx[k] = -sc * c / (c * (v - 0.5) + 0.5)
            elif kind == "logistic":
                dx[k] = -sc * c / (1 + np.exp(c * v))
            elif c * v < 1:
                dx[k] = -sc * c
        return dx
    H, W, C, N = xs
    V = X.reshape(N, C, W, H)
    Dv = dx.reshape(N, C, W, H)
    for n in range(N):
        for j in range(W):
            for i in range(H):
                s = i + H * (j + W * n)
                c = _label(L[s], "class")
                if c == 0:
                    continue
                if c < 1 or c > C:
                    raise DataError(f"class label {c} out of range 1..{C}")
                sc = p * (1.0 if Wt is None else Wt[s])
                col = V[n, :, j, i]
                xc = col[c - 1]
                if kind == "log":
                    if not xc > 0:
                        raise DataError("log loss needs a positive ground-truth score")
                    Dv[n, c - 1, j, i] -= sc / xc
                elif kind == "softmaxlog":
                    e = np.exp(col - col.max())
                    soft = e / e.sum()
                    soft[c - 1] -= 1
                    Dv[n, :, j, i] += sc * soft
                elif kind == "mhinge":
                    if xc < 1:
                        Dv[n, c - 1, j, i] -= sc
                elif kind == "mshinge":
                    others = [k for k in range(C) if k != c - 1]
                    if others:
                        best = others[int(np.argmax(col[others]))]
                        if xc < 1 + col[best]:
                            Dv[n, c - 1, j, i] -= sc
                            Dv[n, best, j, i] += sc
    return dx
