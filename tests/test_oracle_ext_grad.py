"""SPEC.md:775-783 gradient suite for the extended block set, on the oracle
restatement (oracle/ext.py) in double precision: for every block, >= 5
random instances with dims <= 6, the backward against central finite
differences of the forward, max relative error < 1e-4 with the reference's
floored measure fd_rel_err (graph.cpp:685-689).  CPU only."""
import numpy as np
import pytest

import ext as E


def fd_rel_err(a, n):
    return np.abs(a - n) / np.maximum(np.abs(a) + np.abs(n), 1e-2)


def check(f, x, grad, h=1e-6, probes=24, seed=0):
    """grad vs central differences of scalar f at x (flat), on sampled coords."""
    rng = np.random.default_rng(seed)
    idx = rng.choice(x.size, size=min(probes, x.size), replace=False)
    worst = 0.0
    for i in idx:
        xp, xm = x.copy(), x.copy()
        step = h * max(1.0, abs(x[i]))
        xp[i] += step
        xm[i] -= step
        num = (f(xp) - f(xm)) / (2 * step)
        worst = max(worst, float(fd_rel_err(grad[i], num)))
    assert worst < 1e-4, worst


def shapes(seed, n=5):
    rng = np.random.default_rng(seed)
    return [tuple(int(v) for v in rng.integers(1, 7, size=4)) for _ in range(n)]


@pytest.mark.parametrize("xs", shapes(1))
def test_sigmoid_grad(xs):
    rng = np.random.default_rng(sum(xs))
    x = rng.uniform(-4, 4, size=int(np.prod(xs)))
    p = rng.uniform(-1, 1, size=x.size)
    y = E.sigmoid_forward(x)
    check(lambda v: float(p @ E.sigmoid_forward(v)), x, E.sigmoid_backward(y, p))


@pytest.mark.parametrize("xs", shapes(2))
def test_softmax_grad(xs):
    rng = np.random.default_rng(sum(xs) + 1)
    x = rng.uniform(-3, 3, size=int(np.prod(xs)))
    p = rng.uniform(-1, 1, size=x.size)
    y = E.softmax_forward(x, xs)
    check(lambda v: float(p @ E.softmax_forward(v, xs)), x, E.softmax_backward(y, xs, p))


@pytest.mark.parametrize("xs", shapes(3))
def test_spnorm_grad(xs):
    rng = np.random.default_rng(sum(xs) + 2)
    x = rng.uniform(-2, 2, size=int(np.prod(xs)))
    p = rng.uniform(-1, 1, size=x.size)
    wh, ww = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    f = lambda v: float(p @ E.spnorm_forward(v, xs, wh, ww, 0.7, 0.6))  # noqa: E731
    check(f, x, E.spnorm_backward(x, xs, wh, ww, 0.7, 0.6, p))


@pytest.mark.parametrize("xs", shapes(4))
def test_bilinear_grad(xs):
    rng = np.random.default_rng(sum(xs) + 3)
    H, W = max(xs[0], 2), max(xs[1], 2)
    xs = (H, W, xs[2], xs[3])
    gs = (2, int(rng.integers(1, 5)), int(rng.integers(1, 5)), xs[3])
    x = rng.uniform(-1, 1, size=int(np.prod(xs)))
    # grid points away from the tent kinks (integer sample positions)
    g = rng.uniform(-0.9, 0.9, size=int(np.prod(gs)))
    ys = (gs[1], gs[2], xs[2], xs[3])
    p = rng.uniform(-1, 1, size=int(np.prod(ys)))
    dx, dg = E.bilinear_backward(x, xs, g, gs, p)
    check(lambda v: float(p @ E.bilinear_forward(v, xs, g, gs)[0]), x, dx)
    check(lambda v: float(p @ E.bilinear_forward(x, xs, v, gs)[0]), g, dg, h=1e-7)


@pytest.mark.parametrize("pp,no_root", [(1.0, False), (2.0, False), (3.0, True), (1.5, False),
                                        (2.0, True)])
def test_pdist_grad(pp, no_root):
    xs = (3, 2, 4, 2)
    rng = np.random.default_rng(int(pp * 10) + no_root)
    x, t = rng.uniform(-1, 1, size=48), rng.uniform(-1, 1, size=48)
    p = rng.uniform(-1, 1, size=3 * 2 * 2)
    dx, dt = E.pdist_backward(x, t, xs, pp, no_root, p)
    check(lambda v: float(p @ E.pdist_forward(v, t, xs, pp, no_root)), x, dx)
    check(lambda v: float(p @ E.pdist_forward(x, v, xs, pp, no_root)), t, dt)


@pytest.mark.parametrize("kind", ["log", "softmaxlog", "mhinge", "mshinge", "binarylog",
                                  "logistic", "hinge"])
def test_loss_grad(kind):
    rng = np.random.default_rng(len(kind))
    attr = kind in ("binarylog", "logistic", "hinge")
    xs = (2, 3, 5, 2)
    if attr:
        cs = xs
        lab = rng.integers(-1, 2, size=int(np.prod(cs))).astype(float)
        x = rng.uniform(0.1, 0.9, size=int(np.prod(xs))) if kind == "binarylog" else \
            rng.uniform(-2, 2, size=int(np.prod(xs)))
    else:
        cs = (2, 3, 1, 2)
        lab = rng.integers(0, 6, size=int(np.prod(cs))).astype(float)
        x = rng.uniform(0.1, 1.0, size=int(np.prod(xs))) if kind == "log" else \
            rng.uniform(-2, 2, size=int(np.prod(xs)))
    w = rng.uniform(0.5, 2, size=int(np.prod(cs)))
    g = E.loss_backward(x, xs, lab, cs, w, kind, p=0.8)
    check(lambda v: 0.8 * E.loss_forward(v, xs, lab, cs, w, kind), x, g)
