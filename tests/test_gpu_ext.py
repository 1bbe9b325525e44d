"""The rest of the reference block set on the GPU (blocks_ext.cu through the
C ABI) against the oracle restatement (oracle/ext.py, float64) and, where
the kernel follows the reference's float operation order, bit for bit
against the reference itself (oracle/_ref)."""
import numpy as np
import pytest
import torch

import ext as E
import oracle as O

pytestmark = pytest.mark.gpu

B = None


@pytest.fixture(scope="module", autouse=True)
def blocks():
    global B
    from paper_1412_4564_b200 import blocks as _B
    B = _B
    yield


def dev(a, shape):
    return B.as_hwcn(torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda(), shape)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().ravel()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = 1e-2 * np.max(np.abs(b)) + 1e-30
    elem = float(np.max(np.abs(a - b) / np.maximum(np.abs(a) + np.abs(b), floor)))
    norm = float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
    return max(elem, 10 * norm)


def test_sigmoid():
    xs = (17, 9, 5, 3)
    r = O.Rng(21)
    x = r.uniform(O.size(xs), -40, 40)
    y = B.sigmoid_forward(dev(x, xs))
    assert rel(host(y), E.sigmoid_forward(x)) < 1e-6
    dy = r.uniform(O.size(xs))
    # backward: the reference's float expression in its order -> bit-exact
    yh = host(y)
    dx = B.sigmoid_backward(dev(yh, xs), dev(dy, xs))
    assert np.array_equal(host(dx), O.ref_sigmoid(None, dy=dy, y=yh))


@pytest.mark.parametrize("xs", [(13, 11, 7, 2), (1, 1, 1000, 5), (3, 2, 40, 4)])
def test_softmax(xs):
    """Thread-per-site (H*W >= 32) and warp-per-site (fc-shaped) kernels."""
    r = O.Rng(22)
    x = r.uniform(O.size(xs), -8, 8)
    y = host(B.softmax_forward(dev(x, xs)))
    assert rel(y, E.softmax_forward(x, xs)) < 1e-5
    dy = r.uniform(O.size(xs))
    dx = host(B.softmax_backward(dev(y, xs), dev(dy, xs)))
    assert rel(dx, E.softmax_backward(y, xs, dy)) < 1e-4


@pytest.mark.parametrize("win", [(1, 1), (3, 3), (5, 2), (4, 4)])
def test_spnorm(win):
    xs = (19, 14, 3, 2)
    r = O.Rng(23)
    x = r.uniform(O.size(xs), -2, 2)
    p = B.SpnormParams(win[0], win[1], 0.6, 0.75)
    y = host(B.spnorm_forward(dev(x, xs), p))
    assert rel(y, E.spnorm_forward(x, xs, *win, 0.6, 0.75)) < 1e-5
    dy = r.uniform(O.size(xs))
    dx = host(B.spnorm_backward(dev(x, xs), p, dev(dy, xs)))
    assert rel(dx, E.spnorm_backward(x, xs, *win, 0.6, 0.75, dy)) < 1e-4


def test_spnorm_window_error():
    with pytest.raises(B.ShapeError, match="spnorm window must be positive"):
        B.spnorm_forward(dev(np.zeros(8), (2, 2, 2, 1)), B.SpnormParams(0, 1))


@pytest.mark.parametrize("xs,gs", [((9, 7, 4, 2), (2, 6, 5, 2)), ((32, 30, 3, 1), (2, 64, 60, 1))])
def test_bilinear(xs, gs):
    r = O.Rng(24)
    x = r.uniform(O.size(xs))
    g = r.uniform(O.size(gs), -1.1, 1.1)
    y = B.bilinear_forward(dev(x, xs), dev(g, gs))
    ys = B.hwcn_shape(y)
    assert ys == (gs[1], gs[2], xs[2], xs[3])
    # forward: the reference's float expression order -> bit-exact
    assert np.array_equal(host(y), O.ref_bilinear(x, xs, g, gs))
    dy = r.uniform(O.size(ys))
    dx, dg = B.bilinear_backward(dev(x, xs), dev(g, gs), dev(dy, ys))
    rdx, rdg = O.ref_bilinear(x, xs, g, gs, dy=dy)
    assert np.array_equal(host(dg), rdg)      # per-site channel sum, reference order
    assert rel(host(dx), rdx) < 1e-5           # scatter (atomic) order differs
    # vs the double restatement: the reference's own float rounding of the
    # channel sums (cancellation) is ~1e-4 of the largest element
    edx, edg = E.bilinear_backward(x, xs, g, gs, dy)
    assert rel(host(dx), edx) < 1e-4 and rel(host(dg), edg) < 1e-3


def test_bilinear_grid_errors():
    x = dev(np.zeros(2 * 2 * 1 * 2), (2, 2, 1, 2))
    with pytest.raises(B.ShapeError, match="two coordinate channels"):
        B.bilinear_forward(x, dev(np.zeros(3 * 2 * 2 * 2), (3, 2, 2, 2)))
    with pytest.raises(B.ShapeError, match="does not match input batch"):
        B.bilinear_forward(x, dev(np.zeros(2 * 2 * 2 * 1), (2, 2, 2, 1)))


@pytest.mark.parametrize("p,no_root", [(1.0, False), (2.0, False), (3.0, False), (2.0, True),
                                       (1.5, True)])
def test_pdist(p, no_root):
    xs = (11, 6, 9, 3)
    r = O.Rng(25)
    x, t = r.uniform(O.size(xs)), r.uniform(O.size(xs))
    t[:9] = x[:9]  # some coincident sites
    y = host(B.pdist_forward(dev(x, xs), dev(t, xs), p, no_root))
    assert rel(y, E.pdist_forward(x, t, xs, p, no_root)) < 1e-5
    dy = r.uniform(xs[0] * xs[1] * xs[3])
    ys = (xs[0], xs[1], 1, xs[3])
    dx, dt = B.pdist_backward(dev(x, xs), dev(t, xs), dev(dy, ys), p, no_root)
    edx, edt = E.pdist_backward(x, t, xs, p, no_root, dy)
    assert rel(host(dx), edx) < 1e-4
    assert np.array_equal(host(dt), -host(dx))


def test_pdist_errors():
    a = dev(np.zeros(8), (2, 2, 2, 1))
    with pytest.raises(B.ShapeError, match="pdist: shapes differ"):
        B.pdist_forward(a, dev(np.zeros(4), (2, 2, 1, 1)))
    with pytest.raises(B.ShapeError, match="pdist exponent must be positive"):
        B.pdist_forward(a, a, p=0.0)


@pytest.mark.parametrize("kind", range(10))
@pytest.mark.parametrize("fc", [False, True])
def test_loss_kinds(kind, fc):
    r = O.Rng(30 + kind)
    if kind >= 6:
        xs = cs = (4, 3, 5, 3) if not fc else (1, 1, 100, 8)
        x = r.uniform(O.size(xs), 0.0, 1.0) if kind == 7 else r.uniform(O.size(xs), -2, 2)
        lab = (np.floor(r.uniform(O.size(cs), 0, 3)) - 1).astype(np.float32)
    else:
        xs = (4, 3, 7, 3) if not fc else (1, 1, 1000, 8)
        cs = (xs[0], xs[1], 1, xs[3])
        x = r.uniform(O.size(xs), 0.05, 1.0) if kind == 2 else r.uniform(O.size(xs), -2, 2)
        lab = r.labels(O.size(cs), xs[2])
        lab[1] = 0
    w = r.uniform(O.size(cs), 0.5, 2.0)
    for wt in (None, w):
        got = float(host(B.loss_kind_forward(dev(x, xs), dev(lab, cs), kind,
                                             None if wt is None else dev(wt, cs), top_k=3))[0])
        want = E.loss_forward(x, xs, lab, cs, wt, kind, top_k=3)
        assert abs(got - want) <= 1e-5 * max(1.0, abs(want)), (got, want)
        dx = host(B.loss_kind_backward(dev(x, xs), dev(lab, cs), kind,
                                       None if wt is None else dev(wt, cs), p=0.7))
        ref = E.loss_backward(x, xs, lab, cs, wt, kind, p=0.7)
        if np.abs(ref).max() == 0:
            assert np.abs(dx).max() == 0
        elif kind == 7:
            # binarylog: q = c (v - 0.5) + 0.5 cancels in float for v near the
            # label's end (the reference computes it in float too): bit-for-bit
            # with the verbatim reference, 1e-3 of the double restatement
            assert rel(dx, O.ref_loss_grad(x, xs, lab, cs, wt, kind, p=0.7)) < 1e-6
            assert rel(dx, ref) < 1e-3
        else:
            assert rel(dx, ref) < 1e-5


def test_loss_random_ties_matches_reference():
    """classerror with random_ties (loss.cpp:116-131): splitmix64 over ties."""
    xs, cs = (1, 1, 6, 64), (1, 1, 1, 64)
    x = np.zeros(O.size(xs), np.float32)  # every site all-tied
    lab = O.Rng(5).labels(O.size(cs), 6)
    for seed in (0, 7, 12345):
        got = float(host(B.loss_kind_forward(dev(x, xs), dev(lab, cs), "classerror",
                                             random_ties=True, tie_seed=seed))[0])
        want = O.ref_loss(x, xs, lab, cs, None, 0, random_ties=1, tie_seed=seed)
        assert got == want


@pytest.mark.parametrize("kind,bad,msg", [
    ("log", 0.0, "log loss needs a positive ground-truth score"),
    ("binarylog", 1.5, r"binary log loss input must lie in \[0,1\]")])
def test_loss_data_errors(kind, bad, msg):
    if kind == "log":
        xs, cs = (1, 1, 3, 1), (1, 1, 1, 1)
        x, lab = np.array([bad, 0.5, 0.5]), np.array([1.0])
    else:
        xs = cs = (1, 1, 2, 1)
        x, lab = np.array([bad, 0.5]), np.array([1.0, -1.0])
    with pytest.raises(B.DataError, match=msg):
        B.loss_kind_forward(dev(x, xs), dev(lab, cs), kind)
    with pytest.raises(B.DataError, match=r"class label 4 out of range 1..3"):
        B.loss_kind_forward(dev(np.zeros(3), (1, 1, 3, 1)), dev(np.array([4.0]), (1, 1, 1, 1)),
                            "mhinge")
    with pytest.raises(B.DataError, match="attribute label must be -1, 0 or \\+1"):
        B.loss_kind_forward(dev(np.zeros(2), (1, 1, 2, 1)), dev(np.array([2.0, 1.0]),
                                                                (1, 1, 2, 1)), "hinge")
