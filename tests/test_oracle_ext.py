"""Pin the numpy restatement of the extended block set (oracle/ext.py) to the
reference compiled verbatim (oracle/_ref): sigmoid, softmax, spnorm,
bilinear, pdist and every loss kind, plus the SPEC.md known answers for
them.  CPU only."""
import numpy as np
import pytest

import ext as E
import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def close(a, b, tol=1e-5):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(np.abs(b).max(), 1e-30)
    assert np.abs(a - b).max() <= tol * scale, np.abs(a - b).max() / scale


def test_sigmoid_matches_reference():
    r = O.Rng(5)
    x = r.uniform(300, -30, 30)
    close(E.sigmoid_forward(x), O.ref_sigmoid(x), 1e-6)
    y = O.ref_sigmoid(x)
    dy = r.uniform(300)
    close(E.sigmoid_backward(y, dy), O.ref_sigmoid(None, dy=dy, y=y), 1e-6)
    # large magnitudes never overflow (activation.cpp:29-36)
    assert E.sigmoid_forward(np.array([1000.0]))[0] == 1.0
    assert E.sigmoid_forward(np.array([-1000.0]))[0] == 0.0


@pytest.mark.parametrize("xs", [(3, 4, 5, 2), (1, 1, 37, 3)])
def test_softmax_matches_reference(xs):
    r = O.Rng(6)
    x = r.uniform(O.size(xs), -5, 5)
    y = O.ref_softmax(x, xs)
    close(E.softmax_forward(x, xs), y, 1e-6)
    dy = r.uniform(O.size(xs))
    close(E.softmax_backward(y, xs, dy), O.ref_softmax(None, xs, dy=dy, y=y), 1e-5)


@pytest.mark.parametrize("win", [(1, 1), (3, 3), (4, 2), (5, 3)])
def test_spnorm_matches_reference(win):
    xs = (7, 6, 3, 2)
    r = O.Rng(7)
    x = r.uniform(O.size(xs), -2, 2)
    close(E.spnorm_forward(x, xs, *win, 0.5, 0.75), O.ref_spnorm(x, xs, *win, 0.5, 0.75), 1e-5)
    dy = r.uniform(O.size(xs))
    close(E.spnorm_backward(x, xs, *win, 0.5, 0.75, dy),
          O.ref_spnorm(x, xs, *win, 0.5, 0.75, dy=dy), 1e-5)


def test_bilinear_matches_reference():
    xs, gs = (6, 5, 3, 2), (2, 4, 7, 2)
    r = O.Rng(8)
    x = r.uniform(O.size(xs))
    g = r.uniform(O.size(gs), -1.2, 1.2)  # some samples outside [-1, 1] fade out
    y, ys = E.bilinear_forward(x, xs, g, gs)
    assert ys == (4, 7, 3, 2)
    close(y, O.ref_bilinear(x, xs, g, gs), 1e-5)
    dy = r.uniform(O.size(ys))
    dx, dg = E.bilinear_backward(x, xs, g, gs, dy)
    rdx, rdg = O.ref_bilinear(x, xs, g, gs, dy=dy)
    close(dx, rdx, 1e-5)
    close(dg, rdg, 1e-5)


def test_bilinear_identity_grid_reproduces_input():
    """bilinear.cpp:135-152 identity_grid: output == input when sizes match."""
    H, W, C, N = 5, 4, 2, 1
    x = O.Rng(9).uniform(H * W * C * N)
    g = np.zeros((N, W, H, 2))
    for j in range(W):
        for i in range(H):
            g[0, j, i] = (-1 + 2 * i / (H - 1), -1 + 2 * j / (W - 1))
    y, _ = E.bilinear_forward(x, (H, W, C, N), g.ravel(), (2, H, W, N))
    close(y, x, 1e-12)


@pytest.mark.parametrize("p,no_root", [(1.0, 0), (2.0, 0), (3.0, 0), (1.0, 1), (2.0, 1), (1.5, 1)])
def test_pdist_matches_reference(p, no_root):
    xs = (3, 4, 5, 2)
    r = O.Rng(10)
    x, t = r.uniform(O.size(xs)), r.uniform(O.size(xs))
    close(E.pdist_forward(x, t, xs, p, no_root), O.ref_pdist(x, t, xs, p, no_root), 1e-5)
    dy = r.uniform(xs[0] * xs[1] * xs[3])
    dx, dt = E.pdist_backward(x, t, xs, p, no_root, dy)
    rdx, rdt = O.ref_pdist(x, t, xs, p, no_root, dy=dy)
    close(dx, rdx, 1e-4)
    close(dt, rdt, 1e-4)


@pytest.mark.parametrize("kind", range(10))
def test_loss_kinds_match_reference(kind):
    r = O.Rng(11 + kind)
    if kind >= 6:  # attribute kinds: labels in {-1, 0, +1}
        xs = cs = (2, 3, 4, 2)
        x = r.uniform(O.size(xs), 0.0, 1.0) if kind == 7 else r.uniform(O.size(xs), -2, 2)
        lab = (np.floor(r.uniform(O.size(cs), 0, 3)) - 1).astype(np.float32)
    else:
        xs, cs = (2, 3, 7, 2), (2, 3, 1, 2)
        x = r.uniform(O.size(xs), 0.05, 1.0) if kind == 2 else r.uniform(O.size(xs), -2, 2)
        lab = r.labels(O.size(cs), 7)
        lab[3] = 0  # an ignored site
    w = r.uniform(O.size(cs), 0.5, 2.0)
    for wt in (None, w):
        want = O.ref_loss(x, xs, lab, cs, wt, kind, top_k=3)
        got = E.loss_forward(x, xs, lab, cs, wt, kind, top_k=3)
        assert abs(got - want) <= 1e-5 * max(1.0, abs(want)), (got, want)
        close(E.loss_backward(x, xs, lab, cs, wt, kind, p=0.7),
              O.ref_loss_grad(x, xs, lab, cs, wt, kind, p=0.7), 1e-5)


def test_loss_known_answers():
    """SPEC.md:418-452 examples for the other kinds."""
    x, xs, cs = np.array([0.2, 0.8]), (1, 1, 2, 1), (1, 1, 1, 1)
    assert E.loss_forward(x, xs, [2.0], cs, kind="log") == pytest.approx(-np.log(0.8))
    assert E.loss_forward(x, xs, [1.0], cs, kind="classerror") == 1.0
    assert E.loss_forward(x, xs, [2.0], cs, kind="classerror") == 0.0
    assert E.loss_forward(x, xs, [1.0], cs, kind="mhinge") == pytest.approx(0.8)
    assert E.loss_forward(x, xs, [1.0], cs, kind="mshinge") == pytest.approx(1.6)
    with pytest.raises(E.DataError):
        E.loss_forward(x, xs, [3.0], cs)
    with pytest.raises(E.DataError):
        E.loss_forward(np.array([1.5]), (1, 1, 1, 1), [1.0], (1, 1, 1, 1), kind="binarylog")
