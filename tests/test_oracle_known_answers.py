"""Pin the CPU oracle (oracle/ck_oracle.c) to the reference's known-answer
examples and to central finite differences (the reference's own
oracles.hpp:35-68 / grad_check, graph.cpp:685-743).  CPU only."""
import numpy as np
import pytest

import oracle as O


def fd_rel_err(a, b):  # graph.cpp:685-689
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b) / np.maximum(np.abs(a) + np.abs(b), 1e-2))


def fd_projected(fwd, x, p, step=1e-6):  # oracles.hpp:35-50
    x = np.array(x, np.float64)
    g = np.zeros_like(x)
    for e in range(x.size):
        s = x[e]
        h = step * max(1.0, abs(s))
        x[e] = s + h
        up = np.dot(p, fwd(x))
        x[e] = s - h
        dn = np.dot(p, fwd(x))
        x[e] = s
        g[e] = (up - dn) / (2 * h)
    return g


G0 = (1, 1, 0, 0, 0, 0, 1)


# ---- conv ----------------------------------------------------

def test_conv_simple_1d():
    y, ys = O.conv_forward([1, 2, 3], (3, 1, 1, 1), [1, 1], (2, 1, 1, 1), None, G0)
    assert ys == (2, 1, 1, 1) and list(y) == [3, 5]


def test_conv_identity_bank():
    r = O.Rng(3)
    xs = (4, 3, 5, 2)
    x = r.uniform(O.size(xs))
    f = np.eye(5).reshape(-1)  # f[0,0,d,k] = [d == k]
    y, ys = O.conv_forward(x, xs, f, (1, 1, 5, 5), None, G0)
    assert ys == xs and np.array_equal(y, x.astype(np.float64))


def test_conv_fully_connected_is_matmul():
    r = O.Rng(4)
    xs, fs = (3, 3, 2, 4), (3, 3, 2, 5)
    x, f, b = r.uniform(O.size(xs)), r.uniform(O.size(fs)), r.uniform(5)
    y, ys = O.conv_forward(x, xs, f, fs, b, G0)
    X = x.reshape(4, 18).astype(np.float64)
    F = f.reshape(5, 18).astype(np.float64)
    assert ys == (1, 1, 5, 4)
    np.testing.assert_allclose(y.reshape(4, 5), X @ F.T + b, rtol=1e-12, atol=1e-12)


def test_im2row_examples():
    A, rows, cols = O.im2row([1, 2, 3], (3, 1, 1, 1), 2, 1, G0)
    assert (rows, cols) == (2, 2)
    assert A.reshape(cols, rows).T.tolist() == [[1, 2], [2, 3]]
    A, rows, cols = O.im2row([1, 2], (2, 1, 1, 1), 2, 1, (1, 1, 1, 1, 0, 0, 1))
    assert A.reshape(cols, rows).T.tolist() == [[0, 1], [1, 2], [2, 0]]


def test_row2im_overlap_and_adjoint():
    x = O.row2im(np.ones(4), (3, 1, 1, 1), 2, 1, G0)
    assert x.tolist() == [1, 2, 1]
    r = O.Rng(5)
    xs, g = (5, 4, 2, 1), (2, 1, 1, 0, 0, 1, 1)
    x = r.uniform(O.size(xs)).astype(np.float64)
    A, rows, cols = O.im2row(x, xs, 3, 2, g)
    M = r.uniform(rows * cols).astype(np.float64)
    assert abs(np.dot(A, M) - np.dot(x, O.row2im(M, xs, 3, 2, g))) < 1e-12


def test_output_size_law():
    for H in range(1, 9):
        for Hf in range(1, 5):
            for S in range(1, 4):
                for pl in range(0, 3):
                    for ph in range(0, 3):
                        if H + pl + ph < Hf:
                            with pytest.raises(O.OracleError):
                                O.conv_output_shape((H, 1, 1, 1), (Hf, 1, 1, 1), (S, 1, pl, ph, 0, 0, 1))
                            continue
                        count = len(range(-pl, H + ph - Hf + 1, S))
                        assert O.conv_output_shape((H, 1, 1, 1), (Hf, 1, 1, 1),
                                                   (S, 1, pl, ph, 0, 0, 1))[0] == count


def test_conv_shape_errors():
    with pytest.raises(O.OracleError):
        O.conv_output_shape((5, 5, 4, 1), (3, 3, 3, 6), (1, 1, 0, 0, 0, 0, 1))  # channels
    with pytest.raises(O.OracleError):
        O.conv_output_shape((5, 5, 4, 1), (3, 3, 2, 5), (1, 1, 0, 0, 0, 0, 2))  # K % g
    with pytest.raises(O.OracleError):
        O.conv_output_shape((5, 5, 4, 1), (3, 3, 4, 5), (0, 1, 0, 0, 0, 0, 1))  # stride


def test_conv_backward_scalar():
    dx, df, db = O.conv_backward([2.0], (1, 1, 1, 1), [3.0], (1, 1, 1, 1), G0, [5.0])
    assert dx.tolist() == [15.0] and df.tolist() == [10.0] and db.tolist() == [5.0]


def test_conv_backward_fd():  # SPEC.md:152 (5x5x2, 3x3x2x3, S=2, pads 0,1,0,1)
    r = O.Rng(6)
    xs, fs, g = (5, 5, 2, 1), (3, 3, 2, 3), (2, 2, 0, 1, 0, 1, 1)
    x, f, b = (r.uniform(O.size(xs)).astype(np.float64), r.uniform(O.size(fs)).astype(np.float64),
               r.uniform(3).astype(np.float64))
    y, ys = O.conv_forward(x, xs, f, fs, b, g)
    p = r.uniform(O.size(ys)).astype(np.float64)
    dx, df, db = O.conv_backward(x, xs, f, fs, g, p)
    assert fd_rel_err(dx, fd_projected(lambda v: O.conv_forward(v, xs, f, fs, b, g)[0], x, p)) < 1e-6
    assert fd_rel_err(df, fd_projected(lambda v: O.conv_forward(x, xs, v, fs, b, g)[0], f, p)) < 1e-6
    assert fd_rel_err(db, fd_projected(lambda v: O.conv_forward(x, xs, f, fs, v, g)[0], b, p)) < 1e-6


def test_conv_groups_block_diagonal():
    r = O.Rng(7)
    xs, fs, g = (4, 4, 4, 1), (3, 3, 2, 6), (1, 1, 1, 1, 1, 1, 2)
    x = r.uniform(O.size(xs)).astype(np.float64)
    x[16 * 2:] = 0  # zero the second group's channels
    f = r.uniform(O.size(fs))
    y, ys = O.conv_forward(x, xs, f, fs, None, g)
    assert np.all(y.reshape(6, 16)[3:] == 0.0)


# ---- convt ----------------------------------------------------

def test_convt_example():
    y, ys = O.convt_forward([1, 1], (2, 1, 1, 1), [1, 2, 3], (3, 1, 1, 1), (2, 1, 0, 0, 0, 0))
    assert ys == (5, 1, 1, 1) and y.tolist() == [1, 2, 4, 2, 3]


def test_convt_duality():
    r = O.Rng(8)
    for trial in range(10):
        up = 1 + trial % 3
        xs, fs = (3, 4, 2, 2), (3, 2, 3, 2)  # conv: C=3 -> K=2; convt maps 2 -> 3
        cg = (up, 1, trial % 2, 0, 0, trial % 2)
        g = (up, 1, cg[2], cg[3], cg[4], cg[5], 1)
        ys = O.convt_output_shape(xs, (fs[0], fs[1], fs[3], fs[2]), cg)
        # conv maps ys-space (3 channels) to xs-space (2 channels) with f
        y = r.uniform(O.size(ys)).astype(np.float64)
        x = r.uniform(O.size(xs)).astype(np.float64)
        f = r.uniform(O.size(fs)).astype(np.float64)
        cx, cxs = O.conv_forward(y, ys, f, fs, None, g)
        assert cxs == xs
        # convt filter bank: (fh, fw, D=2, K=3) with ft[i,j,d,k] = f[i,j,k,d]
        ft = f.reshape(2, 3, 2, 3).transpose(1, 0, 2, 3).reshape(-1)
        ty, tys = O.convt_forward(x, xs, ft, (fs[0], fs[1], 2, 3), cg)
        assert tys == ys
        assert abs(np.dot(x, cx) - np.dot(ty, y)) < 1e-10 * max(1, abs(np.dot(x, cx)))


def test_convt_backward_fd():
    r = O.Rng(9)
    xs, fs, cg = (3, 2, 2, 1), (3, 2, 2, 3), (2, 1, 1, 0, 0, 1)
    x = r.uniform(O.size(xs)).astype(np.float64)
    f = r.uniform(O.size(fs)).astype(np.float64)
    y, ys = O.convt_forward(x, xs, f, fs, cg)
    p = r.uniform(O.size(ys)).astype(np.float64)
    dx, df = O.convt_backward(x, xs, f, fs, cg, p)
    assert fd_rel_err(dx, fd_projected(lambda v: O.convt_forward(v, xs, f, fs, cg)[0], x, p)) < 1e-6
    assert fd_rel_err(df, fd_projected(lambda v: O.convt_forward(x, xs, v, fs, cg)[0], f, p)) < 1e-6


# ---- pool -----------------------------------------------------------

def test_pool_examples():
    y, _ = O.pool_forward([1, 3, 2], (3, 1, 1, 1), (2, 1, 1, 1, 0, 0, 0, 0, 0))
    assert y.tolist() == [3, 3]
    y, _ = O.pool_forward([4], (1, 1, 1, 1), (2, 1, 1, 1, 0, 1, 0, 0, 1))
    assert y.tolist() == [4]  # cropped area
    y, _ = O.pool_forward(np.full(20, 2.5), (5, 4, 1, 1), (3, 2, 2, 1, 1, 1, 0, 1, 1))
    assert np.all(y == 2.5)


def test_pool_routing_and_ties():
    dx = O.pool_backward([1, 2, 3, 4], (4, 1, 1, 1), (2, 1, 1, 1, 0, 0, 0, 0, 0), [1, 1, 1])
    assert dx.tolist() == [0, 1, 1, 1]  # increasing input -> last element of each window
    dx = O.pool_backward([5, 5], (2, 1, 1, 1), (2, 1, 1, 1, 0, 0, 0, 0, 0), [1])
    assert dx.tolist() == [1, 0]  # first index wins ties


def test_pool_mass_and_shift():
    r = O.Rng(10)
    xs, pg = (9, 7, 3, 2), (3, 3, 2, 2, 1, 1, 0, 1, 0)
    x = r.uniform(O.size(xs))
    y, ys = O.pool_forward(x, xs, pg)
    y2, _ = O.pool_forward(x + np.float32(0.5), xs, pg)
    np.testing.assert_allclose(y2, y + 0.5, rtol=0, atol=1e-6)
    dy = r.uniform(O.size(ys))
    dx = O.pool_backward(x, xs, pg, dy)
    assert abs(dx.sum(dtype=np.float64) - dy.sum(dtype=np.float64)) < 1e-4


def test_pool_output_sweep():
    for H in range(1, 9):
        for w in range(1, 5):
            for S in range(1, 4):
                for pl in range(0, w):
                    for ph in range(0, w):
                        if H + pl + ph < w:
                            continue
                        got = O.pool_output_shape((H, 1, 1, 1), (w, 1, S, 1, pl, ph, 0, 0, 0))[0]
                        assert got == len(range(-pl, H + ph - w + 1, S))


# ---- relu / lrn / bnorm --------------------------------------------

def test_relu():
    assert O.relu_forward([-1, 2, 0]).tolist() == [0, 2, 0]
    assert O.relu_backward([-1, 2, 0], [5, 6, 7]).tolist() == [0, 6, 0]


def test_lrn_identity_and_scalar():
    r = O.Rng(11)
    xs = (3, 3, 7, 2)
    x = r.uniform(O.size(xs)).astype(np.float64)
    assert np.array_equal(O.lrn_forward(x, xs, 5, 1.0, 0.0, 0.75), x)
    y = O.lrn_forward([1.0], (1, 1, 1, 1), 1, 1.0, 1.0, 0.5)
    assert abs(y[0] - 1 / np.sqrt(2)) < 1e-15


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_lrn_backward_fd(n):
    r = O.Rng(12 + n)
    xs = (3, 3, 5, 1)
    x = r.uniform(O.size(xs)).astype(np.float64)
    p = r.uniform(O.size(xs)).astype(np.float64)
    dx = O.lrn_backward(x, xs, n, 2.0, 0.3, 0.75, p)
    fd = fd_projected(lambda v: O.lrn_forward(v, xs, n, 2.0, 0.3, 0.75), x, p)
    assert fd_rel_err(dx, fd) < 1e-6


def test_bnorm_examples():
    y, m, v = O.bnorm_forward(np.full(8, 3.0), (2, 2, 1, 2), [2.0], [0.7], 1e-5)
    assert np.all(y == 0.7)
    y, m, v = O.bnorm_forward([0.0, 2.0], (2, 1, 1, 1), [1.0], [0.0], 1e-5)
    assert m[0] == 1.0 and v[0] == 1.0
    np.testing.assert_allclose(y, [-1 / np.sqrt(1 + 1e-5), 1 / np.sqrt(1 + 1e-5)])


def test_bnorm_backward_fd():
    r = O.Rng(13)
    xs = (2, 2, 2, 3)
    x = r.uniform(O.size(xs)).astype(np.float64)
    w = r.uniform(2).astype(np.float64)
    b = r.uniform(2).astype(np.float64)
    p = r.uniform(O.size(xs)).astype(np.float64)
    dx, dw, db = O.bnorm_backward(x, xs, w, b, 1e-5, p)
    f = lambda v: O.bnorm_forward(v, xs, w, b, 1e-5)[0]
    assert fd_rel_err(dx, fd_projected(f, x, p)) < 1e-5
    assert fd_rel_err(dw, fd_projected(lambda v: O.bnorm_forward(x, xs, v, b, 1e-5)[0], w, p)) < 1e-5
    assert fd_rel_err(db, fd_projected(lambda v: O.bnorm_forward(x, xs, w, v, 1e-5)[0], b, p)) < 1e-5


# ---- softmaxlog ---------------------------------------------

def test_softmaxlog_examples():
    xs, cs = (1, 1, 2, 1), (1, 1, 1, 1)
    assert abs(O.loss_forward([0, 0], xs, [1], cs) - np.log(2)) < 1e-15
    assert O.softmaxlog_backward([0, 0], xs, [1], cs).tolist() == [-0.5, 0.5]
    # stability at +-1000
    l = O.loss_forward([1000, -1000], xs, [2], cs)
    assert np.isfinite(l) and abs(l - 2000) < 1e-9
    # ignore label and instance weights
    xs2, cs2 = (1, 1, 3, 2), (1, 1, 1, 2)
    x = [0.1, 0.5, -0.2, 0.3, 0.0, 0.9]
    l1 = O.loss_forward(x, xs2, [2, 0], cs2)
    l0 = O.loss_forward(x[:3], (1, 1, 3, 1), [2], (1, 1, 1, 1))
    assert l1 == l0
    assert abs(O.loss_forward(x, xs2, [2, 3], cs2, weights=[2, 2]) -
               2 * O.loss_forward(x, xs2, [2, 3], cs2)) < 1e-15
    dx = O.softmaxlog_backward(x, xs2, [2, 0], cs2)
    assert np.all(dx[3:] == 0)


def test_label_errors():
    xs, cs = (1, 1, 3, 1), (1, 1, 1, 1)
    with pytest.raises(O.OracleError) as e:
        O.loss_forward([0, 0, 0], xs, [1.5], cs)
    assert e.value.code == 2
    with pytest.raises(O.OracleError) as e:
        O.loss_forward([0, 0, 0], xs, [4], cs)
    assert e.value.code == 2


def test_metrics():  # SPEC.md:420 classerror example
    xs, cs = (1, 1, 3, 1), (1, 1, 1, 1)
    x = [0.2, 0.7, 0.1]
    assert O.loss_forward(x, xs, [2], cs, kind="classerror") == 0
    assert O.loss_forward(x, xs, [1], cs, kind="classerror") == 1
    assert O.loss_forward(x, xs, [3], cs, kind="topk", top_k=2) == 1
    assert O.loss_forward(x, xs, [1], cs, kind="topk", top_k=2) == 0


def test_sgd():
    w, v = O.sgd_step([1.0, 2.0], [0.5, -0.5], [0.1, 0.2], 0.1, 0.9, 0.01)
    v_ref = np.float32(0.9) * np.float32([0.5, -0.5]) - np.float32(0.1) * (
        np.float32([0.1, 0.2]) + np.float32(0.01) * np.float32([1.0, 2.0]))
    np.testing.assert_array_equal(v, v_ref.astype(np.float32))
    np.testing.assert_array_equal(w, (np.float32([1.0, 2.0]) + v).astype(np.float32))
