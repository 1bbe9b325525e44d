"""Pin the C restatement against the reference itself: the convkit sources
compiled verbatim into oracle/_ref (oracle/Makefile).  CPU only; skipped on
machines where the reference was never built."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b) / np.maximum(np.abs(a) + np.abs(b), 1e-2 * np.sqrt(np.mean(b * b)) + 1e-30))


CONV_CASES = [
    # xs, fs, geom (sh, sw, pt, pb, pl, pr, g)
    ((7, 6, 4, 3), (3, 2, 2, 6), (2, 1, 0, 1, 1, 0, 2)),
    ((9, 9, 3, 2), (3, 3, 3, 4), (1, 1, 1, 1, 1, 1, 1)),
    ((11, 10, 2, 2), (5, 4, 2, 3), (3, 2, 2, 0, 1, 3, 1)),
    ((8, 8, 6, 2), (1, 1, 2, 6), (1, 1, 0, 0, 0, 0, 3)),
    ((27, 27, 8, 1), (5, 5, 4, 8), (1, 1, 2, 2, 2, 2, 2)),      # conv2-like
    ((23, 23, 3, 1), (11, 11, 3, 4), (4, 4, 0, 0, 0, 0, 1)),    # conv1-like
    ((6, 6, 4, 3), (6, 6, 4, 5), (1, 1, 0, 0, 0, 0, 1)),        # fc
]


@pytest.mark.parametrize("xs,fs,g", CONV_CASES)
def test_conv_vs_reference(xs, fs, g):
    r = O.Rng(hash((xs, fs)) % 1000)
    x, f, b = r.uniform(O.size(xs)), r.uniform(O.size(fs)), r.uniform(fs[3])
    y, ys = O.conv_forward(x, xs, f, fs, b, g)
    yr, _ = O.ref_conv_forward(x, xs, f, fs, b, g)
    assert rel(yr, y) < 1e-4  # fp32 reference GEMM vs the double restatement
    dy = r.uniform(O.size(ys))
    for a, c in zip(O.conv_backward(x, xs, f, fs, g, dy), O.ref_conv_backward(x, xs, f, fs, g, dy)):
        assert rel(c, a) < 1e-4


def test_convt_vs_reference():
    r = O.Rng(21)
    xs, fs, cg = (4, 3, 3, 2), (3, 2, 3, 4), (2, 1, 1, 0, 0, 1)
    x, f = r.uniform(O.size(xs)), r.uniform(O.size(fs))
    y, ys = O.convt_forward(x, xs, f, fs, cg)
    yr, _ = O.ref_convt_forward(x, xs, f, fs, cg)
    assert rel(yr, y) < 1e-5
    dy = r.uniform(O.size(ys))
    for a, c in zip(O.convt_backward(x, xs, f, fs, cg, dy), O.ref_convt_backward(x, xs, f, fs, cg, dy)):
        assert rel(c, a) < 1e-5


POOLS = [(3, 3, 2, 2, 0, 1, 0, 1, 0), (3, 3, 2, 2, 0, 1, 0, 1, 1), (2, 2, 2, 2, 0, 0, 0, 0, 0),
         (3, 2, 1, 2, 2, 1, 1, 0, 1), (4, 4, 3, 3, 3, 0, 0, 3, 0)]


@pytest.mark.parametrize("pg", POOLS)
def test_pool_bitexact_vs_reference(pg):
    r = O.Rng(22)
    xs = (13, 11, 3, 2)
    x = r.uniform(O.size(xs))
    x[::7] = x[1::7][: len(x[::7])]  # manufacture ties
    y, ys = O.pool_forward(x, xs, pg)
    yr, _ = O.ref_pool_forward(x, xs, pg)
    assert np.array_equal(y, yr)
    dy = r.uniform(O.size(ys))
    assert np.array_equal(O.pool_backward(x, xs, pg, dy), O.ref_pool_backward(x, xs, pg, dy))


def test_relu_bitexact_vs_reference():
    r = O.Rng(23)
    x = r.uniform(1000)
    x[::10] = 0
    dy = r.uniform(1000)
    assert np.array_equal(O.relu_forward(x), O.ref_relu(x))
    assert np.array_equal(O.relu_backward(x, dy), O.ref_relu(x, dy))


@pytest.mark.parametrize("n,k,a,b", [(5, 1.0, 2e-5, 0.75), (3, 2.0, 1e-1, 0.5), (4, 1.0, 0.5, 0.75)])
def test_lrn_vs_reference(n, k, a, b):
    r = O.Rng(24)
    xs = (5, 4, 9, 2)
    x, dy = r.uniform(O.size(xs)), r.uniform(O.size(xs))
    assert rel(O.ref_lrn_forward(x, xs, n, k, a, b), O.lrn_forward(x, xs, n, k, a, b)) < 1e-6
    assert rel(O.ref_lrn_backward(x, xs, n, k, a, b, dy), O.lrn_backward(x, xs, n, k, a, b, dy)) < 1e-5


def test_bnorm_vs_reference():
    r = O.Rng(25)
    xs = (6, 5, 4, 3)
    x, dy = r.uniform(O.size(xs)), r.uniform(O.size(xs))
    w, b = r.uniform(4), r.uniform(4)
    y, m, v = O.bnorm_forward(x, xs, w, b, 1e-5)
    yr, mr, vr = O.ref_bnorm_forward(x, xs, w, b, 1e-5)
    assert rel(yr, y) < 1e-5 and rel(mr, m) < 1e-5 and rel(vr, v) < 1e-5
    for a, c in zip(O.bnorm_backward(x, xs, w, b, 1e-5, dy), O.ref_bnorm_backward(x, xs, w, b, 1e-5, dy)):
        assert rel(c, a) < 1e-4


def test_loss_vs_reference():
    r = O.Rng(26)
    xs, cs = (2, 3, 17, 4), (2, 3, 1, 4)
    x = r.uniform(O.size(xs)) * 5
    c = r.labels(O.size(cs), 17)
    c[3] = 0
    w = r.uniform(O.size(cs), 0, 2)
    for kind in ("softmaxlog", "classerror", "topk"):
        a = O.loss_forward(x, xs, c, cs, w, kind=kind, top_k=5)
        b = O.ref_loss_forward(x, xs, c, cs, w, kind=kind, top_k=5)
        assert abs(a - b) <= 1e-5 * max(1, abs(a))
    dx = O.softmaxlog_backward(x, xs, c, cs, w, 0.7)
    assert rel(O.ref_loss_backward(x, xs, c, cs, w, p=0.7), dx) < 1e-5
    with pytest.raises(O.OracleError) as e:
        O.ref_loss_forward(x, xs, c + 0.5, cs)
    assert e.value.code == 2


def test_rng_matches_reference_stream():
    """oracle Rng == libck host Rng (both restate rng.cpp)."""
    from paper_1412_4564_b200.nets import Rng as R2
    a, b = O.Rng(77), R2(77)
    assert np.array_equal(a.uniform(1000), b.uniform(1000))
    assert np.array_equal(a.normal(1001, 0.01), b.normal(1001, 0.01))
    assert np.array_equal(a.labels(999, 1000), b.labels(999, 1000))


def test_lenet_graph_vs_reference_engine():
    """The reference DAG engine (graph.cpp:494/548) vs the oracle chain."""
    import chain
    from paper_1412_4564_b200.nets import lenet
    net = lenet(batch=3)
    params, inputs = net.init_params(), net.init_inputs()
    rg = O.RefGraph()
    net.build(type("B", (), {
        "add_input": lambda s, n, sh: rg.add_input(n),
        "add_param": lambda s, n, sh: rg.add_param(n),
        "add_layer": lambda s, *a: rg.add_layer(*a)})())
    rg.finalize()
    for k, v in {**params, **inputs}.items():
        sh = dict(net.inputs).get(k) or next(s for n, s, _ in net.params if n == k)
        rg.bind(k, v, sh)
    rg.run()
    vals, derivs = chain.run(net, params, inputs)
    loss, _ = rg.get("objective")
    assert abs(loss[0] - vals["objective"][0]) < 1e-5 * abs(loss[0])
    for name, _, _ in net.params:
        d, _ = rg.get(name, deriv=True)
        assert rel(d, derivs[name]) < 1e-3, name
