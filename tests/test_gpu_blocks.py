"""Per-block parity of the CUDA kernels (through the C ABI) against the CPU
oracle on identical seeded inputs.

Tolerances (north star): pooling and ReLU bit-exact; FP32 (CK_MATH_FP32)
outputs and derivatives within 1e-4 relative; TF32 (CK_MATH_TF32) within a
stated 1e-2.  Relative error uses the floored denominator of fd_rel_err
(graph.cpp:685-689): |a-b| / max(|a|+|b|, 1e-2 * rms(ref)).
"""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

B = None


@pytest.fixture(scope="module", autouse=True)
def blocks():
    global B
    assert torch.cuda.is_available()
    from paper_1412_4564_b200 import blocks as _B
    B = _B
    yield


def dev(a, shape):
    return B.as_hwcn(torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda(), shape)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().ravel()


def rel(a, b):
    """Per-element relative error with the denominator floored at 1% of the
    tensor's scale (fd_rel_err's floor, graph.cpp:685-689, made scale-aware):
    near-zero outputs produced by cancellation are judged against the
    tensor's magnitude, not their own.  Also bounds the normwise error."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = 1e-2 * np.max(np.abs(b)) + 1e-30
    elem = float(np.max(np.abs(a - b) / np.maximum(np.abs(a) + np.abs(b), floor)))
    norm = float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
    return max(elem, 10 * norm)


TOL = {"fp32": 1e-4, "tf32": 1e-2}


def err(a, b, math):
    """FP32: the per-element floored metric above.  TF32 (10-bit mantissa
    operands, fp32 accumulate): the stated tolerance is normwise --
    max(||a-b|| / ||b||, max|a-b| / max|b|) -- because an input rounding of
    2^-11 per operand makes cancelled outputs meaningless element by element."""
    if math == "fp32":
        return rel(a, b)
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return max(float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)),
               float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-30)))

CONV_CASES = [
    ((7, 6, 4, 3), (3, 2, 2, 6), (2, 1, 0, 1, 1, 0, 2)),
    ((9, 9, 3, 2), (3, 3, 3, 4), (1, 1, 1, 1, 1, 1, 1)),
    ((11, 10, 2, 2), (5, 4, 2, 3), (3, 2, 2, 0, 1, 3, 1)),
    ((8, 8, 6, 2), (1, 1, 2, 6), (1, 1, 0, 0, 0, 0, 3)),
    ((5, 5, 2, 1), (3, 3, 2, 3), (2, 2, 0, 1, 0, 1, 1)),
    # tensor-core paths at odd sizes: channel padding, asymmetric pad, groups,
    # space-to-depth stride 2
    ((9, 7, 32, 3), (3, 2, 32, 48), (1, 1, 1, 0, 1, 1, 1)),
    ((6, 5, 40, 2), (3, 3, 20, 36), (1, 1, 1, 1, 1, 1, 2)),
    ((23, 21, 5, 2), (5, 5, 5, 24), (2, 2, 0, 0, 0, 0, 1)),
    # AlexNet layer shapes at batch 2
    ((227, 227, 3, 2), (11, 11, 3, 96), (4, 4, 0, 0, 0, 0, 1)),
    ((27, 27, 96, 2), (5, 5, 48, 256), (1, 1, 2, 2, 2, 2, 2)),
    ((13, 13, 256, 2), (3, 3, 256, 384), (1, 1, 1, 1, 1, 1, 1)),
    ((13, 13, 384, 2), (3, 3, 192, 384), (1, 1, 1, 1, 1, 1, 2)),
    ((13, 13, 384, 2), (3, 3, 192, 256), (1, 1, 1, 1, 1, 1, 2)),
    ((6, 6, 256, 4), (6, 6, 256, 512), (1, 1, 0, 0, 0, 0, 1)),
    ((1, 1, 512, 4), (1, 1, 512, 100), (1, 1, 0, 0, 0, 0, 1)),
    # FC with a ragged batch and a non-multiple-of-32 output count (MN-major tails)
    ((2, 2, 64, 3), (2, 2, 64, 40), (1, 1, 0, 0, 0, 0, 1)),
]


def tc_expected(xs, fs, g):
    """The shapes the tcgen05 kernels must take (conv_tc.cu envelope): stride
    1 with pads < the filter extent at any channel count, >= 16 channels and
    filters per group, or the stride-s space-to-depth route (groups 1, no
    padding)."""
    groups = g[6]
    if xs[2] // groups >= 16 and fs[3] // groups >= 16:
        return True
    if g[0] == g[1] == 1 and g[2] <= fs[0] - 1 and g[3] <= fs[0] - 1 and g[4] <= fs[1] - 1 \
            and g[5] <= fs[1] - 1:
        return True  # stride 1, any channel count (padded to 32 per group)
    if g[0] == g[1] >= 2 and groups == 1 and not any(g[2:6]):
        return True
    return False


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("xs,fs,g", CONV_CASES)
def test_conv(xs, fs, g, math):
    r = O.Rng(sum(xs) + sum(fs))
    x = r.uniform(O.size(xs))
    f = r.uniform(O.size(fs), -0.1, 0.1)
    b = r.uniform(fs[3])
    geom = B.ConvGeom(*g)
    hd = B.handle()
    tc0 = hd.tc_launches
    y_ref, ys = O.conv_forward(x, xs, f, fs, b, g)
    y = B.conv_forward(dev(x, xs), dev(f, fs), torch.from_numpy(b).cuda(), geom, math=math)
    assert B.hwcn_shape(y) == ys
    assert err(host(y), y_ref, math) < TOL[math]
    dy = r.uniform(O.size(ys))
    dx_ref, df_ref, db_ref = O.conv_backward(x, xs, f, fs, g, dy)
    dx, df, db = B.conv_backward(dev(x, xs), dev(f, fs), geom, dev(dy, ys), math=math)
    assert err(host(dx), dx_ref, math) < TOL[math]
    assert err(host(df), df_ref, math) < TOL[math]
    assert rel(host(db), db_ref) < TOL["fp32"]
    tc = hd.tc_launches - tc0
    if math == "fp32":
        assert tc == 0  # the verification path never touches the tensor cores
    elif tc_expected(xs, fs, g):
        assert tc >= 3, f"TF32 conv ran {tc} tcgen05 GEMMs (fprop+dgrad+wgrad expected)"


@pytest.mark.parametrize("xs,fs,g", [((64, 64, 32, 32), (5, 5, 32, 16), (1, 1, 2, 2, 2, 2, 1)),
                                     ((48, 48, 96, 64), (5, 5, 48, 64), (1, 1, 2, 2, 2, 2, 2))])
def test_conv_blocked_dgrad(xs, fs, g):
    """The 2 x 2-blocked data gradient (conv_tc_dgrad: groups of <= 64
    channels, 5 x 5 filters, >= 2^17 pixels -- AlexNet conv2's route): dx
    against the double oracle (oracle/fastconv.py) at the TF32 bound, on
    tcgen05, and accumulate=1 adding onto dx."""
    import fastconv as FC
    r = np.random.default_rng(5)
    x = r.uniform(-1, 1, O.size(xs)).astype(np.float32)
    f = r.uniform(-0.1, 0.1, O.size(fs)).astype(np.float32)
    geom = B.ConvGeom(*g)
    ys = B.conv_output_shape(xs, fs, geom)
    dy = r.uniform(-1, 1, O.size(ys)).astype(np.float32)
    dx_ref, _, _ = FC.conv_backward(x, xs, f, fs, g, dy, want=(True, False, False))
    hd = B.handle()
    tc0 = hd.tc_launches
    dx, _, _ = B.conv_backward(dev(x, xs), dev(f, fs), geom, dev(dy, ys), want_df=False,
                               want_db=False, math="tf32")
    assert hd.tc_launches > tc0
    assert err(host(dx), dx_ref, "tf32") < TOL["tf32"]
    base = r.uniform(-1, 1, O.size(xs)).astype(np.float32)
    acc = dev(base, xs)
    B.conv_backward(dev(x, xs), dev(f, fs), geom, dev(dy, ys), out=(acc, None, None),
                    math="tf32", accumulate=True)
    assert err(host(acc), dx_ref + base, "tf32") < TOL["tf32"]


def _route_cases():
    """Random geometries on the round-2 GEMM routes: 2 x 2-blocked data
    gradients (groups of 16..64 channels, 5x5 / 7x7 filters, >= 2^17 output
    pixels), role-swapped weight gradients (64 / 96 / 192 / 256 filters per
    group), space-to-depth strides with the swap."""
    r = np.random.default_rng(2026)
    cases = []
    for k in range(10):  # blocked dgrad
        cg = int(r.choice([16, 32, 48, 64]))
        groups = int(r.choice([1, 2]))
        f = int(r.choice([5, 7]))
        side = int(r.integers(20, 40))
        n = int(np.ceil(131072 / (side * side)))
        p = int(r.integers(0, f))
        cases.append(((side, side + int(r.integers(0, 3)), cg * groups, n),
                      (f, f, cg, 16 * int(r.integers(1, 5)) * groups),
                      (1, 1, p, f - 1 - p, p, int(r.integers(0, f)), groups)))
    for k in range(8):  # swapped wgrad (stride 1)
        kg = int(r.choice([64, 96, 192]))
        groups = int(r.choice([1, 2]))
        cg = int(r.choice([32, 64, 96]))
        cases.append(((int(r.integers(7, 20)), int(r.integers(7, 20)), cg * groups,
                       int(r.integers(2, 9))), (3, 3, cg, kg * groups), (1, 1, 1, 1, 1, 1, groups)))
    for k in range(4):  # space-to-depth with 64..96 filters (sizes 3 mod 4: the s2d envelope)
        cases.append(((4 * int(r.integers(8, 15)) + 3, 4 * int(r.integers(8, 15)) + 3, 3,
                       int(r.integers(1, 4))),
                      (int(r.choice([7, 11])), int(r.choice([7, 11])), 3, int(r.choice([64, 96]))),
                      (4, 4, 0, 0, 0, 0, 1)))
    return cases


@pytest.mark.parametrize("xs,fs,g", _route_cases())
def test_conv_round2_routes(xs, fs, g):
    """Forward and backward of random geometries on the blocked-dgrad /
    swapped-wgrad / space-to-depth routes against the double oracle
    (oracle/fastconv.py) at the TF32 bound, on tcgen05."""
    import fastconv as FC
    r = np.random.default_rng(sum(xs) + sum(fs))
    geom = B.ConvGeom(*g)
    try:
        ys = B.conv_output_shape(xs, fs, geom)
    except Exception:
        pytest.skip("invalid geometry")
    x = r.uniform(-1, 1, O.size(xs)).astype(np.float32)
    f = r.uniform(-0.1, 0.1, O.size(fs)).astype(np.float32)
    b = r.uniform(-1, 1, fs[3]).astype(np.float32)
    dy = r.uniform(-1, 1, O.size(ys)).astype(np.float32)
    y_ref, _ = FC.conv_forward(x, xs, f, fs, b, g)
    dx_ref, df_ref, db_ref = FC.conv_backward(x, xs, f, fs, g, dy)
    hd = B.handle()
    tc0 = hd.tc_launches
    y = B.conv_forward(dev(x, xs), dev(f, fs), torch.from_numpy(b).cuda(), geom, math="tf32")
    dx, df, db = B.conv_backward(dev(x, xs), dev(f, fs), geom, dev(dy, ys), math="tf32")
    assert hd.tc_launches - tc0 >= 3
    assert err(host(y), y_ref, "tf32") < TOL["tf32"]
    assert err(host(dx), dx_ref, "tf32") < TOL["tf32"]
    assert err(host(df), df_ref, "tf32") < TOL["tf32"]
    assert rel(host(db), db_ref) < 1e-4


@pytest.mark.parametrize("xs,fs,g", [CONV_CASES[9], CONV_CASES[10], CONV_CASES[8],
                                     CONV_CASES[13]])
def test_conv_accumulate_tensor_cores(xs, fs, g):
    """TF32 backward with accumulate=1 (graph.cpp:595 `+=` fused into the
    tcgen05 epilogues / split-K finishers): dx, df, db land on top of what
    was there, and the GEMMs really ran on the tensor cores."""
    r = O.Rng(sum(xs) + 3)
    x, f = r.uniform(O.size(xs)), r.uniform(O.size(fs), -0.1, 0.1)
    _, ys = O.conv_forward(x, xs, f, fs, None, g)
    dy = r.uniform(O.size(ys))
    dx_ref, df_ref, db_ref = O.conv_backward(x, xs, f, fs, g, dy)
    base_dx, base_df, base_db = (r.uniform(O.size(xs)), r.uniform(O.size(fs), -0.1, 0.1),
                                 r.uniform(fs[3]))
    dx, df = dev(base_dx, xs), dev(base_df, fs)
    db = torch.from_numpy(base_db.copy()).cuda()
    hd = B.handle()
    tc0 = hd.tc_launches
    B.conv_backward(dev(x, xs), dev(f, fs), B.ConvGeom(*g), dev(dy, ys), math="tf32",
                    out=(dx, df, db), accumulate=True)
    assert hd.tc_launches - tc0 >= 2
    assert err(host(dx), dx_ref + base_dx, "tf32") < TOL["tf32"]
    assert err(host(df), df_ref + base_df, "tf32") < TOL["tf32"]
    assert rel(host(db), db_ref + base_db) < 1e-4


def test_conv_accumulate_and_skip():
    r = O.Rng(31)
    xs, fs, g = (9, 8, 4, 2), (3, 3, 2, 6), (1, 1, 1, 1, 1, 1, 2)
    x, f = r.uniform(O.size(xs)), r.uniform(O.size(fs))
    _, ys = O.conv_forward(x, xs, f, fs, None, g)
    dy = r.uniform(O.size(ys))
    dx_ref, df_ref, _ = O.conv_backward(x, xs, f, fs, g, dy)
    base_dx, base_df = r.uniform(O.size(xs)), r.uniform(O.size(fs))
    dx, df = dev(base_dx, xs), dev(base_df, fs)
    B.conv_backward(dev(x, xs), dev(f, fs), B.ConvGeom(*g), dev(dy, ys), math="fp32",
                    out=(dx, df, None), accumulate=True)
    assert rel(host(dx), dx_ref + base_dx) < 1e-4
    assert rel(host(df), df_ref + base_df) < 1e-4


CONVT_CASES = [
    # small channel counts: the FP32 SIMT kernels (outside the tcgen05 envelope)
    ((5, 4, 6, 2), (3, 2, 6, 4), (2, 1, 1, 0, 0, 1), False),
    # >= 16 channels, up = 1 with crops: the stride-1 tcgen05 path
    ((9, 8, 32, 2), (3, 3, 32, 48), (1, 1, 1, 1, 0, 1), True),
    # >= 16 channels, up = 2 (FCN-style 2x upsampling): the space-to-depth tcgen05 path
    ((7, 6, 64, 3), (4, 4, 64, 32), (2, 2, 0, 0, 0, 0), True),
    ((8, 8, 48, 2), (3, 3, 48, 16), (2, 2, 0, 0, 0, 0), True),
]


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("xs,fs,cg,tc", CONVT_CASES)
def test_convt(xs, fs, cg, tc, math):
    """conv.cpp:283-365: y = M^T x, dx = conv of dy with the swapped bank, df."""
    r = O.Rng(32 + sum(xs))
    x, f = r.uniform(O.size(xs)), r.uniform(O.size(fs), -0.2, 0.2)
    y_ref, ys = O.convt_forward(x, xs, f, fs, cg)
    geom = B.ConvTransposeGeom(*cg)
    hd = B.handle()
    tc0 = hd.tc_launches
    y = B.convt_forward(dev(x, xs), dev(f, fs), geom, math=math)
    assert B.hwcn_shape(y) == ys
    assert err(host(y), y_ref, math) < TOL[math]
    dy = r.uniform(O.size(ys))
    dx_ref, df_ref = O.convt_backward(x, xs, f, fs, cg, dy)
    dx, df = B.convt_backward(dev(x, xs), dev(f, fs), geom, dev(dy, ys), math=math)
    assert err(host(dx), dx_ref, math) < TOL[math]
    assert err(host(df), df_ref, math) < TOL[math]
    ran = hd.tc_launches - tc0
    if math == "tf32" and tc:
        assert ran >= 3, f"convt ran {ran} tcgen05 GEMMs"
    if math == "fp32":
        assert ran == 0


def test_conv_shape_errors():
    x = B.from_hwcn((5, 5, 4, 1))
    with pytest.raises(B.ShapeError, match="do not match input channels"):
        B.conv_forward(x, B.from_hwcn((3, 3, 3, 6)), None, B.ConvGeom())
    with pytest.raises(B.ShapeError, match="not divisible by groups"):
        B.conv_forward(x, B.from_hwcn((3, 3, 2, 5)), None, B.ConvGeom(groups=2))
    with pytest.raises(B.ShapeError, match="larger than padded input"):
        B.conv_forward(x, B.from_hwcn((7, 3, 4, 2)), None, B.ConvGeom())
    with pytest.raises(B.ShapeError, match="bias has"):
        B.conv_forward(x, B.from_hwcn((3, 3, 4, 2)), torch.zeros(3, device="cuda"), B.ConvGeom())


POOLS = [(3, 3, 2, 2, 0, 1, 0, 1, 0), (3, 3, 2, 2, 0, 1, 0, 1, 1), (2, 2, 2, 2, 0, 0, 0, 0, 0),
         (3, 2, 1, 2, 2, 1, 1, 0, 1), (4, 4, 3, 3, 3, 0, 0, 3, 0)]


@pytest.mark.parametrize("pg", POOLS)
@pytest.mark.parametrize("xs", [(13, 11, 3, 2), (55, 55, 8, 2), (1, 1, 2, 1), (28, 24, 5, 3)])
def test_pool_bitexact(xs, pg):
    try:
        _, ys = O.pool_forward(np.zeros(O.size(xs)), xs, pg)
    except O.OracleError:
        with pytest.raises(B.ShapeError):
            B.pool_forward(B.from_hwcn(xs, fill=0.0), B.PoolGeom(*pg[:8], mode="max" if pg[8] == 0 else "avg"))
        return
    r = O.Rng(33)
    x = r.uniform(O.size(xs))
    if x.size > 20:
        x[::5] = x[2::5][: len(x[::5])]  # ties
    geom = B.PoolGeom(*pg[:8], mode="max" if pg[8] == 0 else "avg")
    y_ref, ys = O.pool_forward(x, xs, pg)
    y = B.pool_forward(dev(x, xs), geom)
    assert np.array_equal(host(y), y_ref)
    dy = r.uniform(O.size(ys))
    dx = B.pool_backward(dev(x, xs), geom, dev(dy, ys))
    assert np.array_equal(host(dx), O.pool_backward(x, xs, pg, dy))


@pytest.mark.parametrize("pg", POOLS[:3])
def test_pool_shared_argmax_order(pg):
    """Spikes at window corners are the argmax of up to 4 overlapping windows:
    dx sums >= 3 contributions, so the (oj, oi) accumulation order shows."""
    xs = (27, 27, 4, 3)
    r = O.Rng(34)
    x = r.uniform(O.size(xs), -0.01, 0.01).reshape(xs[::-1])
    x[:, :, ::2, ::2] += 1.0 + r.uniform(x[:, :, ::2, ::2].size).reshape(x[:, :, ::2, ::2].shape)
    x = x.ravel()
    geom = B.PoolGeom(*pg[:8], mode="max" if pg[8] == 0 else "avg")
    y_ref, ys = O.pool_forward(x, xs, pg)
    assert np.array_equal(host(B.pool_forward(dev(x, xs), geom)), y_ref)
    dy = r.uniform(O.size(ys), -1e3, 1e3) * r.uniform(O.size(ys), 0.5, 1.5) ** 20
    dx = B.pool_backward(dev(x, xs), geom, dev(dy, ys))
    assert np.array_equal(host(dx), O.pool_backward(x, xs, pg, dy))


def test_relu_bitexact():
    r = O.Rng(34)
    for n in (1000, 1001, 4096 * 7 + 3):
        x = r.uniform(n)
        x[::9] = 0
        dy = r.uniform(n)
        xs = (n, 1, 1, 1)
        assert np.array_equal(host(B.relu_forward(dev(x, xs))), O.relu_forward(x))
        assert np.array_equal(host(B.relu_backward(dev(x, xs), dev(dy, xs))), O.relu_backward(x, dy))


@pytest.mark.parametrize("p", [(5, 1.0, 2e-5, 0.75), (3, 1.0, 5e-5 / 3, 0.75), (4, 2.0, 0.1, 0.5)])
@pytest.mark.parametrize("xs", [(7, 5, 9, 2), (27, 27, 96, 1), (13, 13, 256, 1)])
def test_lrn(xs, p):
    r = O.Rng(35)
    x, dy = r.uniform(O.size(xs)) * 3, r.uniform(O.size(xs))
    lp = B.LrnParams(*p)
    y = B.lrn_forward(dev(x, xs), lp)
    assert rel(host(y), O.lrn_forward(x, xs, *p)) < 1e-5
    dx = B.lrn_backward(dev(x, xs), lp, dev(dy, xs))
    assert rel(host(dx), O.lrn_backward(x, xs, *p, dy)) < 1e-4


@pytest.mark.parametrize("xs", [(6, 5, 4, 3), (28, 28, 64, 8), (1, 1, 7, 5)])
def test_bnorm(xs):
    r = O.Rng(36)
    x, dy = r.uniform(O.size(xs)) * 2 + 0.5, r.uniform(O.size(xs))
    w, b = r.uniform(xs[2]), r.uniform(xs[2])
    wt, bt = torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda()
    y_ref, m_ref, v_ref = O.bnorm_forward(x, xs, w, b, 1e-5)
    y, mom = B.bnorm_forward(dev(x, xs), wt, bt, 1e-5)
    assert rel(host(y), y_ref) < 1e-4
    assert rel(host(mom), np.concatenate([m_ref, v_ref])) < 1e-5
    yi = B.bnorm_infer(dev(x, xs), wt, bt, 1e-5, mom)
    assert rel(host(yi), y_ref) < 1e-4
    dx_ref, dw_ref, db_ref = O.bnorm_backward(x, xs, w, b, 1e-5, dy)
    dx, dw, db = B.bnorm_backward(dev(x, xs), wt, bt, 1e-5, dev(dy, xs))
    assert rel(host(dx), dx_ref) < 1e-4
    assert rel(host(dw), dw_ref) < 1e-4
    assert rel(host(db), db_ref) < 1e-4


def test_softmaxlog():
    r = O.Rng(37)
    for xs in [(1, 1, 1000, 64), (2, 3, 17, 4), (1, 1, 10, 100)]:
        cs = (xs[0], xs[1], 1, xs[3])
        x = r.uniform(O.size(xs)) * 4
        c = r.labels(O.size(cs), xs[2])
        c[1] = 0
        w = r.uniform(O.size(cs), 0, 2)
        for wts in (None, w):
            l_ref = O.loss_forward(x, xs, c, cs, wts)
            l = B.loss_forward(dev(x, xs), dev(c, cs), None if wts is None else dev(wts, cs))
            assert abs(host(l)[0] - l_ref) < 1e-5 * max(1.0, abs(l_ref))
            dx = B.loss_backward(dev(x, xs), dev(c, cs), None if wts is None else dev(wts, cs), 0.5)
            assert rel(host(dx), O.softmaxlog_backward(x, xs, c, cs, wts, 0.5)) < 1e-5
        m = host(B.loss_metrics(dev(x, xs), dev(c, cs), None, 5))
        assert m[0] == O.loss_forward(x, xs, c, cs, None, "classerror")
        assert m[1] == O.loss_forward(x, xs, c, cs, None, "topk", 5)
    # stability at +-1000
    xs, cs = (1, 1, 2, 1), (1, 1, 1, 1)
    l = host(B.loss_forward(dev([1000, -1000], xs), dev([2], cs)))[0]
    assert np.isfinite(l) and abs(l - 2000) < 1e-2


def test_label_errors():
    xs, cs = (1, 1, 3, 1), (1, 1, 1, 1)
    with pytest.raises(B.DataError, match="not an integer"):
        B.loss_forward(dev([0, 0, 0], xs), dev([1.5], cs))
    with pytest.raises(B.DataError, match="out of range"):
        B.loss_forward(dev([0, 0, 0], xs), dev([4], cs))
    with pytest.raises(B.ShapeError, match="classification labels"):
        B.loss_forward(dev([0, 0, 0], xs), dev([1, 1], (1, 1, 1, 2)))


def test_sgd_bitexact():
    r = O.Rng(38)
    n = 10007
    w, v, g = r.uniform(n), r.uniform(n), r.uniform(n)
    wt, vt, gt = (torch.from_numpy(a.copy()).cuda() for a in (w, v, g))
    B.sgd_step(wt, vt, gt, 0.01, 0.9, 5e-4)
    w_ref, v_ref = O.sgd_step(w, v, g, 0.01, 0.9, 5e-4)
    assert np.array_equal(host(vt), v_ref)
    assert np.array_equal(host(wt), w_ref)


@pytest.mark.parametrize("path", ["CK_TC_SHIFT", "CK_TC_HALO"])
@pytest.mark.parametrize("xs,fs,g", [CONV_CASES[5], CONV_CASES[7], CONV_CASES[9], CONV_CASES[8]])
def test_conv_experimental_paths(xs, fs, g, path, monkeypatch):
    """The experimental shifted-grid and halo-reuse kernels (conv_tc.cu, built
    only with -DCK_EXPERIMENTS) stay within the TF32 tolerance of the oracle."""
    from paper_1412_4564_b200._lib import lib
    if b"CK_EXPERIMENTS" not in lib().ck_version():
        pytest.skip("experiment kernels are not in product builds")
    monkeypatch.setenv(path, "1")
    r = O.Rng(sum(xs) + sum(fs) + 7)
    x = r.uniform(O.size(xs))
    f = r.uniform(O.size(fs), -0.1, 0.1)
    b = r.uniform(fs[3])
    geom = B.ConvGeom(*g)
    y_ref, ys = O.conv_forward(x, xs, f, fs, b, g)
    y = B.conv_forward(dev(x, xs), dev(f, fs), torch.from_numpy(b).cuda(), geom, math="tf32")
    assert err(host(y), y_ref, "tf32") < TOL["tf32"]
    dy = r.uniform(O.size(ys))
    dx_ref, _, _ = O.conv_backward(x, xs, f, fs, g, dy)
    dx, _, _ = B.conv_backward(dev(x, xs), dev(f, fs), geom, dev(dy, ys), math="tf32")
    assert err(host(dx), dx_ref, "tf32") < TOL["tf32"]
