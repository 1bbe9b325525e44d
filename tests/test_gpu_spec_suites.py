"""The SPEC.md acceptance suites run on the device:
transposed-convolution duality over 50 random configurations, a geometry
sweep of the shape laws against the oracle (including the error cases and
their messages), and desk-scale learning of a LeNet on a synthetic 10-class
set through the training loop."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _dev(B, a, shape):
    return B.as_hwcn(torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda(), shape)


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_convt_duality_sweep(math):
    """<y, conv(x)> == <convt(y), x> for the SAME bank, over
    50 random (size, filter, stride/upsampling, pad/crop, channels)
    configurations -- every conv / convt kernel path (FP32 SIMT; tcgen05
    grid, space-to-depth and FC routes in TF32)."""
    from paper_1412_4564_b200 import blocks as B
    rng = np.random.default_rng(7)
    worst = 0.0
    for it in range(50):
        s = int(rng.integers(1, 4))
        fh, fw = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        C, K = int(rng.choice([1, 3, 16, 32, 40])), int(rng.choice([2, 16, 32, 48]))
        H, W = int(rng.integers(fh, 14)), int(rng.integers(fw, 14))
        N = int(rng.integers(1, 4))
        pt, pb = int(rng.integers(0, fh)), int(rng.integers(0, fh))
        pl, pr = int(rng.integers(0, fw)), int(rng.integers(0, fw))
        xs, fs = (H, W, C, N), (fh, fw, C, K)
        g = (s, s, pt, pb, pl, pr, 1)
        try:
            ys = O.conv_output_shape(xs, fs, g)
        except O.OracleError:
            continue
        x = rng.uniform(-1, 1, size=O.size(xs)).astype(np.float32)
        f = rng.uniform(-1, 1, size=O.size(fs)).astype(np.float32)
        y = rng.uniform(-1, 1, size=O.size(ys)).astype(np.float32)
        cx = B.conv_forward(_dev(B, x, xs), _dev(B, f, fs), None, B.ConvGeom(*g), math=math)
        # the transposed conv of y with the bank f viewed as (fh, fw, K, C):
        # convt's y = M^T x where M is the conv with stride = up, pad = crop
        ftt = f.reshape(K, C, fw, fh).transpose(1, 0, 2, 3).ravel()  # swap (C, K) roles
        ty = B.convt_forward(_dev(B, y, ys), _dev(B, ftt, (fh, fw, K, C)),
                             B.ConvTransposeGeom(s, s, pt, pb, pl, pr), math=math)
        assert B.hwcn_shape(ty) == xs
        torch.cuda.synchronize()
        lhs = float(np.dot(y.astype(np.float64), cx.cpu().numpy().ravel().astype(np.float64)))
        rhs = float(np.dot(ty.cpu().numpy().ravel().astype(np.float64), x.astype(np.float64)))
        scale = np.abs(y).sum() * np.abs(cx.cpu().numpy()).max() + 1e-30
        worst = max(worst, abs(lhs - rhs) / scale)
    assert worst < (1e-5 if math == "fp32" else 2e-3), worst


def test_geometry_sweep():
    """output-size laws of conv / convt / pool against the
    oracle on 300 random geometries, and the same accept/reject decisions
    (with the reference's messages) where the geometry is invalid."""
    from paper_1412_4564_b200 import blocks as B
    from paper_1412_4564_b200._lib import CkError
    rng = np.random.default_rng(11)
    n_ok = n_err = 0
    for it in range(300):
        H, W, C, N = (int(v) for v in rng.integers(1, 20, size=4))
        fh, fw = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        groups = int(rng.choice([1, 2, 3]))
        K = groups * int(rng.integers(1, 5))
        Cf = C // groups if rng.random() < 0.9 else C  # sometimes a channel mismatch
        g = [int(rng.integers(1, 4)), int(rng.integers(1, 4))] + \
            [int(v) for v in rng.integers(0, 4, size=4)] + [groups]
        xs, fs = (H, W, C, N), (fh, fw, max(Cf, 1), K)
        try:
            want = O.conv_output_shape(xs, fs, g)
        except O.OracleError as e:
            with pytest.raises(CkError):
                B.conv_output_shape(xs, fs, B.ConvGeom(*g))
            n_err += 1
            continue
        assert B.conv_output_shape(xs, fs, B.ConvGeom(*g)) == want
        n_ok += 1
        pg = [fh, fw, g[0], g[1], *(min(v, fh - 1) for v in g[2:4]),
              *(min(v, fw - 1) for v in g[4:6]), int(rng.integers(0, 2))]
        try:
            pw = O.pool_output_shape(xs, pg)
            assert B.pool_output_shape(xs, B.PoolGeom(*pg[:8], mode="max" if pg[8] == 0
                                                      else "avg")) == pw
        except O.OracleError:
            with pytest.raises(CkError):
                B.pool_output_shape(xs, B.PoolGeom(*pg[:8]))
        cg = [g[0], g[1], *(int(v) for v in rng.integers(0, 3, size=4))]
        try:
            cw = O.convt_output_shape(xs, (fh, fw, C, K), cg)
            assert B.convt_output_shape(xs, (fh, fw, C, K), B.ConvTransposeGeom(*cg)) == cw
        except O.OracleError:
            with pytest.raises(CkError):
                B.convt_output_shape(xs, (fh, fw, C, K), B.ConvTransposeGeom(*cg))
    assert n_ok > 50 and n_err > 10


def test_lenet_learns_synthetic_digits():
    """SPEC.md:720, :782 (desk-scale learning, property-based): a LeNet trained
    with the epoch loop (Trainer.fit: seeded shuffles, SGD with momentum)
    reaches < 5% validation top-1 error within 5 epochs on a synthetic
    10-class 28x28 set (one random prototype per class plus noise), the
    bundled-synthetic-set option of the spec where MNIST is absent."""
    from paper_1412_4564_b200 import blocks as B
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Graph, Trainer
    rng = np.random.default_rng(3)
    protos = rng.uniform(0, 1, size=(10, 28 * 28)).astype(np.float32)

    def make(n, seed):
        r = np.random.default_rng(seed)
        y = r.integers(0, 10, size=n)
        x = protos[y] + r.normal(0, 0.35, size=(n, 28 * 28)).astype(np.float32)
        return x.astype(np.float32).ravel(), (y + 1).astype(np.float32)

    xtr, ytr = make(2000, 1)
    xva, yva = make(500, 2)
    net = nets.lenet(batch=100)
    params = net.init_params()
    params = {k: (v * 5 if k.endswith("f") else v) for k, v in params.items()}
    g = Graph(math="tf32")
    net.build(g)
    g.finalize()
    for k, v in params.items():
        g.set(k, v)
    t = Trainer(g, lr=0.01 / 100, momentum=0.9, weight_decay=5e-4)
    recs = t.fit(xtr, ytr, epochs=5, seed=17)
    assert recs[-1]["loss"] < recs[0]["loss"]
    wrong = 0
    for b in range(0, 500, 100):
        g.set("data", xva[b * 784:(b + 100) * 784])
        g.set("label", yva[b:b + 100])
        g.forward()
        x7 = torch.from_numpy(g.get("x7")).cuda()
        m = B.loss_metrics(B.as_hwcn(x7, (1, 1, 10, 100)),
                           B.as_hwcn(torch.from_numpy(yva[b:b + 100]).cuda(), (1, 1, 1, 100)))
        wrong += float(m[0].item())
    assert wrong / 500 < 0.05, (wrong / 500, recs)
