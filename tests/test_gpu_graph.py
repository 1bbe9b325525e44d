"""Whole-network parity: the device DAG engine (engine.cu) vs the oracle
chain (oracle/chain.py, the reference DAG semantics of graph.cpp:494-598)
on the BASELINE.json networks at small batch, plus size-independent
properties at the full AlexNet batch."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = 1e-2 * np.max(np.abs(b)) + 1e-30  # see test_gpu_blocks.rel
    elem = float(np.max(np.abs(a - b) / np.maximum(np.abs(a) + np.abs(b), floor)))
    norm = float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
    return max(elem, 10 * norm)


def device_graph(net, math):
    from paper_1412_4564_b200.graph import Graph
    g = Graph(math=math)
    net.build(g)
    g.finalize()
    return g


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return max(float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)),
               float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-30)))


def test_tf32_operand_rounding_mode():
    """What the tcgen05 kind::tf32 MMA does to an fp32 operand's low 13
    mantissa bits, measured: x = 1 + 3*2^-12 times 1 is 1 if they are dropped
    (round toward zero), 1 + 2^-10 if rounded to nearest.  The TF32-emulating
    oracle (chain.tf32_operand) must use the measured mode."""
    import chain
    from paper_1412_4564_b200 import blocks as B
    xs, fs = (8, 8, 16, 1), (1, 1, 16, 16)
    x = np.zeros(O.size(xs), np.float32)
    x[: 64] = 1 + 3 * 2.0 ** -12       # channel 0 only
    f = np.zeros(O.size(fs), np.float32)
    f[0::16] = 1.0                      # every filter reads channel 0 with weight 1
    hd = B.handle()
    t0 = hd.tc_launches
    y = B.conv_forward(B.as_hwcn(torch.from_numpy(x).cuda(), xs),
                       B.as_hwcn(torch.from_numpy(f).cuda(), fs), None, B.ConvGeom(), math="tf32")
    torch.cuda.synchronize()
    assert hd.tc_launches > t0
    v = float(y.cpu().numpy().ravel()[0])
    mode = {1.0: "rz", 1 + 2.0 ** -10: "rn"}.get(v)
    assert mode is not None, v
    assert chain.TF32_MODE == mode, f"hardware rounds TF32 operands '{mode}'"
    assert chain.tf32_operand(np.array([x[0]]))[0] == v


# Network-level parity (whole forward + backward through the DAG engine vs the
# oracle DAG, oracle/chain.py).
#   FP32: against the exact (double) oracle routed by the device's ReLU masks /
#         max-pool argmaxes (see TF32), every derivative within 1e-4 normwise
#         (max(||a-b||/||b||, max|a-b|/max|b|)); even FP32 flips a pre-activation
#         that sits within an ulp of 0 now and then (VGG: 1 site at relu4).
#   TF32: against the oracle evaluated on the same TF32-rounded conv operands
#         (the passes on TF32 operands, netcheck.tc_passes) AND routed by the
#         device's own ReLU masks / max-pool argmaxes (chain.run gates): every
#         derivative within 1e-2 normwise.  Holding the discrete routing fixed is
#         what makes a network-level TF32 bound meaningful: a 1e-5 difference in
#         a pre-activation flips a handful of ReLUs (tools/tf32_divergence.py:
#         1-30 per layer), each moving one element's full derivative -- the
#         routing decisions themselves are checked bit-exactly, layer by layer,
#         from the device's inputs in test_headline_layers_vs_oracle.  The drift
#         from the exact, free-routing oracle is printed, not bounded.
NET_CASES = [("lenet", 4, {}), ("cifar", 4, {}), ("alexnet", 2, {}), ("vgg16bn", 2, {"image": 64})]


def _gates(net, g):
    return {l[2][0]: g.get(l[2][0]) for l in net.layers if l[0] in ("relu", "pool")}


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("name,batch,kw", NET_CASES)
def test_network_fwd_bwd(name, batch, kw, math, capsys):
    import chain
    import netcheck
    from paper_1412_4564_b200 import nets
    net = nets.NETS[name](batch=batch, **kw)
    params, inputs = net.init_params(), net.init_inputs()
    if name == "vgg16bn":  # make the deep net's logits non-degenerate
        params = {k: (v * 20 if k.endswith("f") else v) for k, v in params.items()}
    g = device_graph(net, math)
    for k, v in {**params, **inputs}.items():
        g.set(k, v)
    g.forward()
    g.backward("objective")
    vals, derivs = chain.run(net, params, inputs)
    # routed by the device's ReLU masks / max-pool argmaxes in both modes: a
    # pre-activation within an ulp of 0 may flip between summation orders
    # (FP32 VGG: 1 site of 2 x 64 x 32 x 32 x 128 at relu4 moves conv1f by
    # 9e-4 normwise, 7e-6 once routed); the routing itself is checked
    # bit-exactly in test_headline_layers_vs_oracle
    tvals, tderivs = chain.run(net, params, inputs,
                               tf32=netcheck.tc_passes(net) if math == "tf32" else False,
                               gates=_gates(net, g))
    loss = g.get("objective")[0]
    tol = 1e-4 if math == "fp32" else 1e-2
    assert abs(loss - tvals["objective"][0]) <= tol * abs(tvals["objective"][0])
    worst, drift = 0.0, 0.0
    for pname in [p[0] for p in net.params] + ["data"]:
        ours, ref = g.get(pname, deriv=True), tderivs[pname]
        scale = max(np.abs(tderivs[pname.rstrip("bw") + "f"]).max() if pname.rstrip("bw") + "f"
                    in tderivs else 0.0, np.abs(ref).max())
        if np.abs(ref).max() < 1e-7 * scale:
            # mathematically zero (a conv bias followed by bnorm): only check smallness
            assert np.abs(ours).max() < 1e-3 * scale, pname
            continue
        e = normwise(ours, ref)
        worst = max(worst, e)
        drift = max(drift, normwise(ours, derivs[pname]))
        assert e < tol, (pname, e)
    with capsys.disabled():
        print(f"\n  [{name} b={batch} {math}] worst derivative error {worst:.2e}"
              f" (vs exact free-routing oracle: {drift:.2e})")
    assert g.last_launches > 0


@pytest.mark.parametrize("math", ["tf32", "fp32"])
def test_headline_layers_vs_oracle(math, capsys):
    """The exact bench configuration (AlexNet b=256, bench.py) layer by layer:
    every layer re-evaluated on the CPU from the device's own inputs
    (tests/netcheck.py) -- conv fprop/dgrad/wgrad against the double oracle
    at the same M = 256*OH*OW that selects the bench's tile heights, split-K
    factors and persistent waves (conv_tc.cu pick_bm / split_for /
    wgrad_splits_for): TF32 within 1e-2 normwise of the exact oracle and
    within 1e-4 of the TF32-operand oracle, FP32 within 1e-4; pooling (pool1
    55x55 -> SEG 32 strips, pool2 27x27 -> 16, pool5 13x13 -> 8) and ReLU
    bit-exact; LRN / loss 1e-4 -- including the fused conv+ReLU epilogues and
    the LRN-backward -> conv dy-grid writers the bench step runs."""
    import netcheck
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=256)
    g = device_graph(net, math)
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        g.set(k, v)
    hd = g.hd
    tc0 = hd.tc_launches
    g.forward()
    g.backward("objective")
    torch.cuda.synchronize()
    if math == "tf32":
        assert hd.tc_launches - tc0 >= 3 * 8 - 1  # every conv/fc pass on tcgen05
    rep = netcheck.check_layers(net, g, math)
    with capsys.disabled():
        worst = {}
        for (layer, what), e in rep.items():
            worst[what] = max(worst.get(what, 0.0), e)
        print(f"\n  [alexnet b=256 {math}] worst per quantity: "
              + ", ".join(f"{k}={v:.1e}" for k, v in sorted(worst.items())))


def test_trainer_step_matches_oracle_sgd():
    import chain
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Trainer
    net = nets.lenet(batch=8)
    params, inputs = net.init_params(), net.init_inputs()
    vals, derivs = chain.run(net, params, inputs)
    g = device_graph(net, "fp32")
    for k, v in {**params, **inputs}.items():
        g.set(k, v)
    t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
    loss = t.step()
    assert abs(loss - vals["objective"][0]) < 1e-4 * vals["objective"][0]
    for pname, _, _ in net.params:
        w_ref, _ = O.sgd_step(params[pname], np.zeros_like(params[pname]),
                              derivs[pname].astype(np.float32), 0.01, 0.9, 5e-4)
        assert rel(g.get(pname), w_ref) < 1e-4, pname
    # a few steps reduce the loss on a fixed batch
    for _ in range(5):
        last = t.step()
    assert last < loss


def test_alexnet_full_batch_properties():
    """Full BASELINE size (b=256): properties the oracle need not run."""
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=256)
    g = device_graph(net, "tf32")
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        g.set(k, v)
    g.forward()
    g.backward("objective")
    loss = g.get("objective")[0]
    # random init: logits ~0 -> loss ~ 256 ln 1000
    assert abs(loss - 256 * np.log(1000)) < 0.01 * 256 * np.log(1000)
    # softmaxlog derivative sums to zero per image (loss.cpp:263-275)
    d8 = g.get("f8", deriv=True).reshape(256, 1000)
    assert np.abs(d8.sum(axis=1)).max() < 1e-4
    # max-pool backward conserves mass: sum dx = sum dy
    assert abs(g.get("r5", deriv=True).sum(dtype=np.float64) -
               g.get("p5", deriv=True).sum(dtype=np.float64)) < 1e-3 * (
                   np.abs(g.get("p5", deriv=True)).sum() + 1e-12)
    # relu backward is a mask of its input's sign
    r6, c6 = g.get("r6", deriv=True), g.get("f6")
    assert np.all(g.get("f6", deriv=True)[c6 <= 0] == 0)
    assert np.isfinite(g.get("conv1f", deriv=True)).all()


def test_fused_conv_relu_derivative_materialized_on_request():
    """A fused conv -> relu backward leaves the conv output's derivative
    unstored (only its grid form feeds the GEMMs); requesting it computes the
    relu backward (activation.cpp:14-22) exactly: d(conv) = conv > 0 ? d(relu) : 0."""
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=32)
    g = device_graph(net, "tf32")
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        g.set(k, v)
    for _ in range(2):  # the second backward must not see the first one's derivative
        g.forward()
        g.backward("objective")
        for c, r in [("c1", "r1"), ("c2", "r2"), ("c3", "r3"), ("c4", "r4"), ("c5", "r5"),
                     ("f6", "r6"), ("f7", "r7")]:
            dc, cv, dr = g.get(c, deriv=True), g.get(c), g.get(r, deriv=True)
            assert np.array_equal(dc, np.where(cv > 0, dr, np.float32(0))), c


def test_vgg224_layers_vs_oracle(capsys):
    """VGG-16-bn at its real 224x224 image (b=2), TF32, layer by layer from
    the device's own inputs (netcheck): the first conv's 3-channel tcgen05
    path (channels padded to 32, last_k skipping the zero K steps), the fused
    bnorm -> relu apply / gated backward, the 2x2 pooling kernels, the fc6
    7x7x512 layer -- exact pooling/ReLU, TF32 convs 1e-2 (1e-4 against the
    TF32-operand oracle), bnorm 1e-4."""
    import netcheck
    from paper_1412_4564_b200 import nets
    net = nets.vgg16_bn(batch=2, image=224)
    params = {k: (v * 20 if k.endswith("f") else v) for k, v in net.init_params().items()}
    g = device_graph(net, "tf32")
    for k, v in {**params, **net.init_inputs()}.items():
        g.set(k, v)
    g.forward()
    g.backward("objective")
    rep = netcheck.check_layers(net, g, "tf32")
    with capsys.disabled():
        worst = {}
        for (layer, what), e in rep.items():
            worst[what] = max(worst.get(what, 0.0), e)
        print("\n  [vgg16bn 224 b=2 tf32] worst per quantity: "
              + ", ".join(f"{k}={v:.1e}" for k, v in sorted(worst.items())))


def test_fused_bnorm_relu_derivative_materialized_on_request():
    """bnorm -> relu (VGG): the bnorm apply writes relu(y) too, the backward
    gates the relu output's derivative by y > 0 inside both bnorm passes, and
    the bnorm output's derivative is computed on request -- exactly the relu
    backward (activation.cpp:14-22)."""
    from paper_1412_4564_b200 import nets
    net = nets.vgg16_bn(batch=2, image=32)
    g = device_graph(net, "tf32")
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        g.set(k, v)
    for _ in range(2):
        g.forward()
        g.backward("objective")
        for k in (1, 5, 13):
            b, r = f"b{k}", f"r{k}"
            bv, dr = g.get(b), g.get(r, deriv=True)
            assert np.array_equal(g.get(r), np.maximum(bv, 0)), r
            assert np.array_equal(g.get(b, deriv=True), np.where(bv > 0, dr, np.float32(0))), b


@pytest.mark.parametrize("net_name,batch", [("alexnet", 16), ("alexnet", 3), ("cifar", 8)])
def test_lrn_writes_conv_dy_grid(net_name, batch, monkeypatch):
    """conv -> relu -> lrn chains (TF32): the LRN backward writes the conv's
    ReLU-gated dy grid and bias partials directly (lrn_backward_grid); the
    relu output's and conv output's derivatives are computed on request.
    Everything but the conv biases' gradients (32-pixel float partials, then
    double, in another fixed order) is bit-identical to the unfused engine;
    those agree to 1e-5 of the largest."""
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=batch) if net_name == "alexnet" else nets.cifar(batch=batch)
    out = []
    for fuse in (True, False):
        g = device_graph(net, "tf32")
        g.set_option("lrn_grid", fuse)
        for k, v in {**net.init_params(), **net.init_inputs()}.items():
            g.set(k, v)
        g.forward()
        g.backward("objective")
        names = set(net.inputs) | {p[0] for p in net.params} | \
            {o for layer in net.layers for o in layer[3]}
        out.append({name: g.get(name, deriv=True) for name in sorted(names) if name != "label"})
    biases = {p[0] for p in net.params if p[0].endswith("b")}
    for name in out[1]:
        a, b = out[0][name], out[1][name]
        if name in biases:
            assert np.abs(a - b).max() <= 1e-5 * (np.abs(b).max() + 1e-30), name
        else:
            assert np.array_equal(a, b), name


@pytest.mark.parametrize("batch", [3, 32])
def test_lrn_maxpool_fusion_bitexact(batch):
    """lrn -> 3x3/2 max pool (AlexNet norm1/pool1, norm2/pool2) as one kernel
    (kernels.cu lrn_maxpool3s2_k): every value and derivative of the network is
    bit-identical to the unfused blocks (normalize.cpp:47-71 then
    pool.cpp:49-80, same float operations, same argmax routing)."""
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=batch)
    out = []
    for fuse in (True, False):
        g = device_graph(net, "tf32")
        g.set_option("lrn_pool", fuse)
        for k, v in {**net.init_params(), **net.init_inputs()}.items():
            g.set(k, v)
        hd = g.hd
        l0 = hd.launches
        g.forward()
        launches = hd.launches - l0
        g.backward("objective")
        names = set(net.inputs) | {p[0] for p in net.params} | \
            {o for layer in net.layers for o in layer[3]}
        out.append(({n: g.get(n) for n in sorted(names)},
                    {n: g.get(n, deriv=True) for n in sorted(names) if n != "label"}, launches))
    (v0, d0, l0), (v1, d1, l1) = out
    assert l0 == l1 - 2  # the two pool layers launched nothing of their own
    for n in v1:
        assert np.array_equal(v0[n], v1[n]), n
    for n in d1:
        assert np.array_equal(d0[n], d1[n]), n


@pytest.mark.parametrize("batch", [5, 32])
def test_producer_written_x_grid_bitexact(batch):
    """conv3 -> relu3 -> conv4 -> relu4 -> conv5 (TF32): each forward epilogue
    also writes relu(y) into the next conv's padded pixel-major x grid, whose
    forward and weight gradient then skip their input transform.  Every
    value and derivative is bit-identical to the transform path, and the
    engine launches two kernels fewer per forward."""
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=batch)
    out = []
    for on in (True, False):
        g = device_graph(net, "tf32")
        g.set_option("producer_grid", on)
        for k, v in {**net.init_params(), **net.init_inputs()}.items():
            g.set(k, v)
        l0 = g.hd.launches
        g.forward()
        launches = g.hd.launches - l0
        g.backward("objective")
        names = set(net.inputs) | {p[0] for p in net.params} | \
            {o for layer in net.layers for o in layer[3]}
        out.append(({n: g.get(n) for n in sorted(names)},
                    {n: g.get(n, deriv=True) for n in sorted(names) if n != "label"}, launches))
    (v0, d0, l0), (v1, d1, l1) = out
    assert l0 == l1 - 2
    for n in v1:
        assert np.array_equal(v0[n], v1[n]), n
    for n in d1:
        assert np.array_equal(d0[n], d1[n]), n


@pytest.mark.parametrize("batch", [3, 16])
def test_dgrad_writes_conv_dy_grid(batch):
    """conv -> relu -> conv backward (AlexNet conv3 -> conv4 -> conv5): the
    second conv's data-gradient epilogue also writes the first conv's
    ReLU-gated dy grid and bias partials, so the first conv's backward skips
    its dy transform (2 fewer launches).  Every value and derivative is
    bit-identical to the unfused engine except the conv3/conv4 bias gradients
    (32-row float partials in another fixed order): 1e-5 of the largest."""
    from paper_1412_4564_b200 import nets
    net = nets.alexnet(batch=batch)
    out = []
    for on in (True, False):
        g = device_graph(net, "tf32")
        g.set_option("dgrad_grid", on)
        for k, v in {**net.init_params(), **net.init_inputs()}.items():
            g.set(k, v)
        g.forward()
        l0 = g.hd.launches
        g.backward("objective")
        launches = g.hd.launches - l0
        names = set(net.inputs) | {p[0] for p in net.params} | \
            {o for layer in net.layers for o in layer[3]}
        out.append(({n: g.get(n) for n in sorted(names)},
                    {n: g.get(n, deriv=True) for n in sorted(names) if n != "label"}, launches))
    (v0, d0, l0), (v1, d1, l1) = out
    assert l0 == l1 - 2, (l0, l1)
    for n in v1:
        assert np.array_equal(v0[n], v1[n]), n
    for n in d1:
        if n in ("conv3b", "conv4b"):
            assert np.abs(d0[n] - d1[n]).max() <= 1e-5 * (np.abs(d1[n]).max() + 1e-30), n
        else:
            assert np.array_equal(d0[n], d1[n]), n


@pytest.mark.parametrize("image", [32, 64])
def test_bnorm_writes_conv_dy_grid(image):
    """conv -> bnorm (-> relu) backward (VGG-16-bn): the bnorm backward writes
    its producer conv's dy grid and bias partials (bnorm_backward_grid), the
    conv's backward skips its dy transform, and the conv output's derivative
    is computed on request; the fused bnorm -> relu forward stores only
    relu(y), y being recomputed from x on request (bn_lazy_y), and when the
    relu output feeds only a conv it goes straight into that conv's x grid
    (producer_grid), the HWCN relu output recomputed on request.  Every value
    and derivative is bit-identical to
    the unfused engine except the conv bias gradients (mathematically zero in
    front of a bnorm; 32-pixel float partials in another fixed order): 1e-5 of
    the largest filter gradient."""
    from paper_1412_4564_b200 import nets
    net = nets.vgg16_bn(batch=2, image=image)
    out = []
    for on in (True, False):
        g = device_graph(net, "tf32")
        g.set_option("bn_grid", on)
        g.set_option("bn_lazy_y", on)
        g.set_option("producer_grid", on)
        for k, v in {**net.init_params(), **net.init_inputs()}.items():
            g.set(k, v)
        g.forward()
        l0 = g.hd.launches
        g.backward("objective")
        launches = g.hd.launches - l0
        names = set(net.inputs) | {p[0] for p in net.params} | \
            {o for layer in net.layers for o in layer[3]}
        out.append(({n: g.get(n) for n in sorted(names)},
                    {n: g.get(n, deriv=True) for n in sorted(names) if n != "label"}, launches))
    (v0, d0, l0), (v1, d1, l1) = out
    assert l0 < l1, (l0, l1)
    for n in v1:
        assert np.array_equal(v0[n], v1[n]), n
    for n in d1:
        if n.startswith("conv") and n.endswith("b"):
            scale = np.abs(d1[n[:-1] + "f"]).max()
            assert np.abs(d0[n] - d1[n]).max() <= 1e-5 * scale, n
        else:
            assert np.array_equal(d0[n], d1[n]), n


def test_unstored_values_after_trainer_step():
    """Values and derivatives a fusion left unstored (bn_lazy_y, bn_grid,
    producer_grid) are recomputed on request with the parameters of the
    forward they belong to -- also after the trainer's SGD has moved them:
    one training step with every fusion on equals the unfused engine's
    stored tape (every layer output's value and derivative) bit for bit."""
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Trainer
    net = nets.vgg16_bn(batch=2, image=32)
    out = []
    for on in (True, False):
        g = device_graph(net, "tf32")
        for opt in ("bn_grid", "bn_lazy_y", "producer_grid", "dgrad_grid", "lrn_grid"):
            g.set_option(opt, on)
        for k, v in {**net.init_params(), **net.init_inputs()}.items():
            g.set(k, v)
        t = Trainer(g, lr=0.05, momentum=0.9, weight_decay=5e-4)
        t.step()
        names = {o for layer in net.layers for o in layer[3]}
        out.append(({n: g.get(n) for n in sorted(names)},
                    {n: g.get(n, deriv=True) for n in sorted(names)}))
    (v0, d0), (v1, d1) = out
    for n in v1:
        assert np.array_equal(v0[n], v1[n]), n
    for n in d1:
        assert np.array_equal(d0[n], d1[n]), n


@pytest.mark.parametrize("cout,groups,size", [(64, 2, 5), (48, 1, 5), (96, 1, 3), (64, 1, 4)])
def test_lrn_grid_envelope(cout, groups, size, monkeypatch):
    """conv -> relu -> lrn -> pool -> fc on a small image: inside the fused
    kernel's envelope (channels per group a multiple of 32, LRN size 3 or 5)
    the LRN writes the conv's dy grid, outside it the engine falls back; both
    agree with the unfused engine (bias gradients to 1e-5 of the largest)."""
    from paper_1412_4564_b200.nets import Net
    n = Net("lrnchain", 4, 10)
    n.inputs = {"data": (15, 15, 16, 4), "label": (1, 1, 1, 4)}
    x = n.conv("conv1", "data", "c1", 3, 3, 16, cout, pad=(1, 1, 1, 1), groups=groups)
    x = n.relu("relu1", x, "r1")
    x = n.lrn("norm1", x, "n1", size, 1.0, 1e-4, 0.75)
    x = n.pool("pool1", x, "p1", 3, 2)
    x = n.conv("fc", x, "f", 7, 7, cout, 10)
    n.loss(x)
    out = []
    for fuse in (True, False):
        g = device_graph(n, "tf32")
        g.set_option("lrn_grid", fuse)
        for k, v in {**n.init_params(), **n.init_inputs()}.items():
            g.set(k, v)
        g.forward()
        g.backward("objective")
        names = set(n.inputs) | {p[0] for p in n.params} | {o for l in n.layers for o in l[3]}
        out.append({name: g.get(name, deriv=True) for name in sorted(names) if name != "label"})
    for name in out[1]:
        a, b = out[0][name], out[1][name]
        if name == "conv1b":
            assert np.abs(a - b).max() <= 1e-5 * (np.abs(b).max() + 1e-30), name
        else:
            assert np.array_equal(a, b), name


@pytest.mark.parametrize("side,win", [(55, 3), (27, 3), (13, 3), (28, 2), (112, 2)])
@pytest.mark.parametrize("pad", [(0, 0, 0, 0), (0, 1, 0, 1)])
def test_engine_pool_argmax_route_bitexact(pad, side, win):
    """In a graph the max pool records its argmax in the forward and the
    backward routes from it (engine.cu / kernels.cu pool_max3s2_bwd_strip_k:
    SEG 32 / 16 / 8 lane segments at AlexNet's 55 / 27 / 13 planes): dx
    must equal the oracle pool backward (pool.cpp:83-126) of the same dy
    bit for bit, spikes making >= 3 windows share an argmax."""
    from paper_1412_4564_b200.graph import Graph
    if win == 2 and pad != (0, 0, 0, 0):
        pad = (0, 1, 0, 1)  # pads must stay below the window: 2x2 with a clipped last window
    xs, n = (side, side, 4, 3), 3
    r = O.Rng(41)
    x = r.uniform(O.size(xs), -0.01, 0.01).reshape(xs[::-1])
    x[:, :, ::2, ::2] += 1.0 + r.uniform(x[:, :, ::2, ::2].size).reshape(x[:, :, ::2, ::2].shape)
    x = x.ravel()
    pg = (win, win, 2, 2, *pad, 0)
    _, ps = O.pool_forward(x, xs, pg)
    g = Graph(math="fp32")
    g.add_input("x", xs)
    g.add_input("label", (1, 1, 1, n))
    g.add_layer("pool", "pool1", ["x"], ["p1"], list(pg))
    # average the pooled map to 1x1 so every window gets a gradient
    g.add_layer("pool", "pool2", ["p1"], ["p2"], [ps[0], ps[1], 1, 1, 0, 0, 0, 0, 1])
    g.add_layer("loss", "loss", ["p2", "label"], ["objective"], [])
    g.finalize()
    g.set("x", x)
    g.set("label", np.array([1, 3, 2], np.float32))
    g.forward()
    g.backward("objective")
    dp1 = g.get("p1", deriv=True)
    assert np.abs(dp1).max() > 0
    assert np.array_equal(g.get("x", deriv=True), O.pool_backward(x, xs, pg, dp1))


@pytest.mark.parametrize("side", [55, 27, 29, 61, 63])
def test_pool_forward_special_values(side):
    """The compile-time 3x3/2 max-pool forward (kernels.cu pool_max_fwd_t)
    picks the reference's winner (pool.cpp:49-80: the first strict maximum in
    (column, row) order) under heavy ties, -inf and NaN: the pooled values
    equal the oracle's (NaN where it has NaN), and in a graph the argmax codes
    it records route the backward exactly as the oracle's dx (heavy ties)."""
    from paper_1412_4564_b200 import blocks as B
    from paper_1412_4564_b200.graph import Graph
    xs, n = (side, side, 5, 3), 3
    r = O.Rng(43)
    x = np.floor(r.uniform(O.size(xs), 0.0, 4.0)).astype(np.float32)  # many ties
    m = r.uniform(O.size(xs))
    x[m < 0.05] = -np.inf
    pg = (3, 3, 2, 2, 0, 0, 0, 0, 0)
    geom = B.PoolGeom(3, 3, 2, 2, 0, 0, 0, 0, mode="max")
    xn = x.copy()
    xn[m > 0.97] = np.nan
    yn_ref, ps = O.pool_forward(xn, xs, pg)
    yn = B.pool_forward(B.as_hwcn(torch.from_numpy(xn).cuda(), xs), geom)
    assert np.array_equal(yn.cpu().numpy().ravel(), yn_ref, equal_nan=True)
    assert np.isnan(yn_ref).any()
    g = Graph(math="fp32")
    g.add_input("x", xs)
    g.add_input("label", (1, 1, 1, n))
    g.add_layer("pool", "pool1", ["x"], ["p1"], list(pg))
    g.add_layer("pool", "pool2", ["p1"], ["p2"], [ps[0], ps[1], 1, 1, 0, 0, 0, 0, 1])
    g.add_layer("loss", "loss", ["p2", "label"], ["objective"], [])
    g.finalize()
    xf = np.where(np.isinf(x), np.float32(-1.0), x)  # heavy ties, finite
    g.set("x", xf)
    g.set("label", np.array([1, 3, 2], np.float32))
    g.forward()
    y_ref, _ = O.pool_forward(xf, xs, pg)
    assert np.array_equal(g.get("p1"), y_ref)
    g.backward("objective")
    dp1 = g.get("p1", deriv=True)
    assert np.isfinite(dp1).all()
    assert np.array_equal(g.get("x", deriv=True), O.pool_backward(xf, xs, pg, dp1))


@pytest.mark.parametrize("net_name", ["cifar", "alexnet", "vgg16bn"])
def test_trainer_cuda_graph_replay_matches_eager(net_name):
    """ck_trainer_set_graph: the captured step replays the same deterministic
    kernels, so parameters after 4 steps are bit-identical to eager steps --
    through every fused route of the nets (AlexNet: LRN / dgrad / producer
    grids; VGG: bnorm grid kernels, unstored bnorm values), and the values a
    fusion left unstored are recomputed identically after a replayed step."""
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Trainer
    net = {"cifar": lambda: nets.cifar(batch=8), "alexnet": lambda: nets.alexnet(batch=4),
           "vgg16bn": lambda: nets.vgg16_bn(batch=2, image=32)}[net_name]()
    params, inputs = net.init_params(), net.init_inputs()
    results = []
    for graph_mode in (False, True):
        g = device_graph(net, "tf32")
        for k, v in {**params, **inputs}.items():
            g.set(k, v)
        t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
        t.set_graph(graph_mode)
        before = g.hd.launches
        stream = torch.cuda.Stream()  # graph capture needs a non-default stream
        losses = [t.step(stream=stream.cuda_stream) for _ in range(4)]
        assert g.hd.launches - before > 4 * 10  # replayed launches are still counted
        g.forward()  # (eager) the values of the current parameters, then read them all
        vals = {o: g.get(o) for layer in net.layers for o in layer[3]}
        results.append((losses, {p: g.get(p) for p, _, _ in net.params}, vals))
    (l0, p0, v0), (l1, p1, v1) = results
    assert l0 == l1
    for k in p0:
        assert np.array_equal(p0[k], p1[k]), k
    for k in v0:
        assert np.array_equal(v0[k], v1[k]), k


def test_feeder_bound_inputs_match_copied_inputs():
    """graph.Feeder binds the graph's inputs to two alternating device buffers
    (ck_graph_bind_input; one captured graph per binding): a replayed training
    run over alternating batches is bit-identical to eager steps that copy each
    batch into the graph's own input buffers."""
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Feeder, Trainer
    net = nets.alexnet(batch=4)
    params = net.init_params()
    batches = [net.init_inputs(data_seed=1 + 100 * k, label_seed=3 + 100 * k) for k in range(2)]
    hosts = [{n: torch.from_numpy(np.ascontiguousarray(b[n], np.float32)).pin_memory()
              for n in ("data", "label")} for b in batches]
    steps = 6
    # eager reference: copy each batch in, one step each
    g = device_graph(net, "tf32")
    for k, v in params.items():
        g.set(k, v)
    t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
    ref = []
    for i in range(steps):
        for n, v in batches[i % 2].items():
            g.set(n, v)
        ref.append(t.step())
    ref_params = {p: g.get(p) for p, _, _ in net.params}
    # bound inputs + graph replay (after one eager step, as bench.py does)
    g = device_graph(net, "tf32")
    for k, v in params.items():
        g.set(k, v)
    t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
    t.set_graph(True)
    stream = torch.cuda.Stream()
    feed = Feeder(g, ["data", "label"], stream)
    feed.put(hosts[0])
    for i in range(steps):
        feed.take()
        if i + 1 < steps:
            feed.put(hosts[(i + 1) % 2])
        t.step(want_loss=False, stream=stream.cuda_stream)
        feed.result("objective")
    got = [float(v[0]) for v in feed.collect()]
    feed.unbind()
    assert got == ref
    for p, _, _ in net.params:
        assert np.array_equal(g.get(p), ref_params[p]), p


@pytest.mark.parametrize("graph_mode", [False, True])
def test_trainer_nccl_single_rank(graph_mode):
    """The data-parallel step on a one-rank NCCL communicator (the only
    topology one GPU allows; ck_trainer_init_dp builds it for world 1 too):
    per-layer ncclAllReduce on the comm stream,
    event hand-off, SGD, loss allreduce -- eagerly and captured into a CUDA
    graph -- must equal the plain single-GPU step bit for bit (a sum over one
    rank is the identity)."""
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Trainer
    net = nets.lenet(batch=8)
    params, inputs = net.init_params(), net.init_inputs()
    out = []
    for dp in (False, True):
        g = device_graph(net, "tf32")
        for k, v in {**params, **inputs}.items():
            g.set(k, v)
        t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
        if dp:
            t.init_dp(Trainer.unique_id(), 0, 1)
        t.set_graph(graph_mode)
        stream = torch.cuda.Stream()
        losses = [t.step(stream=stream.cuda_stream) for _ in range(3)]
        if dp:  # the real communicator path ran (engine.cu ck_trainer::done)
            assert t.allreduces >= len(net.params) // 2
        out.append((losses, {p: g.get(p) for p, _, _ in net.params}))
    (l0, p0), (l1, p1) = out
    assert l0 == l1
    for k in p0:
        assert np.array_equal(p0[k], p1[k]), k


def _net(name, batch, inputs, params, layers):
    from paper_1412_4564_b200.nets import Net
    n = Net(name, batch, 10)
    n.inputs = inputs
    n.params = params
    n.layers = layers
    return n


def _graph_vs_oracle(net, params, inputs, math, tol):
    import chain
    import netcheck
    tc = netcheck.tc_passes(net) if math == "tf32" else None
    g = device_graph(net, math)
    for k, v in {**params, **inputs}.items():
        g.set(k, v)
    hd = g.hd
    tc0 = hd.tc_launches
    g.forward()
    g.backward("objective")
    vals, derivs = chain.run(net, params, inputs, tf32=tc if tc else False,
                             gates=_gates(net, g) if tc else None)
    assert abs(g.get("objective")[0] - vals["objective"][0]) <= tol * abs(vals["objective"][0])
    for name in list(inputs) + [p[0] for p in net.params] + \
            [o for layer in net.layers for o in layer[3]]:
        if name.startswith("label") or name.startswith("attr"):
            continue
        assert normwise(g.get(name), vals[name]) < tol, ("value", name)
        if np.abs(derivs[name]).max() > 0:
            assert normwise(g.get(name, deriv=True), derivs[name]) < tol, ("deriv", name)
    return g, hd.tc_launches - tc0


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_dag_fanout_shared_params_sum_split(math):
    """The reference DAG semantics the chain networks never exercise
    (graph.cpp:548-598): a parameter shared by two conv layers
    (its derivative is the SUM of both contributions), a variable read by
    two layers (fan-out: r1 feeds `split` and `sum`), a `split` layer, a
    three-way `sum`, and two loss layers summed into the objective -- so a
    loss layer's projection is a propagated derivative, not the seed (read
    on the device, engine.cu).  Accumulation on the tensor-core path is the
    tcgen05 epilogue's acc=1 (c2 and c3 both add into r1's derivative, c1
    and c2 into W's)."""
    C = 32
    r = O.Rng(77)
    inputs = {"data": r.uniform(9 * 9 * C * 3), "label": r.labels(3, 10)}
    params = {"W": r.normal(3 * 3 * C * C, 0.08), "b1": r.uniform(C, -0.1, 0.1),
              "b2": r.uniform(C, -0.1, 0.1), "V": r.normal(3 * 3 * C * C, 0.08),
              "F": r.normal(4 * 4 * C * 10, 0.2), "bF": np.zeros(10, np.float32)}
    pad = [1, 1, 1, 1, 1, 1, 1]
    net = _net("dag", 3, {"data": (9, 9, C, 3), "label": (1, 1, 1, 3)},
               [("W", (3, 3, C, C), "normal"), ("b1", (1, 1, C, 1), "zeros"),
                ("b2", (1, 1, C, 1), "zeros"), ("V", (3, 3, C, C), "normal"),
                ("F", (4, 4, C, 10), "normal"), ("bF", (1, 1, 10, 1), "zeros")],
               [("conv", "c1", ["data", "W", "b1"], ["x1"], pad),
                ("relu", "r1", ["x1"], ["y1"], []),
                ("split", "sp", ["y1"], ["s1", "s2"], []),
                ("conv", "c2", ["s1", "W", "b2"], ["x2"], pad),     # W shared with c1
                ("conv", "c3", ["s2", "V"], ["x3"], pad),
                ("sum", "u", ["x2", "x3", "y1"], ["u1"], []),       # y1 fans out
                ("spnorm", "sn", ["u1"], ["n1"], [3, 3, 0.5, 0.75]),
                ("pool", "p", ["n1"], ["p1"], [3, 3, 2, 2, 0, 0, 0, 0, 1]),
                ("sigmoid", "sg", ["p1"], ["g1"], []),
                ("conv", "fc", ["g1", "F", "bF"], ["z"], [1, 1, 0, 0, 0, 0, 1]),
                ("softmax", "sm", ["z"], ["pr"], []),
                ("loss", "l1", ["z", "label"], ["o1"], [3]),        # softmaxlog
                ("loss", "l2", ["pr", "label"], ["o2"], [2]),       # log loss of the softmax
                ("sum", "obj", ["o1", "o2"], ["objective"], [])])
    g, tc = _graph_vs_oracle(net, params, inputs, math, 1e-4 if math == "fp32" else 1e-2)
    if math == "tf32":
        assert tc >= 9  # c1, c2, c3 fprop/dgrad/wgrad on tcgen05 (acc=1 epilogues included)


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_graph_extended_kinds(math):
    """bilinear (x and grid derivatives), pdist (x and target derivatives),
    an attribute loss (hinge) and a mshinge loss through the device engine."""
    C = 16
    r = O.Rng(78)
    inputs = {"data": r.uniform(8 * 8 * C * 2), "grid": r.uniform(2 * 6 * 6 * 2, -1.05, 1.05),
              "target": r.uniform(6 * 6 * C * 2),
              "attr": (np.floor(r.uniform(6 * 6 * 2, 0, 3)) - 1).astype(np.float32),
              "label": r.labels(2, 10)}
    params = {"W": r.normal(3 * 3 * C * C, 0.1), "F": r.normal(6 * 6 * C * 10, 0.1)}
    net = _net("ext", 2, {"data": (8, 8, C, 2), "grid": (2, 6, 6, 2), "target": (6, 6, C, 2),
                          "attr": (6, 6, 1, 2), "label": (1, 1, 1, 2)},
               [("W", (3, 3, C, C), "normal"), ("F", (6, 6, C, 10), "normal")],
               [("bilinear", "bl", ["data", "grid"], ["b1"], []),
                ("conv", "c", ["b1", "W"], ["c1"], [1, 1, 1, 1, 1, 1, 1]),
                ("pdist", "pd", ["c1", "target"], ["d1"], [2, 0]),
                ("loss", "l1", ["d1", "attr"], ["o1"], [9]),          # hinge (attribute)
                ("conv", "fc", ["c1", "F"], ["z"], [1, 1, 0, 0, 0, 0, 1]),
                ("loss", "l2", ["z", "label"], ["o2"], [5]),          # mshinge
                ("sum", "obj", ["o1", "o2"], ["objective"], [])])
    _graph_vs_oracle(net, params, inputs, math, 1e-4 if math == "fp32" else 1e-2)


def test_replay_survives_workspace_reallocation():
    """a captured training step holds raw pointers into the
    handle's workspaces; a larger call on the same handle reallocates them.
    The trainer must notice (workspace generation) and re-capture: steps stay
    bit-identical to an eager trainer fed the same batches."""
    from paper_1412_4564_b200 import blocks as B
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Trainer
    net = nets.cifar(batch=8)
    params, inputs = net.init_params(), net.init_inputs()
    runs = []
    for graph_mode in (False, True):
        g = device_graph(net, "tf32")
        for k, v in {**params, **inputs}.items():
            g.set(k, v)
        t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
        t.set_graph(graph_mode)
        stream = torch.cuda.Stream()
        losses = [t.step(stream=stream.cuda_stream) for _ in range(3)]
        # a much larger conv on the same (thread's) handle grows every workspace
        x = B.from_hwcn((64, 64, 64, 16)).uniform_(-1, 1)
        f = B.from_hwcn((5, 5, 64, 64)).uniform_(-0.05, 0.05)
        y = B.conv_forward(x, f, None, B.ConvGeom(2, 2, 2, 2, 2, 2), math="tf32")
        B.conv_backward(x, f, B.ConvGeom(2, 2, 2, 2, 2, 2), torch.ones_like(y), math="tf32")
        torch.cuda.synchronize()
        losses += [t.step(stream=stream.cuda_stream) for _ in range(3)]
        runs.append((losses, {p: g.get(p) for p, _, _ in net.params}))
    (l0, p0), (l1, p1) = runs
    assert l0 == l1
    for k in p0:
        assert np.array_equal(p0[k], p1[k]), k


def test_unreached_parameter_gets_zero_derivative():
    """a parameter whose consumer does not feed the objective has
    the reference's zero derivative (graph.cpp:551-554) -- also when the
    trainer updates it (weight decay only) -- not uninitialised memory."""
    from paper_1412_4564_b200.graph import Graph, Trainer
    g = Graph(math="fp32")
    g.add_input("data", (6, 6, 4, 2))
    g.add_input("label", (1, 1, 1, 2))
    g.add_param("F", (6, 6, 4, 10))
    g.add_param("G", (3, 3, 4, 5))                      # feeds a dead branch
    g.add_layer("conv", "fc", ["data", "F"], ["z"], [1, 1, 0, 0, 0, 0, 1])
    g.add_layer("conv", "side", ["data", "G"], ["s"], [1, 1, 0, 0, 0, 0, 1])
    g.add_layer("loss", "loss", ["z", "label"], ["objective"], [])
    g.finalize()
    r = O.Rng(5)
    g.set("data", r.uniform(6 * 6 * 4 * 2))
    g.set("label", np.array([1, 2], np.float32))
    G0 = r.uniform(3 * 3 * 4 * 5)
    g.set("G", G0)
    g.set("F", r.uniform(6 * 6 * 4 * 10, -0.1, 0.1))
    t = Trainer(g, lr=0.1, momentum=0.0, weight_decay=0.01)
    t.step()
    assert np.all(g.get("G", deriv=True) == 0)
    w_ref, _ = O.sgd_step(G0, np.zeros_like(G0), np.zeros_like(G0), 0.1, 0.0, 0.01)
    assert np.array_equal(g.get("G"), w_ref)
