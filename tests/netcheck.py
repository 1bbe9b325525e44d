"""Layer-by-layer parity of a device DAG evaluation -- TEST INFRASTRUCTURE.

After the device engine (engine.cu) has run forward + backward on a network,
every layer is re-evaluated on the CPU from the DEVICE's own inputs to that
layer (its input values and its output derivative), with the reference's
block functions (oracle/_ref: the convkit sources compiled verbatim,
OpenBLAS float GEMM), and compared with what the device produced:

  * forward:  layer(device inputs)            vs device output value
  * backward: layer_backward(device x, dy)     vs device input derivatives

Because each comparison starts from the device's own tensors, errors do not
compound through the network: every kernel the engine launched for this
exact configuration -- the batch-dependent tile heights, split-K factors,
persistent waves, fused epilogues and LRN->grid writers -- is held to the
block-level tolerance (north star: pooling/ReLU bit-exact, FP32 1e-4
relative, TF32 1e-2 normwise).  Only chain networks (each variable with one
consumer) are supported, which is what nets.py builds.
"""
from __future__ import annotations

import numpy as np

import chain
import fastconv as FC
import oracle as O

TOL = {"fp32": 1e-4, "tf32": 1e-2}
# TF32 passes against the double oracle evaluated on the same TF32-rounded
# operands (chain.tf32_operand): what remains is fp32 accumulation order
TOL_TF32_EMULATED = 1e-4


def rel(a, b):
    """Per-element relative error, denominator floored at 1% of the tensor's
    max (test_gpu_blocks.rel), and 10x the normwise error."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = 1e-2 * np.max(np.abs(b)) + 1e-30
    elem = float(np.max(np.abs(a - b) / np.maximum(np.abs(a) + np.abs(b), floor)))
    norm = float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
    return max(elem, 10 * norm)


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return max(float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)),
               float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-30)))


def conv_err(a, b, math):
    """Relative error of a contraction: normwise (max(||a-b||/||b||,
    max|a-b|/max|b|)).  At b=256 a weight gradient sums 186k products per
    element; element-by-element relative error of cancelled sums is not a
    property of either implementation (the float reference itself misses the
    double oracle by 1e-4 there), so FP32 is held to 1e-4 normwise."""
    return normwise(a, b)


def check_layers(net, g, math, report=None, strict=True, tc=None):
    """Compare every layer of `net` evaluated on device graph `g` (forward and
    backward already run).  Returns {(layer, what): error}; asserts.

    Convolutions are checked against the double oracle (oracle/fastconv.py)
    -- exact operands at TOL[math]; in TF32, the passes that ran on tcgen05
    (tc: tc_passes(net)) also against TF32-rounded operands at
    TOL_TF32_EMULATED (keys 'y~', 'dx~', 'df~')."""
    report = {} if report is None else report
    if math == "tf32" and tc is None:
        tc = tc_passes(net)
    shapes = {}
    val, der = {}, {}

    def V(n):
        if n not in val:
            val[n] = g.get(n)
            shapes[n] = g.shape(n)
        return val[n]

    def D(n):
        if n not in der:
            der[n] = g.get(n, deriv=True)
        return der[n]

    def put(key, e, tol):
        report[key] = e
        if strict:
            assert e <= tol, f"{key}: error {e:.3e} > {tol:.1e}"

    def exact(key, a, b):
        report[key] = 0.0 if np.array_equal(a, b) else float(np.abs(a - b).max())
        if strict:
            assert np.array_equal(a, b), f"{key}: not bit-exact"

    for kind, name, ins, outs, p in net.layers:
        x = V(ins[0])
        xs = shapes[ins[0]]
        y = V(outs[0])
        dy = D(outs[0])
        if kind == "conv":
            f, fs = V(ins[1]), shapes[ins[1]]
            b = V(ins[2]) if len(ins) > 2 else None
            yr, _ = FC.conv_forward(x, xs, f, fs, b, p)
            put((name, "y"), conv_err(y, yr, math), TOL[math])
            dxr, dfr, dbr = FC.conv_backward(x, xs, f, fs, p, dy)
            put((name, "dx"), conv_err(D(ins[0]), dxr, math), TOL[math])
            put((name, "df"), conv_err(D(ins[1]), dfr, math), TOL[math])
            if b is not None:
                # db = sum of dy: a plain (fixed-order, double) reduction on both paths
                put((name, "db"), rel(D(ins[2]), dbr), 1e-4)
            if math == "tf32":
                fw, dg, wg = tc[name]
                q = chain.tf32_operand
                if fw:
                    ye, _ = FC.conv_forward(x, xs, f, fs, b, p, q=q)
                    put((name, "y~"), normwise(y, ye), TOL_TF32_EMULATED)
                if dg:
                    dxe, _, _ = FC.conv_backward(x, xs, f, fs, p, dy, (True, False, False), q=q)
                    put((name, "dx~"), normwise(D(ins[0]), dxe), TOL_TF32_EMULATED)
                if wg:
                    _, dfe, _ = FC.conv_backward(x, xs, f, fs, p, dy, (False, True, False), q=q)
                    put((name, "df~"), normwise(D(ins[1]), dfe), TOL_TF32_EMULATED)
        elif kind == "relu":
            exact((name, "y"), y, O.ref_relu(x))
            exact((name, "dx"), D(ins[0]), O.ref_relu(x, dy))
        elif kind == "pool":
            yr, _ = O.ref_pool_forward(x, xs, p)
            exact((name, "y"), y, yr)
            exact((name, "dx"), D(ins[0]), O.ref_pool_backward(x, xs, p, dy))
        elif kind == "lrn":
            n_, k_, a_, b_ = int(p[0]), p[1], p[2], p[3]
            put((name, "y"), rel(y, O.ref_lrn_forward(x, xs, n_, k_, a_, b_)), 1e-4)
            put((name, "dx"), rel(D(ins[0]), O.ref_lrn_backward(x, xs, n_, k_, a_, b_, dy)),
                1e-4)
        elif kind == "bnorm":
            w, b = V(ins[1]), V(ins[2])
            # the double restatement: dw / db are sums over H*W*N (100k+ terms
            # at VGG sizes) that the float reference itself only gets to ~1e-4
            yr, _, _ = O.bnorm_forward(x, xs, w, b, p[0])
            put((name, "y"), rel(y, yr), 1e-4)
            dxr, dwr, dbr = O.bnorm_backward(x, xs, w, b, p[0], dy)
            put((name, "dx"), rel(D(ins[0]), dxr), 1e-4)
            put((name, "dw"), rel(D(ins[1]), dwr), 1e-4)
            put((name, "db"), rel(D(ins[2]), dbr), 1e-4)
        elif kind == "loss":
            lab, ls = V(ins[1]), shapes[ins[1]]
            lr = O.ref_loss_forward(x, xs, lab, ls)
            put((name, "y"), abs(float(y[0]) - lr) / abs(lr), 1e-5)
            put((name, "dx"), rel(D(ins[0]), O.ref_loss_backward(x, xs, lab, ls, p=float(dy[0]))),
                1e-4)
        else:
            raise ValueError(kind)
    return report


def format_report(report):
    worst = {}
    for (layer, what), e in report.items():
        worst[f"{layer}.{what}"] = e
    return ", ".join(f"{k}={v:.1e}" for k, v in worst.items())


def tc_passes(net):
    """{conv layer: (fprop, dgrad, wgrad) ran on tcgen05} for a net's conv
    layers in TF32, measured with the handle's tensor-core launch counter on
    batch-1 copies of each layer's shapes (the envelope does not depend on
    the batch)."""
    import torch

    from paper_1412_4564_b200 import blocks as B
    out = {}
    hd = B.handle()
    for name, xs, fs, p in net.conv_layers():
        xs1 = (xs[0], xs[1], xs[2], 1)
        x = B.from_hwcn(xs1, fill=0.5)
        f = B.from_hwcn(tuple(fs), fill=0.01)
        g = B.ConvGeom(*p)
        ys = B.conv_output_shape(xs1, tuple(fs), g)
        dy = B.from_hwcn(ys, fill=1.0)
        res = []
        for want in ((True, False, False), (False, True, False)):
            t0 = hd.tc_launches
            B.conv_backward(x, f, g, dy, want_dx=want[0], want_df=want[1], want_db=False)
            res.append(hd.tc_launches > t0)
        t0 = hd.tc_launches
        B.conv_forward(x, f, None, g)
        torch.cuda.synchronize()
        out[name] = (hd.tc_launches > t0, res[0], res[1])
    return out
