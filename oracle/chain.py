"""Network-level oracle -- TEST INFRASTRUCTURE ONLY.

Evaluates a layer list (paper_1412_4564_b200.nets.Net.layers, declared in
dependency order) with the C / numpy restatements of the blocks, following
the reference DAG engine's semantics (graph.cpp:494-598): forward in
declaration order keeping every value, backward seeded with d(objective)=1
in reverse order, derivs[in] += d for every input slot -- so fan-out
(a variable read by several layers), shared parameters, `sum` and `split`
layers accumulate exactly as the reference does.  Conv/LRN/bnorm/loss run in
double, pool/relu in float (their reference precision).

tf32 = {conv layer: (fprop, dgrad, wgrad)} evaluates those convolution
passes on operands rounded to TF32 (the 10-bit-mantissa values the tensor
cores multiply, see tf32_operand) and accumulates in double -- the
arithmetic the CK_MATH_TF32 path performs where its tcgen05 kernels run
(tests/netcheck.tc_passes) -- so the device result can be held to a
tolerance that does not depend on how far TF32 rounding drifts a deep
network.  tf32=True rounds every pass.
"""
from __future__ import annotations

import numpy as np

import ext as E
import oracle as O

TF32_MODE = "rz"  # set by tests/test_gpu_tf32_mode.py's measurement


def tf32_operand(a, mode=None):
    """fp32 -> the TF32 value an MMA multiplies: 'rz' drops the low 13
    mantissa bits (round toward zero), 'rn' rounds to nearest even."""
    mode = mode or TF32_MODE
    a = np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32))
    u = a.view(np.uint32).copy()
    if mode == "rn":
        lsb = (u >> np.uint32(13)) & np.uint32(1)
        u = u + np.uint32(0xFFF) + lsb
    u &= np.uint32(0xFFFFE000)
    return u.view(np.float32).astype(np.float64)


def run(net, params: dict, inputs: dict, backward=True, tf32=False, gates=None):
    """gates = {var: values} routes the backward of the ReLU / max-pool layers
    reading `var` by the given values' signs / window maxima instead of the
    oracle's own: a comparison that holds the device's discrete routing
    fixed (each of its decisions is checked bit-exactly, layer by layer, in
    tests/netcheck.py) so the continuous arithmetic around it can be bounded."""
    gates = gates or {}
    shapes = dict(net.inputs)
    for name, shape, _ in net.params:
        shapes[name] = tuple(shape)
    vals = {k: np.asarray(v, np.float64) for k, v in {**params, **inputs}.items()}
    ident = (lambda a: a)

    def q_for(name, k):
        if tf32 is True or (tf32 and tf32.get(name, (False,) * 3)[k]):
            return tf32_operand
        return ident
    for kind, name, ins, outs, p in net.layers:
        x, xs = vals[ins[0]], shapes[ins[0]]
        if kind == "conv":
            b = vals[ins[2]] if len(ins) > 2 else None
            q = q_for(name, 0)
            y, ys = O.conv_forward(q(x), xs, q(vals[ins[1]]), shapes[ins[1]], b, p)
        elif kind == "relu":
            y, ys = O.relu_forward(x).astype(np.float64), xs
        elif kind == "pool":
            y, ys = O.pool_forward(x, xs, p)
            y = y.astype(np.float64)
        elif kind == "lrn":
            y, ys = O.lrn_forward(x, xs, int(p[0]), p[1], p[2], p[3]), xs
        elif kind == "bnorm":
            y, _, _ = O.bnorm_forward(x, xs, vals[ins[1]], vals[ins[2]], p[0])
            ys = xs
        elif kind == "loss":
            lk = int(p[0]) if len(p) else 3
            w = vals[ins[2]] if len(ins) > 2 else None
            y = np.array([E.loss_forward(x, xs, vals[ins[1]], shapes[ins[1]], w, lk,
                                         top_k=int(p[1]) if len(p) > 1 else 5,
                                         threshold=p[2] if len(p) > 2 else 0.0)])
            ys = (1, 1, 1, 1)
        elif kind == "sum":
            y, ys = sum(vals[i] for i in ins), xs
        elif kind == "split":
            for o in outs:
                vals[o], shapes[o] = x.copy(), xs
            continue
        elif kind == "sigmoid":
            y, ys = E.sigmoid_forward(x), xs
        elif kind == "softmax":
            y, ys = E.softmax_forward(x, xs), xs
        elif kind == "spnorm":
            y, ys = E.spnorm_forward(x, xs, int(p[0]), int(p[1]), p[2], p[3]), xs
        elif kind == "bilinear":
            y, ys = E.bilinear_forward(x, xs, vals[ins[1]], shapes[ins[1]])
        elif kind == "pdist":
            pp, nr = (p[0] if len(p) else 2.0), (len(p) > 1 and p[1] != 0)
            y, ys = E.pdist_forward(x, vals[ins[1]], xs, pp, nr), (xs[0], xs[1], 1, xs[3])
        else:
            raise ValueError(kind)
        vals[outs[0]], shapes[outs[0]] = y, ys
    if not backward:
        return vals, {}
    derivs = {k: np.zeros(v.size) for k, v in vals.items()}
    derivs["objective"][0] = 1.0
    for kind, name, ins, outs, p in reversed(net.layers):
        dy = derivs[outs[0]]
        if not any(np.any(derivs[o]) for o in outs) and kind != "loss":
            continue  # no live projection: the reference adds zeros
        x, xs = vals[ins[0]], shapes[ins[0]]
        if kind == "conv":
            f, fs = vals[ins[1]], shapes[ins[1]]
            q = q_for(name, 1)
            dx, _, _ = O.conv_backward(x, xs, q(f), fs, p, q(dy), (True, False, False))
            q = q_for(name, 2)
            _, df, _ = O.conv_backward(q(x), xs, f, fs, p, q(dy), (False, True, False))
            derivs[ins[0]] += dx
            derivs[ins[1]] += df
            if len(ins) > 2:
                derivs[ins[2]] += O.conv_backward(x, xs, f, fs, p, dy, (False, False, True))[2]
        elif kind == "relu":
            gx = gates.get(ins[0], x)
            derivs[ins[0]] += np.where(gx > 0, dy, 0.0)
        elif kind == "pool":
            gx = gates.get(ins[0], x) if p[8] == 0 else x
            derivs[ins[0]] += O.pool_backward(gx, xs, p, dy).astype(np.float64)
        elif kind == "lrn":
            derivs[ins[0]] += O.lrn_backward(x, xs, int(p[0]), p[1], p[2], p[3], dy)
        elif kind == "bnorm":
            dx, dw, db = O.bnorm_backward(x, xs, vals[ins[1]], vals[ins[2]], p[0], dy)
            derivs[ins[0]] += dx
            derivs[ins[1]] += dw
            derivs[ins[2]] += db
        elif kind == "loss":
            lk = int(p[0]) if len(p) else 3
            w = vals[ins[2]] if len(ins) > 2 else None
            derivs[ins[0]] += E.loss_backward(x, xs, vals[ins[1]], shapes[ins[1]], w, lk, dy[0])
        elif kind == "sum":
            for i in ins:
                derivs[i] += dy
        elif kind == "split":
            for o in outs:
                derivs[ins[0]] += derivs[o]
        elif kind == "sigmoid":
            derivs[ins[0]] += E.sigmoid_backward(vals[outs[0]], dy)
        elif kind == "softmax":
            derivs[ins[0]] += E.softmax_backward(vals[outs[0]], xs, dy)
        elif kind == "spnorm":
            derivs[ins[0]] += E.spnorm_backward(x, xs, int(p[0]), int(p[1]), p[2], p[3], dy)
        elif kind == "bilinear":
            dx, dg = E.bilinear_backward(x, xs, vals[ins[1]], shapes[ins[1]], dy)
            derivs[ins[0]] += dx
            derivs[ins[1]] += dg
        elif kind == "pdist":
            pp, nr = (p[0] if len(p) else 2.0), (len(p) > 1 and p[1] != 0)
            dx, dt = E.pdist_backward(x, vals[ins[1]], xs, pp, nr, dy)
            derivs[ins[0]] += dx
            derivs[ins[1]] += dt
    return vals, derivs
