"""Network-level oracle -- TEST INFRASTRUCTURE ONLY.

Evaluates a layer list (paper_1412_4564_b200.nets.Net.layers) with the C
restatement's blocks, following the reference DAG engine's semantics
(graph.cpp:494-598): forward in firing order keeping every value, backward
seeded with d(objective)=1 in reverse order, derivs[in] += d.  Conv/LRN/
bnorm/loss run in double, pool/relu in float (their reference precision).
"""
from __future__ import annotations

import numpy as np

import oracle as O


def run(net, params: dict, inputs: dict, backward=True):
    shapes = dict(net.inputs)
    for name, shape, _ in net.params:
        shapes[name] = tuple(shape)
    vals = {k: np.asarray(v, np.float64) for k, v in {**params, **inputs}.items()}
    for kind, name, ins, outs, p in net.layers:
        x, xs = vals[ins[0]], shapes[ins[0]]
        if kind == "conv":
            b = vals[ins[2]] if len(ins) > 2 else None
            y, ys = O.conv_forward(x, xs, vals[ins[1]], shapes[ins[1]], b, p)
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
            y = np.array([O.loss_forward(x, xs, vals[ins[1]], shapes[ins[1]])])
            ys = (1, 1, 1, 1)
        else:
            raise ValueError(kind)
        vals[outs[0]], shapes[outs[0]] = y, ys
    if not backward:
        return vals, {}
    derivs = {k: np.zeros(v.size) for k, v in vals.items()}
    derivs["objective"][0] = 1.0
    for kind, name, ins, outs, p in reversed(net.layers):
        dy = derivs[outs[0]]
        x, xs = vals[ins[0]], shapes[ins[0]]
        if kind == "conv":
            dx, df, db = O.conv_backward(x, xs, vals[ins[1]], shapes[ins[1]], p, dy)
            derivs[ins[0]] += dx
            derivs[ins[1]] += df
            if len(ins) > 2:
                derivs[ins[2]] += db
        elif kind == "relu":
            derivs[ins[0]] += np.where(x > 0, dy, 0.0)
        elif kind == "pool":
            derivs[ins[0]] += O.pool_backward(x, xs, p, dy).astype(np.float64)
        elif kind == "lrn":
            derivs[ins[0]] += O.lrn_backward(x, xs, int(p[0]), p[1], p[2], p[3], dy)
        elif kind == "bnorm":
            dx, dw, db = O.bnorm_backward(x, xs, vals[ins[1]], vals[ins[2]], p[0], dy)
            derivs[ins[0]] += dx
            derivs[ins[1]] += dw
            derivs[ins[2]] += db
        elif kind == "loss":
            derivs[ins[0]] += O.softmaxlog_backward(x, xs, vals[ins[1]], shapes[ins[1]], None,
                                                    dy[0])
    return vals, derivs
