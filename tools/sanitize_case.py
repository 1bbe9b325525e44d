"""Small workloads for compute-sanitizer (memcheck / synccheck / racecheck):
every tcgen05 GEMM path (stride-1 grid fprop/dgrad/wgrad, space-to-depth,
FC, small channels, convt), pooling, LRN (incl. the dy-grid writer), bnorm,
the extended blocks, and two captured training steps of a small AlexNet.
Run: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_1412_4564_b200 import blocks as B  # noqa: E402
from paper_1412_4564_b200 import nets  # noqa: E402
from paper_1412_4564_b200.graph import Graph, Trainer  # noqa: E402


def rnd(shape, s=1.0):
    return B.from_hwcn(shape).uniform_(-s, s)


def main():
    cases = [((13, 13, 64, 2), (3, 3, 64, 96), (1, 1, 1, 1, 1, 1, 1)),
             ((27, 27, 96, 2), (5, 5, 48, 64), (1, 1, 2, 2, 2, 2, 2)),
             ((35, 35, 3, 2), (11, 11, 3, 32), (4, 4, 0, 0, 0, 0, 1)),
             ((6, 6, 64, 3), (6, 6, 64, 40), (1, 1, 0, 0, 0, 0, 1)),
             ((16, 16, 3, 2), (3, 3, 3, 16), (1, 1, 1, 1, 1, 1, 1))]
    for xs, fs, g in cases:
        x, f = rnd(xs), rnd(fs, 0.1)
        geom = B.ConvGeom(*g)
        y = B.conv_forward(x, f, torch.zeros(fs[3], device="cuda"), geom, math="tf32")
        B.conv_backward(x, f, geom, torch.ones_like(y), math="tf32")
    x, f = rnd((7, 6, 64, 2)), rnd((4, 4, 64, 32), 0.1)
    cg = B.ConvTransposeGeom(2, 2, 0, 0, 0, 0)
    y = B.convt_forward(x, f, cg)
    B.convt_backward(x, f, cg, torch.ones_like(y))
    x = rnd((27, 27, 8, 3))
    for pg in (B.PoolGeom(3, 3, 2, 2, 0, 1, 0, 1), B.PoolGeom(2, 2, 2, 2, 0, 0, 0, 0)):
        y = B.pool_forward(x[:, :, :26, :26].contiguous() if pg.window_h == 2 else x, pg)
    lp = B.LrnParams(5, 1.0, 2e-5, 0.75)
    x = rnd((13, 13, 96, 2))
    B.lrn_backward(x, lp, B.lrn_forward(x, lp))
    w, b = torch.ones(96, device="cuda"), torch.zeros(96, device="cuda")
    y, m = B.bnorm_forward(x, w, b)
    B.bnorm_backward(x, w, b, 1e-5, y)
    B.softmax_backward(B.softmax_forward(x), x)
    B.spnorm_backward(x, B.SpnormParams(3, 3, 0.5, 0.75), x)
    grid = rnd((2, 9, 9, 2), 1.1)
    yb = B.bilinear_forward(x, grid)
    B.bilinear_backward(x, grid, yb)
    net = nets.alexnet(batch=2)
    gr = Graph(math="tf32")
    net.build(gr)
    gr.finalize()
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        gr.set(k, v)
    tr = Trainer(gr, lr=0.001)
    tr.set_graph(True)
    st = torch.cuda.Stream()
    for _ in range(3):
        tr.step(stream=st.cuda_stream)
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
