"""Time (CUDA events) AlexNet's non-conv blocks at batch 256 through the C ABI
and report effective HBM bandwidth (algorithmic bytes / time)."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1412_4564_b200 import blocks as B

ap = argparse.ArgumentParser()
ap.add_argument("--only", default="")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
N = 256
LRN = B.LrnParams(5, 1.0, 1e-4, 0.75)
P = B.PoolGeom(3, 3, 2, 2)
cases = []
for name, shape in [("1", (55, 55, 96)), ("2", (27, 27, 256)), ("5", (13, 13, 256))]:
    xs = shape + (N,)
    x = B.from_hwcn(xs).uniform_(-1, 1)
    n = x.numel() * 4
    ys = B.pool_output_shape(xs, P)
    dyp = torch.randn(ys[3], ys[2], ys[1], ys[0], device="cuda")
    ny = dyp.numel() * 4
    dy = torch.randn_like(x)
    cases += [
        (f"pool{name} fwd", lambda x=x: B.pool_forward(x, P), n + ny),
        (f"pool{name} bwd", lambda x=x, d=dyp: B.pool_backward(x, P, d), 2 * n + ny),
        (f"relu{name} fwd", lambda x=x: B.relu_forward(x), 2 * n),
        (f"relu{name} bwd", lambda x=x, d=dy: B.relu_backward(x, d), 3 * n),
    ]
    if name != "5":
        cases += [
            (f"norm{name} fwd", lambda x=x: B.lrn_forward(x, LRN), 2 * n),
            (f"norm{name} bwd", lambda x=x, d=dy: B.lrn_backward(x, LRN, d), 3 * n),
        ]
for label, fn, nbytes in cases:
    if a.only and a.only not in label:
        continue
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{label:12s} {ms:7.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s", flush=True)
