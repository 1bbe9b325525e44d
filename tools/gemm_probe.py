"""Plain-GEMM throughput of the tcgen05 kernel: an FC fprop (1x1xK input,
N outputs) at a large batch is y[b, n] = sum_k x[b, k] F[k, n] (OP_TILED_K x2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1412_4564_b200 import blocks as B
for batch, K, N in [(8192, 4096, 4096), (4096, 4096, 4096), (16384, 2048, 2048)]:
    x = B.from_hwcn((1, 1, K, batch)).uniform_(-1, 1)
    f = B.from_hwcn((1, 1, K, N)).uniform_(-0.1, 0.1)
    geom = B.ConvGeom(1, 1, 0, 0, 0, 0, 1)
    for _ in range(2):
        B.conv_forward(x, f, None, geom)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        B.conv_forward(x, f, None, geom)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"gemm M={batch} N={N} K={K}: {ms:.3f} ms {2.0 * batch * N * K / ms / 1e9:.1f} TF/s")
