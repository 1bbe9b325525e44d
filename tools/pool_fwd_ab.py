"""Time the 3x3/2 max-pool forward (CUDA events) at AlexNet's pool1 / pool2 / pool5
shapes, b=256, through the block API, with the achieved HBM rate (x read + y write).
Used for the round-2 A/B of a column-strip forward (rejected list);
pass --lib to time a variant library."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--lib" in sys.argv:
    from paper_1412_4564_b200 import _lib
    _lib.LIB_PATH = sys.argv[sys.argv.index("--lib") + 1]
import torch
from paper_1412_4564_b200 import blocks as B
geom = B.PoolGeom(3, 3, 2, 2, 0, 0, 0, 0, mode="max")
for name, xs in (("pool1", (55, 55, 96, 256)), ("pool2", (27, 27, 256, 256)),
                 ("pool5", (13, 13, 256, 256))):
    x = B.from_hwcn(xs).uniform_(-1, 1)
    y = B.pool_forward(x, geom)
    for _ in range(3):
        B.pool_forward(x, geom)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 50
    e0.record()
    for _ in range(reps):
        B.pool_forward(x, geom)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = 4 * (x.numel() + y.numel())
    print(f"{name} {ms * 1e3:7.1f} us  {byts / ms / 1e6:6.0f} GB/s", flush=True)
