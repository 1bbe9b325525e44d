"""First-layer (few input channels) convs: tensor-core (tf32) vs SIMT (fp32) time per pass."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1412_4564_b200 import blocks as B
CASES = {"lenet1": ((28, 28, 1, 100), (5, 5, 1, 20), (1, 1, 0, 0, 0, 0, 1)),
         "cifar1": ((32, 32, 3, 128), (5, 5, 3, 32), (1, 1, 2, 2, 2, 2, 1)),
         "vgg1": ((224, 224, 3, 64), (3, 3, 3, 64), (1, 1, 1, 1, 1, 1, 1))}
for name, (xs, fs, g) in CASES.items():
    x = B.from_hwcn(xs).uniform_(-1, 1)
    f = B.from_hwcn(fs).uniform_(-0.1, 0.1)
    geom = B.ConvGeom(*g)
    y = B.conv_forward(x, f, None, geom)
    dy = torch.randn_like(y)
    dx, df = torch.empty_like(x), torch.empty_like(f)
    out = []
    for math in ("tf32", "fp32"):
        for p in "fdw":
            def run():
                if p == "f":
                    B.conv_forward(x, f, None, geom, math=math)
                elif p == "d":
                    B.conv_backward(x, f, geom, dy, out=(dx, None, None), math=math)
                else:
                    B.conv_backward(x, f, geom, dy, out=(None, df, None), math=math)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(10):
                run()
            e1.record()
            torch.cuda.synchronize()
            out.append(f"{math}.{p} {e0.elapsed_time(e1) / 10:.3f}")
    print(name, "  ".join(out), flush=True)
