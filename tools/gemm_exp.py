"""Pure GEMM launch times (ck_set_kernel_profiling) of AlexNet conv layers,
for the CK_TC_EXP experiments: 0 = normal, 1 = no MMAs, 2 = no TMA loads."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1412_4564_b200 import blocks as B
LAYERS = {
    "conv1": ((227, 227, 3), (11, 11, 3, 96), (4, 4, 0, 0, 0, 0, 1)),
    "conv2": ((27, 27, 96), (5, 5, 48, 256), (1, 1, 2, 2, 2, 2, 2)),
    "conv3": ((13, 13, 256), (3, 3, 256, 384), (1, 1, 1, 1, 1, 1, 1)),
    "conv4": ((13, 13, 384), (3, 3, 192, 384), (1, 1, 1, 1, 1, 1, 2)),
    "conv5": ((13, 13, 384), (3, 3, 192, 256), (1, 1, 1, 1, 1, 1, 2)),
}
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--only", default="")
ap.add_argument("--fwd-only", action="store_true")
a = ap.parse_args()
hd = B.handle()
for name, ((H, W, C), fs, g) in LAYERS.items():
    if a.only and name != a.only:
        continue
    x = B.from_hwcn((H, W, C, 256)).uniform_(-1, 1)
    f = B.from_hwcn(fs).uniform_(-0.1, 0.1)
    geom = B.ConvGeom(*g)
    y = B.conv_forward(x, f, None, geom)
    dy = torch.randn_like(y)
    dx, df = torch.empty_like(x), torch.empty_like(f)
    for _ in range(2):
        B.conv_forward(x, f, None, geom)
        if not a.fwd_only:
            B.conv_backward(x, f, geom, dy, out=(dx, df, None))
    torch.cuda.synchronize()
    hd.kernel_profiling(True)
    for _ in range(3):
        B.conv_forward(x, f, None, geom)
        if not a.fwd_only:
            B.conv_backward(x, f, geom, dy, out=(dx, df, None))
    torch.cuda.synchronize()
    prof = hd.kernel_profile()
    hd.kernel_profiling(False)
    agg = {}
    for lab, ms, fl in prof:
        k = lab.split()[0]
        agg.setdefault(k, []).append((ms, fl))
    print(name, "  ".join(f"{k}: {min(m for m, _ in v):.3f} ms {v[0][1] / min(m for m, _ in v) / 1e9:6.1f} TF/s"
                          for k, v in agg.items()), flush=True)
