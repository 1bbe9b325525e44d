"""Time (CUDA events) one AlexNet conv layer's fprop / dgrad / wgrad through the C ABI."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if "--lib" in sys.argv:  # an explicitly built variant (build.py --experiments)
    from paper_1412_4564_b200 import _lib
    _lib.LIB_PATH = sys.argv[sys.argv.index("--lib") + 1]
from paper_1412_4564_b200 import blocks as B
LAYERS = {
    "conv1": ((227, 227, 3), (11, 11, 3, 96), (4, 4, 0, 0, 0, 0, 1)),
    "conv2": ((27, 27, 96), (5, 5, 48, 256), (1, 1, 2, 2, 2, 2, 2)),
    "conv3": ((13, 13, 256), (3, 3, 256, 384), (1, 1, 1, 1, 1, 1, 1)),
    "conv4": ((13, 13, 384), (3, 3, 192, 384), (1, 1, 1, 1, 1, 1, 2)),
    "conv5": ((13, 13, 384), (3, 3, 192, 256), (1, 1, 1, 1, 1, 1, 2)),
    "fc6": ((6, 6, 256), (6, 6, 256, 4096), (1, 1, 0, 0, 0, 0, 1)),
    "fc7": ((1, 1, 4096), (1, 1, 4096, 4096), (1, 1, 0, 0, 0, 0, 1)),
    "vgg1": ((224, 224, 3), (3, 3, 3, 64), (1, 1, 1, 1, 1, 1, 1)),
    "vgg2": ((224, 224, 64), (3, 3, 64, 64), (1, 1, 1, 1, 1, 1, 1)),
    "vgg4": ((112, 112, 128), (3, 3, 128, 128), (1, 1, 1, 1, 1, 1, 1)),
    "vgg6": ((56, 56, 256), (3, 3, 256, 256), (1, 1, 1, 1, 1, 1, 1)),
}
ap = argparse.ArgumentParser()
ap.add_argument("--layers", default=",".join(LAYERS))
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--passes", default="f,d,w")
ap.add_argument("--lib", default="")
a = ap.parse_args()
for name in a.layers.split(","):
    (H, W, C), fs, g = LAYERS[name]
    xs = (H, W, C, a.batch)
    x = B.from_hwcn(xs).uniform_(-1, 1)
    f = B.from_hwcn(fs).uniform_(-0.1, 0.1)
    geom = B.ConvGeom(*g)
    y = B.conv_forward(x, f, None, geom)
    dy = torch.randn_like(y)
    dx, df = torch.empty_like(x), torch.empty_like(f)
    oh, ow = B.hwcn_shape(y)[:2]
    flop = 2.0 * a.batch * oh * ow * fs[3] * fs[0] * fs[1] * fs[2]
    res = []
    for p in a.passes.split(","):
        def run():
            if p == "f":
                B.conv_forward(x, f, None, geom)
            elif p == "d":
                B.conv_backward(x, f, geom, dy, out=(dx, None, None))
            else:
                B.conv_backward(x, f, geom, dy, out=(None, df, None))
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        res.append(f"{p}: {ms:7.3f} ms {flop / ms / 1e9:6.1f} TF/s")
    print(f"{name:6s} " + "  ".join(res), flush=True)
