"""Isolate the conv wgrad (shifted-window) TC kernel."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import oracle as O
from paper_1412_4564_b200 import blocks as B
cases = [((8, 8, 32, 1), (3, 3, 32, 32), (1, 1, 1, 1, 1, 1, 1)),
         ((13, 13, 64, 2), (3, 3, 64, 128), (1, 1, 1, 1, 1, 1, 1)),
         ((27, 27, 96, 2), (5, 5, 48, 256), (1, 1, 2, 2, 2, 2, 2))]
for xs, fs, g in cases:
    r = O.Rng(5)
    x, f = r.uniform(O.size(xs)), r.uniform(O.size(fs), -0.1, 0.1)
    _, ys = O.conv_forward(x, xs, f, fs, None, g)
    dy = r.uniform(O.size(ys))
    _, df_ref, _ = O.conv_backward(x, xs, f, fs, g, dy, want=(False, True, False))
    dev = lambda a, s: B.as_hwcn(torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda(), s)
    df = torch.zeros_like(dev(f, fs))
    try:
        B.conv_backward(dev(x, xs), dev(f, fs), B.ConvGeom(*g), dev(dy, ys), math="tf32",
                        out=(None, df, None))
        torch.cuda.synchronize()
        d = df.cpu().numpy().ravel()
        print(xs, fs, "err", float(np.abs(d - df_ref).max() / np.abs(df_ref).max()), flush=True)
    except Exception as e:
        print(xs, fs, "FAILED", e, flush=True)
        break
