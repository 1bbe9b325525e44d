"""Layer-by-layer drift of TF32 vs FP32 on VGG16-bn (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1412_4564_b200 import nets
from paper_1412_4564_b200.graph import Graph
net = nets.vgg16_bn(batch=2, image=64)
params = {k: (v * 20 if k.endswith("f") else v) for k, v in net.init_params().items()}
inputs = net.init_inputs()
gs = {}
for math in ("fp32", "tf32"):
    g = Graph(math=math); net.build(g); g.finalize()
    for k, v in {**params, **inputs}.items(): g.set(k, v)
    g.forward(); g.backward("objective"); torch.cuda.synchronize()
    gs[math] = g
def nerr(a, b): return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
for kind, name, ins, outs, p in net.layers:
    o = outs[0]
    print(f"{name:10s} val {nerr(gs['tf32'].get(o), gs['fp32'].get(o)):.2e}  "
          f"dval {nerr(gs['tf32'].get(o, True), gs['fp32'].get(o, True)):.2e}")
for pname in ("conv1f", "conv2f", "conv13f", "fc6f"):
    print(pname, nerr(gs['tf32'].get(pname, True), gs['fp32'].get(pname, True)))
