"""Where does the device TF32 network diverge from the TF32-operand oracle?
Prints value / derivative normwise differences per variable in layer order."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import chain  # noqa: E402
import netcheck  # noqa: E402
from paper_1412_4564_b200 import nets  # noqa: E402
from paper_1412_4564_b200.graph import Graph  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "alexnet"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kw = {"image": 64} if name == "vgg16bn" else {}
net = nets.NETS[name](batch=batch, **kw)
params, inputs = net.init_params(), net.init_inputs()
if name == "vgg16bn":
    params = {k: (v * 20 if k.endswith("f") else v) for k, v in params.items()}
tc = netcheck.tc_passes(net)
print("tc passes:", tc)
vals, derivs = chain.run(net, params, inputs, tf32=tc)
g = Graph(math="tf32")
net.build(g)
g.finalize()
for k, v in {**params, **inputs}.items():
    g.set(k, v)
g.forward()
g.backward("objective")
for kind, lname, ins, outs, p in net.layers:
    o = outs[0]
    v, d = g.get(o), g.get(o, deriv=True)
    dv = netcheck.normwise(v, vals[o])
    dd = netcheck.normwise(d, derivs[o]) if np.abs(derivs[o]).max() > 0 else 0
    extra = ""
    if kind == "relu":
        x = vals[ins[0]]
        xd = g.get(ins[0])
        flips = int(((x > 0) != (xd > 0)).sum())
        near = float(np.sort(np.abs(x[x != 0]))[:3].max()) if (x != 0).any() else 0
        extra = f" relu flips {flips}/{x.size} zeros(oracle)={int((x == 0).sum())} zeros(dev)={int((xd == 0).sum())}"
    print(f"{lname:8s} {kind:6s} value {dv:.2e}  deriv {dd:.2e}{extra}")
for pn, _, _ in net.params:
    print(f"param {pn:8s} deriv {netcheck.normwise(g.get(pn, deriv=True), derivs[pn]):.2e}")
