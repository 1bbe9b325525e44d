"""A/B of one training step between library builds (e.g. build.py variants):
    python tools/ab_step.py [--lib path] [--net alexnet] [--steps 30]
Prints ms/step of the CUDA-graph-replayed step (CUDA events)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default="")
ap.add_argument("--net", default="alexnet")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--option", action="append", default=[], help="engine option name=value")
ap.add_argument("--layers", default="", help="also print these layers' eager fwd/bwd ms (5-step mean)")
a = ap.parse_args()
if a.lib:
    from paper_1412_4564_b200 import _lib
    _lib.LIB_PATH = a.lib
import torch  # noqa: E402

from paper_1412_4564_b200 import nets  # noqa: E402
from paper_1412_4564_b200.graph import Graph, Trainer  # noqa: E402

net = nets.NETS[a.net](batch=a.batch or nets.DEFAULT_BATCH[a.net])
g = Graph(math="tf32")
net.build(g)
g.finalize()
for o in a.option:
    k, v = o.split("=")
    g.set_option(k, int(v))
for k, v in {**net.init_params(), **net.init_inputs()}.items():
    g.set(k, v)
t = Trainer(g, lr=0.01 / net.batch)  # cnn_train: the step is scaled by the batch (sum loss)
t.set_graph(True)
st = torch.cuda.Stream()
for _ in range(5):
    t.step(want_loss=False, stream=st.cuda_stream)
torch.cuda.synchronize()
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st)
    for _ in range(a.steps):
        t.step(want_loss=False, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / a.steps)
print(f"{a.net} {a.lib or 'libck.so'} {' '.join(a.option)}: ms/step "
      + " ".join(f"{v:.3f}" for v in res))
if a.layers:
    want = a.layers.split(",")
    acc = {}
    g.set_profiling(True)
    t.set_graph(False)
    for _ in range(5):
        t.step(want_loss=False, stream=st.cuda_stream)
        torch.cuda.synchronize()
        for n, f, b in g.layer_times():
            if n in want:
                acc.setdefault(n, []).append((f, b))
    g.set_profiling(False)
    print("  " + "  ".join(f"{n} fwd {sum(v[0] for v in acc[n]) / len(acc[n]):.4f} bwd "
                          f"{sum(v[1] for v in acc[n]) / len(acc[n]):.4f}" for n in want if n in acc))
