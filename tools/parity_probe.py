"""Print observed parity errors (not a test): network-level (device engine vs
oracle chain / verbatim reference graph) and layer-level (tests/netcheck.py)
for the BASELINE networks.  Run on the GPU box:
    python tools/parity_probe.py [--full]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import chain  # noqa: E402
import netcheck  # noqa: E402
import oracle as O  # noqa: E402
from paper_1412_4564_b200 import nets  # noqa: E402
from paper_1412_4564_b200.graph import Graph  # noqa: E402


def dev_graph(net, math, params, inputs):
    g = Graph(math=math)
    net.build(g)
    g.finalize()
    for k, v in {**params, **inputs}.items():
        g.set(k, v)
    g.forward()
    g.backward("objective")
    return g


def net_errors(net, g, derivs, loss_ref):
    out = {"loss": abs(float(g.get("objective")[0]) - loss_ref) / abs(loss_ref)}
    for pname, _, _ in net.params:
        ref = derivs[pname]
        if np.abs(ref).max() == 0:
            continue
        out[pname] = netcheck.normwise(g.get(pname, deriv=True), ref)
    out["data"] = netcheck.normwise(g.get("data", deriv=True), derivs["data"])
    return out


def main():
    full = "--full" in sys.argv
    for name, batch, kw in [("lenet", 4, {}), ("cifar", 4, {}), ("alexnet", 2, {}),
                            ("vgg16bn", 2, {"image": 64})]:
        net = nets.NETS[name](batch=batch, **kw)
        params, inputs = net.init_params(), net.init_inputs()
        if name == "vgg16bn":
            params = {k: (v * 20 if k.endswith("f") else v) for k, v in params.items()}
        vals, derivs = chain.run(net, params, inputs)
        for math in ("fp32", "tf32"):
            g = dev_graph(net, math, params, inputs)
            e = net_errors(net, g, derivs, vals["objective"][0])
            worst = max(v for k, v in e.items() if k != "loss")
            print(f"NET {name} b={batch} {math}: loss {e['loss']:.2e} worst deriv {worst:.2e} | "
                  + " ".join(f"{k}={v:.1e}" for k, v in e.items()), flush=True)
            rep = {}
            try:
                netcheck.check_layers(net, g, math, rep, strict=False)
            except AssertionError as ex:
                print("  FAIL", ex)
            print(f"LAYERS {name} b={batch} {math}: " + netcheck.format_report(rep), flush=True)
    if not full:
        return
    for name, batch in [("alexnet", 256)]:
        net = nets.NETS[name](batch=batch)
        params, inputs = net.init_params(), net.init_inputs()
        t0 = time.time()
        import bench
        rg, _ = bench.ref_graph_for(net)
        rg.run()
        t_ref = time.time() - t0
        for math in ("tf32", "fp32"):
            g = dev_graph(net, math, params, inputs)
            e = {"loss": abs(float(g.get("objective")[0]) - float(rg.get("objective")[0][0]))}
            for pname, _, _ in net.params + [("data", None, None)]:
                ref, _ = rg.get(pname, deriv=True)
                if np.abs(ref).max() == 0:
                    continue
                e[pname] = netcheck.normwise(g.get(pname, deriv=True), ref)
            print(f"NET-REF {name} b={batch} {math} (ref {t_ref:.1f}s): " +
                  " ".join(f"{k}={v:.1e}" for k, v in e.items()), flush=True)
            t0 = time.time()
            rep = {}
            try:
                netcheck.check_layers(net, g, math, rep, strict=False)
            except AssertionError as ex:
                print("  FAIL", ex)
            print(f"LAYERS {name} b={batch} {math} ({time.time() - t0:.1f}s): "
                  + netcheck.format_report(rep), flush=True)


if __name__ == "__main__":
    main()
