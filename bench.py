#!/usr/bin/env python
"""AlexNet fwd+bwd training throughput on B200 (BASELINE.json metric).

One step = forward + backward + gradient allreduce (N>1) + SGD of
imagenet-caffe-alex at 256 images per GPU, through the device DAG engine of
libck.so.  Launch: `python bench.py` (N=1) or under torch.distributed.run
with --gpus N (one process per GPU, NCCL).  Rank 0 prints one JSON line.

`--impl reference` times the reference's own CPU implementation (the convkit
sources compiled verbatim into oracle/_ref) on this box's host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AlexNet fwd+bwd images/sec"
UNIT = "images/s"
PUBLISHED = 264.1  # MatConvNet CuDNN v2, 1x Titan Black, batch 256
WORKLOAD = "imagenet-caffe-alex 227x227x3, fwd+bwd+SGD, 256 images/GPU"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--net", default="alexnet")
    p.add_argument("--batch", type=int, default=256)
    p.add_argument("--math", default="tf32", choices=["tf32", "fp32"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="launch every kernel (no CUDA graph)")
    p.add_argument("--profile-layers", action="store_true", help="print per-layer times to stderr")
    # internal: CPU sample run in a subprocess
    p.add_argument("--cpu-sample", type=int, default=0)
    p.add_argument("--cpu-reps", type=int, default=1)
    return p.parse_args()


# ---------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------- CPU reference --

def ref_graph_for(net):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    rg = O.RefGraph()

    class _B:
        def add_input(self, n, sh):
            rg.add_input(n)

        def add_param(self, n, sh):
            rg.add_param(n)

        def add_layer(self, *a):
            rg.add_layer(*a)

    net.build(_B())
    rg.finalize()
    shapes = dict(net.inputs)
    for n, s, _ in net.params:
        shapes[n] = s
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        rg.bind(k, v, shapes[k])
    return rg, O


def cpu_sample_main(args):
    """Child process: time `reps` reference fwd+bwd passes at batch `cpu_sample`."""
    from paper_1412_4564_b200 import nets
    net = nets.NETS[args.net](batch=args.cpu_sample)
    rg, O = ref_graph_for(net)
    rg.run()  # warm
    t0 = time.perf_counter()
    for _ in range(args.cpu_reps):
        rg.run()
    dt = time.perf_counter() - t0
    loss, _ = rg.get("objective")
    print(json.dumps({"seconds": dt, "images": args.cpu_sample * args.cpu_reps,
                      "loss": float(loss[0])}))


def run_cpu_sample(net_name, batch, reps, threads, timeout=900):
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads))
    env.pop("CUDA_VISIBLE_DEVICES", None)
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-sample", str(batch), "--cpu-reps",
           str(reps), "--net", net_name]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def cpu_baseline(net_name):
    """The verbatim reference on this box's host cores, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    batch = 128  # ~10 s of reference CPU work
    res = run_cpu_sample(net_name, batch, 1, threads)
    return {"value": res["images"] / res["seconds"], "unit": UNIT, "cores": threads,
            "kind": "reference",
            "sample": f"1 fwd+bwd of {net_name} at batch {batch} through the reference DAG engine "
                      f"(graph.cpp:494/548), OpenBLAS GEMM with {threads} threads, "
                      f"{res['seconds']:.1f} s", "cpu": cpu_model()}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_main(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_1412_4564_b200 import nets
    threads = os.cpu_count() or 1
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (verbatim reference "
                                                              "build) missing on this box"}))
        return 0
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    batch = 8  # bounded sample per step (~0.7 s each)
    net = nets.NETS[args.net](batch=batch)
    rg, _ = ref_graph_for(net)
    for _ in range(args.warmup):
        rg.run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rg.run()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = batch * args.steps / total
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (xoshiro256**: U[-1,1) data, 0.01 N(0,1) weights, random labels)",
           "impl": "reference",
           "config": {"workload": WORKLOAD + f" (sample: {batch} images per step)",
                      "per_step_batch": batch, "threads": threads},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"{args.steps} steps x fwd+bwd at batch {batch}, reference "
                                      f"convkit sources (oracle/_ref), OpenBLAS {threads} threads",
                            "cpu": cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------- ours --

def main():
    args = parse()
    if args.cpu_sample:
        return cpu_sample_main(args)
    if args.impl == "reference":
        return reference_main(args)

    import numpy as np
    import torch

    from paper_1412_4564_b200 import lib, nets
    from paper_1412_4564_b200.graph import Graph, Trainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    net = nets.NETS[args.net](batch=args.batch)
    g = Graph(math=args.math)
    net.build(g)
    g.finalize()
    for k, v in net.init_params().items():
        g.set(k, v)
    inputs = net.init_inputs(data_seed=1 + rank, label_seed=3 + rank)
    for k, v in inputs.items():
        g.set(k, v)
    # cnn_train scales the step by the batch: the loss is a SUM over images
    tr = Trainer(g, lr=0.01 / args.batch, momentum=0.9, weight_decay=5e-4)
    if world > 1:
        from paper_1412_4564_b200 import dp
        tr.init_dp(dp.share_unique_id(Trainer.unique_id, rank), rank, world)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput -------------------------------------
    # CUDA-graph replay of the step: warm-up step 1 runs eagerly (sizes every
    # workspace), step 2 is captured, the rest (and the timed steps) replay it.
    tr.set_graph(not args.no_graph)
    for _ in range(max(args.warmup, 3)):
        tr.step(want_loss=False, stream=sp)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = g.hd.launches
    with torch.cuda.stream(stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            tr.step(want_loss=False, stream=sp)
        e1.record(stream)
    barrier()
    clk = clocks.stop()
    launches = g.hd.launches - launches0  # total inside the timed region
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = world * args.batch / (ms / 1e3)
    loss = tr.step(want_loss=True, stream=sp)

    # ---- per-layer breakdown + roofline of the dominant kernel ----------
    # One more step with per-layer events and per-launch events around every
    # tensor-core GEMM (ck_set_kernel_profiling), all on the evaluation stream.
    g.set_profiling(True)
    g.hd.kernel_profiling(True)
    tr.step(want_loss=False, stream=sp)
    torch.cuda.synchronize()
    times = g.layer_times()
    kprof = g.hd.kernel_profile()
    g.hd.kernel_profiling(False)
    g.set_profiling(False)
    flops = {}
    for name, xs, fs, p in net.conv_layers():
        s, pt, pb, pl, pr = p[0], p[2], p[3], p[4], p[5]
        oh = (xs[0] + pt + pb - fs[0]) // s + 1
        ow = (xs[1] + pl + pr - fs[1]) // s + 1
        flops[name] = 2.0 * xs[3] * oh * ow * fs[3] * fs[0] * fs[1] * fs[2]
    conv_ms = sum(f + b for n, f, b in times if n in flops)
    step_layers_ms = sum(f + b for _, f, b in times)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    bf16 = peaks.get("bf16_tflops_sustained") or 1400.0
    tf32_peak, peak_src = bf16 / 2.0, ("0.5 x MEASURED_PEAKS.json bf16_tflops_sustained "
                                       "(TF32 = half the bf16 rate)")
    try:  # measured full-chip TF32 MMA rate (tools/shift_probe.cu full), sustained
        tp = json.load(open(os.path.join(ROOT, "profiles", "tf32_peak.json")))
        tf32_peak = tp["tf32_tflops_sustained"]
        peak_src = ("profiles/tf32_peak.json tf32_tflops_sustained: measured full-chip "
                    "tcgen05.mma.kind::tf32 stream, sustained (the kernel runs inside a long step)")
    except (OSError, ValueError, KeyError):
        pass
    if args.math != "tf32":
        tf32_peak, peak_src = 74.0, "FP32 FFMA nominal 148 SM x 128 x 2 x 1.965 GHz"
    if kprof:
        # dominant kernel = the GEMM launch with the largest time in the step
        lab, kms, kfl = max(kprof, key=lambda r: r[1])
        achieved = kfl / (kms / 1e3) / 1e12
        traffic = None
        try:  # dram bytes of this launch from a committed ncu --set full capture
            traffic = json.load(open(os.path.join(ROOT, "profiles", "kernel_traffic.json"))).get(lab)
        except (OSError, ValueError):
            pass
        gemm_ms = sum(r[1] for r in kprof)
        roofline = {"bound": "tensor", "kernel": f"tc_gemm_kernel: {lab}", "achieved": achieved,
                    "peak": tf32_peak, "unit": "TFLOP/s", "frac": achieved / tf32_peak,
                    "traffic": traffic, "peak_source": peak_src, "launch_ms": kms,
                    "algorithmic_flop": kfl,
                    "share_of_step": kms / max(step_layers_ms, 1e-9),
                    "all_gemm": {"achieved": sum(r[2] for r in kprof) / (gemm_ms / 1e3) / 1e12,
                                 "ms": gemm_ms, "launches": len(kprof)},
                    "all_conv_layers": {"achieved": 3 * sum(flops.values()) / (conv_ms / 1e3) / 1e12,
                                        "ms": conv_ms,
                                        "frac_of_step": conv_ms / max(step_layers_ms, 1e-9)}}
    else:  # FP32 path: no tensor-core GEMMs; report the dominant conv layer
        dom = max((t for t in times if t[0] in flops), key=lambda t: t[1] + t[2])
        achieved = 3 * flops[dom[0]] / ((dom[1] + dom[2]) / 1e3) / 1e12
        roofline = {"bound": "fp32", "kernel": f"{dom[0]} fprop+dgrad+wgrad",
                    "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": achieved / tf32_peak, "traffic": None, "peak_source": peak_src}
    if args.profile_layers and rank == 0:
        for n, f, b in times:
            print(f"  {n:8s} fwd {f:8.3f} ms  bwd {b:8.3f} ms", file=sys.stderr)
        for lab, kms, kfl in sorted(kprof, key=lambda r: -r[1]):
            print(f"  gemm {lab:44s} {kms:7.3f} ms {kfl / kms / 1e9:7.1f} TF/s", file=sys.stderr)

    # ---- end to end through the public API with host buffers ------------
    e2e = None
    if not args.no_e2e:
        from paper_1412_4564_b200.graph import Feeder
        # two host batches in pinned memory, alternated so every step copies
        # a fresh batch; the copy of batch i+1 overlaps step i (cnn_train prefetch)
        hosts = []
        for k in range(2):
            b = net.init_inputs(data_seed=1 + rank + 100 * k, label_seed=3 + rank + 100 * k)
            hosts.append({n: torch.from_numpy(np.ascontiguousarray(b[n], np.float32)).pin_memory()
                          for n in ("data", "label")})
        feed = Feeder(g, ["data", "label"], stream)

        def e2e_run(n):
            feed.put(hosts[0])
            for i in range(n):
                feed.take()
                if i + 1 < n:
                    feed.put(hosts[(i + 1) % 2])
                tr.step(want_loss=False, stream=sp)
                feed.result("objective")  # async D2H of this step's loss
            return feed.collect()

        e2e_run(2)
        barrier()
        t0 = time.perf_counter()
        losses = e2e_run(args.steps)
        barrier()
        e2e_ms = max_over_ranks(1e3 * (time.perf_counter() - t0) / args.steps)
        assert len(losses) == args.steps and all(np.isfinite(v).all() for v in losses)
        e2e = {"value": world * args.batch / (e2e_ms / 1e3), "unit": UNIT,
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": feed.h2d_bytes,
               "d2h_bytes_per_step": 4,
               "note": "wall clock; per-step H2D of a fresh pinned batch on a copy stream "
                       "overlapping the previous step (cnn_train prefetch), async loss D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.net)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"failed: {ex}"[:300]}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
               "higher_is_better": True, "scaling": "weak",
               "vs_baseline": value / PUBLISHED, "dtype": args.math,
               "data": "synthetic (xoshiro256**: U[-1,1) data, 0.01 N(0,1) weights, random labels)",
               "config": {"workload": WORKLOAD, "global_batch": world * args.batch,
                          "per_gpu_batch": args.batch, "parallelism": f"dp{world}",
                          "math": args.math, "cuda_graph": not args.no_graph,
                          "l2": "inputs larger than L2: the step streams ~4 GB of activations "
                                "(input batch alone 158 MB > 126 MB L2)",
                          "vs_baseline_ref": "MatConvNet CuDNN v2 AlexNet b=256 on 1x Titan "
                                             "Black, 264.1 img/s (PAPER.md:126)"},
               "loss": loss, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(launches), "clocks": clk}
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
