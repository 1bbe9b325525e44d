#!/usr/bin/env python
"""Training throughput of the BASELINE.json networks on B200 (headline:
AlexNet fwd+bwd images/sec, batch 256 per GPU).

One step = forward + backward + gradient allreduce (N>1) + SGD of the
network through the device DAG engine of libck.so.  `python bench.py` runs
N=1; `python bench.py --gpus N` re-launches itself under
torch.distributed.run with one process per GPU (NCCL) when it is not already
a rank; rank 0 prints one JSON line.  `--net lenet|cifar|alexnet|vgg16bn`
selects the other BASELINE configs (each at its BASELINE batch).

`--impl reference` times the reference's own CPU implementation (the convkit
sources compiled verbatim into oracle/_ref, driven through its DAG engine) on
this box's host cores; it loads nothing from paper_1412_4564_b200's library.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "images/s"
PUBLISHED = 264.1  # MatConvNet CuDNN v2, AlexNet b=256, 1x Titan Black
WORKLOADS = {
    "alexnet": "imagenet-caffe-alex 227x227x3, fwd+bwd+SGD, 256 images/GPU",
    "vgg16bn": "VGG-VD-16 with batch norm, 224x224x3, fwd+bwd+SGD, 64 images/GPU",
    "cifar": "CIFAR-10 quick with LRN, 32x32x3, fwd+bwd+SGD, 128 images/GPU",
    "lenet": "MNIST LeNet, 28x28x1, fwd+bwd+SGD, 100 images/GPU",
}
# nets whose whole training-step working set fits in the 126 MB L2: timed
# with an L2 flush between steps; the others stream more than L2 every step
L2_RESIDENT = ("lenet", "cifar")
L2_NOTES = {"alexnet": "inputs larger than L2: the step streams the whole activation set "
                       "(b=256: ~4 GB; the input batch alone is 158 MB > 126 MB L2)",
            "vgg16bn": "inputs larger than L2: the step streams the whole activation set "
                       "(b=64: ~6 GB; conv1_1 output alone is 822 MB > 126 MB L2)"}
NAMES = {"alexnet": "AlexNet", "vgg16bn": "VGG-16-bn", "cifar": "CIFAR-10 quick",
         "lenet": "LeNet"}
# SURVEY.md §8d CPU sample batches for the reference (per-image linear)
REF_SAMPLE = {"alexnet": 16, "vgg16bn": 2, "cifar": 128, "lenet": 100}


def metric_for(net):
    return f"{NAMES[net]} fwd+bwd images/sec"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--net", default="alexnet", choices=sorted(WORKLOADS))
    p.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: BASELINE's)")
    p.add_argument("--math", default="tf32", choices=["tf32", "fp32"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="launch every kernel (no CUDA graph)")
    p.add_argument("--profile-layers", action="store_true", help="print per-layer times to stderr")
    p.add_argument("--l2-flush", default="auto", choices=["auto", "on", "off"],
                   help="write a 256 MB buffer between timed steps (auto: nets whose step "
                        "working set fits in the 126 MB L2, i.e. lenet and cifar)")
    # internal: CPU sample run in a subprocess
    p.add_argument("--cpu-sample", type=int, default=0)
    p.add_argument("--cpu-reps", type=int, default=1)
    a = p.parse_args()
    if not a.batch:
        a.batch = {"lenet": 100, "cifar": 128, "alexnet": 256, "vgg16bn": 64}[a.net]
    return a


def ck_env_guard():
    """Every CK_* variable in the environment, recorded; the run is refused
    when one is set (product builds ignore them -- knob() in capi.cu -- but a
    number must not be taken under a tuning override either way)."""
    env = {k: v for k, v in os.environ.items() if k.startswith("CK_") and k != "CK_EXTRA_NVCC"}
    if env:
        print(f"bench.py: refusing to run with CK_* overrides set: {env}", file=sys.stderr)
        sys.exit(2)
    return env


def relaunch_distributed(args):
    """--gpus N outside torch.distributed.run: become N ranks (one per GPU)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # init log (nranks, NVLS) on stderr
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, which):
        """Host time of the timed region's start ('t0') / end ('t1')."""
        setattr(self, which, time.perf_counter())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)  # let a sample land after a short timed region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        # samples inside the timed region (100 ms period, so a short region
        # is bracketed by the nearest sample on either side)
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        lines = [ln for t, ln in self.lines if t0 is None or (t0 - 0.1 <= t <= t1 + 0.1)]
        if not lines and self.lines:
            lines = [min(self.lines, key=lambda tl: abs(tl[0] - (t0 or 0)))[1]]
        sm, mx, reasons = [], [], set()
        for ln in lines:
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

def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_graph_for(net):
    """The reference DAG engine (oracle/_ref) with the network and its
    synthetic inputs -- generated by the oracle's restatement of the
    reference generator (oracle.Rng; identical stream to rng.cpp, pinned by
    tests/test_oracle_vs_ref.py), so nothing of libck is loaded."""
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
    for k, v in {**net.init_params(rng=O.Rng), **net.init_inputs(rng=O.Rng)}.items():
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
    """The verbatim reference on this box's host cores, bounded samples at the
    SURVEY §8d batch: reference-faithful single-threaded BLAS (the reference
    has no OpenMP) and the generous all-cores BLAS."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    nproc = os.cpu_count() or 1
    batch = REF_SAMPLE[net_name]
    many = run_cpu_sample(net_name, batch, 1, nproc)
    one = run_cpu_sample(net_name, batch, 1, 1)
    return {"value": many["images"] / many["seconds"], "unit": UNIT, "cores": nproc,
            "kind": "reference",
            "sample": f"1 fwd+bwd of {net_name} at batch {batch} through the reference DAG engine "
                      f"(graph.cpp:494/548), OpenBLAS GEMM with {nproc} threads, "
                      f"{many['seconds']:.1f} s",
            "single_thread": {"value": one["images"] / one["seconds"], "cores": 1,
                              "sample": f"same, OPENBLAS_NUM_THREADS=1 (reference-faithful: "
                                        f"no OpenMP in the reference build), "
                                        f"{one['seconds']:.1f} s"},
            "nproc": nproc, "cpu": cpu_model()}


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
    batch = REF_SAMPLE[args.net]  # bounded sample per step
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
    out = {"metric": metric_for(args.net), "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (xoshiro256**: U[-1,1) data, 0.01 N(0,1) weights, random labels)",
           "impl": "reference",
           "config": {"workload": WORKLOADS[args.net] + f" (sample: {batch} images per step)",
                      "per_step_batch": batch, "threads": threads},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"{args.steps} steps x fwd+bwd at batch {batch}, reference "
                                      f"convkit sources (oracle/_ref), OpenBLAS {threads} threads",
                            "cpu": cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# --------------------------------------------------- roofline helpers --

def mem_layers(net):
    """Memory-bound layers with SURVEY.md §8d compulsory bytes per pass:
    (layer, kind, fwd bytes, bwd bytes)."""
    shapes = dict(net.inputs)
    for n, s, _ in net.params:
        shapes[n] = s
    out = []
    # a relu whose input has no other reader is fused into its producer (the
    # bnorm apply writes relu(y), the backward gates inside the bnorm passes):
    # its compulsory bytes (8n fwd, 12n bwd) are charged to that entry
    readers = {}
    for kind, name, ins, outs, p in net.layers:
        for i in ins:
            readers[i] = readers.get(i, 0) + 1
    fused_relu = {ins[0] for kind, name, ins, outs, p in net.layers
                  if kind == "relu" and readers.get(ins[0]) == 1}
    for kind, name, ins, outs, p in net.layers:
        xs = shapes[ins[0]]
        nx = xs[0] * xs[1] * xs[2] * xs[3]
        if kind == "conv":
            fs = shapes[ins[1]]
            ys = ((xs[0] + p[2] + p[3] - fs[0]) // p[0] + 1,
                  (xs[1] + p[4] + p[5] - fs[1]) // p[1] + 1, fs[3], xs[3])
        elif kind == "pool":
            ys = ((xs[0] + p[4] + p[5] - p[0]) // p[2] + 1,
                  (xs[1] + p[6] + p[7] - p[1]) // p[3] + 1, xs[2], xs[3])
            ny = ys[0] * ys[1] * ys[2] * ys[3]
            out.append((name, "pool", 4 * (nx + ny), 4 * (2 * nx + ny)))
        elif kind == "loss":
            ys = (1, 1, 1, 1)
        else:
            ys = xs
            if kind == "bnorm" and outs[0] in fused_relu:
                out.append((name, "bnorm+relu", 16 * nx, 24 * nx))
            elif kind in ("lrn", "bnorm"):
                out.append((name, kind, 8 * nx, 12 * nx))
        shapes[outs[0]] = ys
    return out


# ---------------------------------------------------------------- ours --

def main():
    args = parse()
    if args.cpu_sample:
        return cpu_sample_main(args)
    ck_env = ck_env_guard()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    if args.impl == "reference":
        return reference_main(args)

    import numpy as np
    import torch

    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200._lib import lib
    from paper_1412_4564_b200.graph import Graph, Trainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE {world} != --gpus {args.gpus}", file=sys.stderr)
        return 2
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
    clocks = ClockSampler(local)
    clocks.start()  # running through the warm-up: samples exist when the region is short
    for _ in range(max(args.warmup, 3)):
        tr.step(want_loss=False, stream=sp)
    barrier()
    clocks.mark("t0")
    launches0, tc0 = g.hd.launches, g.hd.tc_launches
    flush = args.l2_flush == "on" or (args.l2_flush == "auto" and args.net in L2_RESIDENT)
    with torch.cuda.stream(stream):
        if flush:
            # per-step event pairs with an L2 flush (a 256 MB write, > 126 MB L2)
            # between timed steps, outside the timed intervals
            fbuf = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            for a, b in ev:
                fbuf.fill_(1.0)
                a.record(stream)
                tr.step(want_loss=False, stream=sp)
                b.record(stream)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                tr.step(want_loss=False, stream=sp)
            e1.record(stream)
    barrier()
    clocks.mark("t1")
    clk = clocks.stop()
    launches = g.hd.launches - launches0  # total inside the timed region
    tc_launches = g.hd.tc_launches - tc0
    if flush:
        ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps)
        l2_note = ("L2 flushed between timed steps: a 256 MB device write outside per-step "
                   "event pairs (the step's working set fits in the 126 MB L2)")
    else:
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        l2_note = L2_NOTES.get(args.net, "no flush between steps (--l2-flush off)")
    value = world * args.batch / (ms / 1e3)
    loss = tr.step(want_loss=True, stream=sp)
    if not np.isfinite(loss):
        print(f"bench.py: non-finite loss {loss}", file=sys.stderr)
        return 3

    # ---- per-layer breakdown + roofline of the dominant kernel ----------
    # One more step, eager, with per-layer events and per-launch events around
    # every tensor-core GEMM (ck_set_kernel_profiling), on the step's stream;
    # the trainer's step events give the allreduce-complete tail.
    g.set_profiling(True)
    g.hd.kernel_profiling(True)
    ar0 = tr.allreduces
    tr.step(want_loss=False, stream=sp)
    ar_step = tr.allreduces - ar0
    torch.cuda.synchronize()
    times = g.layer_times()
    kprof = g.hd.kernel_profile()
    fwd_ms, bwd_ms, tail_ms = tr.last_timing()
    g.hd.kernel_profiling(False)
    g.set_profiling(False)
    flops = {}
    for name, xs, fs, p in net.conv_layers():
        s_, pt, pb, pl, pr = p[0], p[2], p[3], p[4], p[5]
        oh = (xs[0] + pt + pb - fs[0]) // s_ + 1
        ow = (xs[1] + pl + pr - fs[1]) // s_ + 1
        flops[name] = 2.0 * xs[3] * oh * ow * fs[3] * fs[0] * fs[1] * fs[2]
    conv_ms = sum(f + b for n, f, b in times if n in flops)
    step_layers_ms = sum(f + b for _, f, b in times)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs") or 6512.0
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
    traffic_db = {}
    try:
        traffic_db = json.load(open(os.path.join(ROOT, "profiles", "kernel_traffic.json")))
    except (OSError, ValueError):
        pass
    if kprof:
        # dominant kernel = the GEMM launch with the largest time in the step
        lab, kms, kfl = max(kprof, key=lambda r: r[1])
        achieved = kfl / (kms / 1e3) / 1e12
        gemm_ms = sum(r[1] for r in kprof)
        roofline = {"bound": "tensor", "kernel": f"tc_gemm_kernel: {lab}", "achieved": achieved,
                    "peak": tf32_peak, "unit": "TFLOP/s", "frac": achieved / tf32_peak,
                    "traffic": traffic_db.get(lab), "peak_source": peak_src, "launch_ms": kms,
                    "algorithmic_flop": kfl,
                    # the same launch against TF32 = half the pool's measured bf16 rate
                    # (MEASURED_PEAKS.json), burst and sustained: looser denominators
                    "frac_vs_half_bf16": {
                        "burst": achieved / ((peaks.get("bf16_tflops") or 1653.5) / 2.0),
                        "sustained": achieved / ((peaks.get("bf16_tflops_sustained") or 1397.0) / 2.0)},
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
    if ms < 1.0:
        roofline["note"] = (f"latency-bound step: {launches / max(args.steps, 1):.0f} kernels in "
                            f"{ms:.3f} ms; the dominant launch's fraction is not the bound")
    # memory-bound layers: SURVEY §8d compulsory bytes / event time / HBM peak
    tmap = {n: (f, b) for n, f, b in times}
    hbm = []
    for name, kind, fb, bb in mem_layers(net):
        f, b = tmap.get(name, (0.0, 0.0))
        for pas, byts, t in (("fwd", fb, f), ("bwd", bb, b)):
            if t > 0:
                gbs = byts / (t / 1e3) / 1e9
                hbm.append({"layer": f"{name} {pas}", "kind": kind, "bytes": byts, "ms": t,
                            "achieved": gbs, "frac": gbs / hbm_peak,
                            "traffic": traffic_db.get(f"{name} {pas}")})
    roofline["hbm"] = {"peak": hbm_peak, "unit": "GB/s",
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)", "layers": hbm}
    if args.profile_layers and rank == 0:
        for n, f, b in times:
            print(f"  {n:8s} fwd {f:8.3f} ms  bwd {b:8.3f} ms", file=sys.stderr)
        for lab, kms, kfl in sorted(kprof, key=lambda r: -r[1]):
            print(f"  gemm {lab:44s} {kms:7.3f} ms {kfl / kms / 1e9:7.1f} TF/s", file=sys.stderr)
        for h in hbm:
            print(f"  hbm {h['layer']:12s} {h['ms']:7.3f} ms {h['achieved']:7.0f} GB/s "
                  f"{h['frac']:.2f}", file=sys.stderr)

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

    dp_info = {"allreduce_groups_per_step": ar_step,
               "profiled_step": {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                                 "exchange_tail_ms": tail_ms,
                                 "note": "eager profiled step: time from the last backward "
                                         "kernel to the completion of the last gradient "
                                         "allreduce + SGD (communication not hidden by "
                                         "backward); single GPU: the update-stream tail"}}
    if rank == 0:
        out = {"metric": metric_for(args.net), "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
               "higher_is_better": True, "scaling": "weak",
               "vs_baseline": value / PUBLISHED if args.net == "alexnet" else None,
               "dtype": args.math,
               "data": "synthetic (xoshiro256**: U[-1,1) data, 0.01 N(0,1) weights, random labels)",
               "config": {"workload": WORKLOADS[args.net] if args.batch == nets.DEFAULT_BATCH[
                              args.net] else f"{args.net} batch {args.batch}",
                          "global_batch": world * args.batch, "per_gpu_batch": args.batch,
                          "parallelism": f"dp{world}", "math": args.math,
                          "cuda_graph": not args.no_graph,
                          "l2": l2_note,
                          "ck_env": ck_env, "libck": lib().ck_version().decode(),
                          "vs_baseline_ref": "MatConvNet CuDNN v2 AlexNet b=256 on 1x Titan "
                                             "Black, 264.1 img/s (PAPER.md:126)"},
               "loss": loss, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "dp": dp_info, "gpu_launches": int(launches), "tc_launches": int(tc_launches),
               "clocks": clk}
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
