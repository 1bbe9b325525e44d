"""The data-parallel training step on real NCCL communicators (ck_trainer,
engine.cu): one process per GPU, the batch sharded, every layer's parameter
derivatives allreduced on the comm stream as soon as backward finishes them,
then SGD.

Parity: after one step, the parameters of every rank equal those of a single
GPU stepping on the concatenated batch -- the loss is a sum over images
(loss.cpp:182), so the summed shard gradients are the full-batch gradient --
within 1e-5 relative (FP32 path; only the summation order differs).  World
sizes above the visible GPU count are skipped; world 1 always runs and
exercises the real one-rank communicator (ncclAllReduce, event hand-off,
comm-stream SGD, CUDA-graph capture of all of it)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, gb, graph_mode, q):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    from paper_1412_4564_b200 import dp, nets
    from paper_1412_4564_b200.graph import Graph, Trainer
    full = nets.lenet(batch=gb)
    params, inputs = full.init_params(), full.init_inputs()
    lo, hi = dp.shard(gb, rank, world)
    net = nets.lenet(batch=hi - lo)
    g = Graph(math="fp32")
    net.build(g)
    g.finalize()
    for k, v in params.items():
        g.set(k, v)
    g.set("data", inputs["data"][lo * 784:hi * 784])
    g.set("label", inputs["label"][lo:hi])
    t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
    t.init_dp(dp.share_unique_id(Trainer.unique_id, rank), rank, world)
    t.set_graph(graph_mode)
    stream = torch.cuda.Stream()
    losses = [t.step(stream=stream.cuda_stream) for _ in range(2)]
    res = {p: g.get(p) for p, _, _ in net.params}
    ar = t.allreduces
    dist.destroy_process_group()
    q.put((rank, losses, res, ar))


def _single(gb, steps=2):
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Graph, Trainer
    net = nets.lenet(batch=gb)
    g = Graph(math="fp32")
    net.build(g)
    g.finalize()
    for k, v in {**net.init_params(), **net.init_inputs()}.items():
        g.set(k, v)
    t = Trainer(g, lr=0.01, momentum=0.9, weight_decay=5e-4)
    losses = [t.step() for _ in range(steps)]
    return losses, {p: g.get(p) for p, _, _ in net.params}


@pytest.mark.parametrize("graph_mode", [False, True])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_dp_step_equals_full_batch_step(world, graph_mode):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    import torch.multiprocessing as mp
    gb = 8 * world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, gb, graph_mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_losses, ref = _single(gb)
    for rank, losses, res, ar in out:
        assert ar > 0, "the DP step issued no NCCL allreduce"
        # the reported loss is the allreduced (global) objective
        assert abs(losses[0] - ref_losses[0]) <= 1e-5 * abs(ref_losses[0])
        for k in ref:
            a, b = res[k].astype(np.float64), ref[k].astype(np.float64)
            assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max(), (rank, k)
    if world > 1:  # every replica ends bit-identical (same reduced gradient)
        for _, _, res, _ in out[1:]:
            for k in res:
                assert np.array_equal(res[k], out[0][2][k])


def test_dp_bucket_plan_matches_engine():
    """dp.bucket_plan (the host mirror) lists the parameters in the order the
    engine's trainer finishes and reduces them (finalize's arena order)."""
    from paper_1412_4564_b200 import dp, nets
    from paper_1412_4564_b200.graph import Graph, Trainer
    net = nets.alexnet(batch=2)
    g = Graph(math="tf32")
    net.build(g)
    g.finalize()
    plan = dp.bucket_plan(net)
    # arena order = the order of the derivative addresses
    addr = {p: g.view(p, deriv=True).data for p, _, _ in net.params}
    flat = [p for _, ps in plan for p in ps]
    assert flat == sorted(addr, key=lambda p: addr[p])
    Trainer(g)  # builds the same per-layer buckets without error
