"""Multi-rank host logic of the data-parallel step on CPU (gloo, world size 2).

The device path (ck_trainer: NCCL allreduce per layer bucket, overlapped with
backward) needs several GPUs; here we check what it relies on:
  * summing the per-rank gradients of the shards equals the gradient of the
    concatenated batch (the loss is a sum over images, loss.cpp:182) --
    computed with the CPU oracle chain on each rank and reduced with gloo;
  * the per-rank loss sums to the global loss;
  * the NCCL unique-id exchange and the bucket plan.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import chain
    from paper_1412_4564_b200 import dp, nets

    gb = 6
    full = nets.lenet(batch=gb)
    params = full.init_params()
    inputs = full.init_inputs()
    lo, hi = dp.shard(gb, rank, world)
    local = nets.lenet(batch=hi - lo)
    per_img = 28 * 28
    shard_in = {"data": inputs["data"][lo * per_img:hi * per_img],
                "label": inputs["label"][lo:hi]}
    vals, derivs = chain.run(local, params, shard_in)
    loss = torch.tensor([vals["objective"][0]], dtype=torch.float64)
    dist.all_reduce(loss)
    grads = {}
    for name, _, _ in local.params:
        t = torch.from_numpy(derivs[name].copy())
        dist.all_reduce(t)  # the NCCL allreduce of ck_trainer, here over gloo
        grads[name] = t.numpy()
    uid = dp.share_unique_id(lambda: bytes(range(128)), rank)
    if rank == 0:
        vals_f, derivs_f = chain.run(full, params, inputs)
        out.put({"loss": float(loss[0]), "loss_full": float(vals_f["objective"][0]),
                 "err": max(float(np.abs(grads[n] - derivs_f[n]).max() /
                                  (np.abs(derivs_f[n]).max() + 1e-30)) for n in grads),
                 "uid_ok": uid == bytes(range(128))})
    dist.destroy_process_group()


def test_dp_gradient_sum_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert abs(res["loss"] - res["loss_full"]) < 1e-9 * abs(res["loss_full"])
    assert res["err"] < 1e-12
    assert res["uid_ok"]


def test_bucket_plan_alexnet():
    from paper_1412_4564_b200 import dp, nets
    plan = dp.bucket_plan(nets.alexnet(batch=1))
    assert [l for l, _ in plan] == ["fc8", "fc7", "fc6", "conv5", "conv4", "conv3", "conv2",
                                    "conv1"]
    assert plan[0][1] == ["fc8f", "fc8b"]
    assert sum(len(ps) for _, ps in plan) == 16


def test_shard():
    from paper_1412_4564_b200 import dp
    assert dp.shard(512, 1, 2) == (256, 512)
    with pytest.raises(ValueError):
        dp.shard(10, 0, 3)
