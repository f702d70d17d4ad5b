"""Data-parallel step.

CPU (gloo, world size 2): the NCCL unique-id exchange that TSMNet.dp_init
performs through torch.distributed.
GPU (>= 2 devices, one process per GPU over NCCL): the allreduced gradient of
two ranks with one clip each equals the single-GPU gradient of both clips
(the Sigma-loss makes gradients sums over the batch, net.cpp:141-146), and
parameters stay identical across ranks after an SGD step."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _id_exchange(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C

    from paper_1910_00932_b200 import _lib
    from paper_1910_00932_b200 import network  # noqa: F401  (declares tsm_nccl_unique_id)
    buf = (C.c_char * 128)()
    if rank == 0:
        _lib.check(_lib.lib.tsm_nccl_unique_id(buf))
    obj = [bytes(buf)]
    dist.broadcast_object_list(obj, src=0)
    q.put((rank, obj[0]))
    dist.destroy_process_group()


def test_nccl_id_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_id_exchange, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert got[0] == got[1] and len(got[0]) == 128 and any(got[0])


def _dp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_1910_00932_b200.network import TSMNet
    g = torch.Generator(device=dev).manual_seed(5)
    xs = torch.randn(world, 8, 3, 224, 224, device=dev, generator=g)
    net = TSMNet(batch=1, device=dev).init_random(seed=3).dp_init(bucket_bytes=8 << 20)
    net.train_step(xs[rank:rank + 1], update=False)
    torch.cuda.synchronize()
    dp_grads = net.grads.clone()
    out = {}
    if rank == 0:
        full = TSMNet(batch=world, device=dev).init_random(seed=3)
        full.train_step(xs, update=False)
        torch.cuda.synchronize()
        out["rel"] = float((dp_grads - full.grads).norm() / full.grads.norm())
    # one SGD step: parameters must stay bitwise identical across ranks
    net.train_step(xs[rank:rank + 1], lr=1e-12)
    torch.cuda.synchronize()
    p = net.params.clone()
    ref = p.clone()
    dist.broadcast(ref, src=0)
    out["same_params"] = bool(torch.equal(p, ref))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_dp_allreduce_matches_full_batch():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    print("dp vs full-batch grad rel-L2", res[0]["rel"])
    assert res[0]["rel"] < 1e-3
    assert all(r["same_params"] for r in res.values())


def _max_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    # bench.py's timing rule: every rank reports its own ms, rank 0 prints the max
    q.put((rank, bench.allreduce_max(10.0 * (rank + 1), dist, world, torch.device("cpu"))))
    dist.destroy_process_group()


def test_bench_max_over_ranks_gloo():
    """bench.py's multi-GPU timing takes the max over ranks (world size 2, gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_max_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert got == {0: 20.0, 1: 20.0}
