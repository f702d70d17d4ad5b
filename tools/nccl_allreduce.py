#!/usr/bin/env python3
"""NCCL allreduce of the TSM-R50 gradient (24,301,072 fp32) on N GPUs: time
(CUDA events, max over ranks) and ring bus bandwidth 2(N-1)/N * bytes / t —
the calibration input of paper_1910_00932_b200.scaling.b200_profile.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_allreduce.py
"""
import json
import os

import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
dist.init_process_group("nccl")
out = {}
for label, n in (("full", 24_301_072), ("bucket25MB", (25 << 20) // 4)):
    x = torch.ones(n, device="cuda")
    for _ in range(5):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    iters = 20
    a.record()
    for _ in range(iters):
        dist.all_reduce(x)
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters * 1e-3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t)
    out[label] = {"bytes": n * 4, "seconds": sec,
                  "busbw_GBps": 2 * (world - 1) / world * n * 4 / sec / 1e9}
if rank == 0:
    print(json.dumps({"world": world, **out}))
dist.destroy_process_group()
