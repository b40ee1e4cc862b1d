"""All-gather time of the sharded window's packed record buffer size (development aid).
    torchrun --nproc-per-node P scripts/nccl_probe.py"""
import os

import torch
import torch.distributed as dist

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
P = dist.get_world_size()
for mb in (0.5, 1.0, 2.5, 5.0):
    n = int(mb * 1e6 / 8)
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty(P * n, dtype=torch.float64, device="cuda")
    for _ in range(5):
        dist.all_gather_into_tensor(y, x)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        dist.all_gather_into_tensor(y, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    if dist.get_rank() == 0:
        print(f"P={P} all_gather {mb} MB/rank: {ms * 1e3:.1f} us, {P * mb / ms:.0f} GB/s out", flush=True)
dist.destroy_process_group()
