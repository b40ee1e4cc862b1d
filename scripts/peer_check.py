"""Multi-process check of the fused peer exchange: on every rank, the window
through exchange="peer" (CUDA IPC + the stats kernel's NVLink stores) equals
the window through the NCCL all-gather, over several windows. Every window
has its own logits and draft tokens (a stale record left in a reused buffer
set would differ), and the batch doubles at window 3, so the exchange is
remapped (the old mapping released collectively) partway through.
    torchrun --nproc-per-node P scripts/peer_check.py"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402
from paper_2511_11733_b200.sharded import (ShardedVerifier, TorchComm, contiguous_slice,  # noqa: E402
                                           slice_bounds)

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
comm = TorchComm()
v = Verifier(local)
sv_n, sv_p = ShardedVerifier(v), ShardedVerifier(v)
G, V = 8, 128256
p = VerifyParams(gamma=G, tau=0.2, seed=5)
lo, n = slice_bounds(V, comm.size, comm.rank)
bad = 0
for w in range(6):
    B = (64 if w < 3 else 128) * comm.size
    draft_f, target_f = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=7 + w)
    p.window = w
    tokens = v.draft_sample(draft_f, p, vocab=V)
    draft, target = contiguous_slice(draft_f, lo, n), contiguous_slice(target_f, lo, n)
    del draft_f, target_f
    a = sv_n.verify(draft, target, tokens, p, V, lo, n, comm, exchange="nccl").to_host()
    b = sv_p.verify(draft, target, tokens, p, V, lo, n, comm, exchange="peer").to_host()
    for k in a:
        x, y = torch.as_tensor(a[k]), torch.as_tensor(b[k])
        same = torch.equal(x, y) or (x.is_floating_point() and
                                     torch.equal(x.nan_to_num(7.0), y.nan_to_num(7.0)))
        bad += 0 if same else 1
    bad += int((b["status"] != 0).sum())
torch.cuda.synchronize()
t = torch.tensor([bad], device="cuda")
dist.all_reduce(t)
if comm.rank == 0:
    print(f"peer_check P={comm.size} B={B}: {'OK' if int(t.item()) == 0 else 'MISMATCH'} "
          f"({int(t.item())} differing fields over 6 windows x {comm.size} ranks)", flush=True)
dist.destroy_process_group()
