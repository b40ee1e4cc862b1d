"""Per-phase device time of one vocabulary-sharded window with the peer
exchange, the phases of dsdv_shard_verify_peers enqueued one by one with CUDA
events between them (development aid).
    torchrun --nproc-per-node P scripts/shard_phases_onecall.py"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams, WindowResult  # noqa: E402
from paper_2511_11733_b200.sharded import (PeerExchange, ShardedVerifier, TorchComm,  # noqa: E402
                                           contiguous_slice, slice_bounds)

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
comm = TorchComm()
v = Verifier(local)
sv = ShardedVerifier(v)
B, G, V = 256 * comm.size, 8, 128256
draft_f, target_f = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft_f, p, vocab=V)
lo, n = slice_bounds(V, comm.size, comm.rank)
draft, target = contiguous_slice(draft_f, lo, n), contiguous_slice(target_f, lo, n)
del draft_f, target_f
_, size = sv.exchange_layout(B, G, p.top_m)
ex = PeerExchange(v, comm.size, comm.rank, size, comm=comm)
status = torch.zeros(1, dtype=torch.int32, device="cuda")
names = ["stats", "wait1", "merge", "wait2", "resolve", "wait3", "tokens"]
acc = [0.0] * len(names)
for it in range(13):
    p.window = it
    w = it + 1
    f = 3 * w
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    ev[0].record()
    sv.stats_peers(ex, w, draft, target, tokens, p, V, lo, n, flag=f)
    ev[1].record()
    sv.wait_peers(ex, f, status)
    ev[2].record()
    out, position, u = sv.merge_peers(ex, w, draft, target, tokens, p, V, lo, n)
    sv.signal_peers(ex, f + 1)
    ev[3].record()
    sv.wait_peers(ex, f + 1, status)
    ev[4].record()
    sv.resolve_peers(ex, w, draft, target, tokens, p, V, lo, n, out, position, u)
    sv.signal_peers(ex, f + 2)
    ev[5].record()
    sv.wait_peers(ex, f + 2, status)
    ev[6].record()
    sv.tokens_max_peers(ex, w, B, G, p.top_m, out.extra_token)
    ev[7].record()
    torch.cuda.synchronize()
    if it >= 3:
        for i in range(len(names)):
            acc[i] += ev[i].elapsed_time(ev[i + 1]) / 10
print(f"rank {comm.rank}: " + ", ".join(f"{k} {t:.3f}" for k, t in zip(names, acc)) +
      f" total {sum(acc):.3f} ms", flush=True)
dist.destroy_process_group()
