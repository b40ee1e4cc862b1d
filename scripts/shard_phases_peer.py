"""Per-phase device time of one vocabulary-sharded window with the fused peer
exchange (development aid).
    torchrun --nproc-per-node P scripts/shard_phases_peer.py"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402
from paper_2511_11733_b200.sharded import (SHARD_RESOLVE, PeerExchange, ShardedVerifier,  # noqa: E402
                                           TorchComm, contiguous_slice, slice_bounds)

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
_, size = sv.packed_layout(B, G, p.top_m)
ex = PeerExchange(v, comm.size, comm.rank, size, comm=comm)
status = torch.zeros(1, dtype=torch.int32, device="cuda")
names = ["stats+signal", "wait", "merge", "gather_masses", "resolve", "allreduce", "copy"]
acc = [0.0] * len(names)
for it in range(13):
    p.window = it
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    ev[0].record()
    sv.stats_peers(ex, it + 1, draft, target, tokens, p, V, lo, n)
    ev[1].record()
    sv.wait_peers(ex, it + 1, status)
    ev[2].record()
    out, pos, u, mass = sv.merge(draft, target, tokens, p, V, lo, n,
                                 (ex.set_bases(it + 1)[ex.rank], ex.P, ex.stride))
    ev[3].record()
    masses = comm.all_gather(mass)
    ev[4].record()
    tok = sv.sample(SHARD_RESOLVE, comm.rank, comm.size, draft, target, tokens, p, V, lo, n, out,
                    pos, u, masses, tiles=sv._tiles)
    ev[5].record()
    comm.all_reduce_max(tok)
    ev[6].record()
    out.extra_token.copy_(tok)
    ev[7].record()
    torch.cuda.synchronize()
    if it >= 3:
        for i in range(len(names)):
            acc[i] += ev[i].elapsed_time(ev[i + 1]) / 10
print(f"rank {comm.rank}: " + ", ".join(f"{k} {t:.3f}" for k, t in zip(names, acc)) +
      f" total {sum(acc):.3f} ms", flush=True)
dist.destroy_process_group()
