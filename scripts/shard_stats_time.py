"""Device time of the partial-mode stats pass of one vocabulary shard on one GPU
(development aid): rank 0 of P, B = 256 P sequences, slice V / P.
    P=4 python scripts/shard_stats_time.py"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402
from paper_2511_11733_b200.sharded import (PeerExchange, ShardedVerifier,  # noqa: E402
                                           contiguous_slice, slice_bounds)

P = int(os.environ.get("P", 4))
B, G, V = 256 * P, 8, 128256
v = Verifier(0)
sv = ShardedVerifier(v)
R = int(os.environ.get("R", 0))
lo, n = slice_bounds(V, P, R)
draft_f, target_f = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft_f, p, vocab=V)
draft, target = contiguous_slice(draft_f, lo, n), contiguous_slice(target_f, lo, n)
del draft_f, target_f
PEER = os.environ.get("PEER") == "1"  # stores into P local buffers (no NVLink)
if PEER:
    _, size = sv.packed_layout(B, G, p.top_m)
    ex = PeerExchange(v, P, R, size, bases=PeerExchange.allocate_local(v, P, size))


def run(w):
    if PEER:
        sv.stats_peers(ex, w + 1, draft, target, tokens, p, V, lo, n)
    else:
        sv.stats(draft, target, tokens, p, V, lo, n)


for w in range(3):
    p.window = w
    run(w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for w in range(20):
    p.window = 100 + w
    run(100 + w)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
gb = B * (2 * G + 1) * n * 2 / 1e9
print(f"P={P} slice={n} peer={PEER} stats ms {ms:.4f} GB/s {gb / ms * 1e3:.0f}")
