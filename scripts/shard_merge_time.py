"""Device time of rank 0's merge (+ fused MASS) of one vocabulary-sharded
window, with every rank's stats computed on this one GPU (development aid).
    P=4 python scripts/shard_merge_time.py"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402
from paper_2511_11733_b200.sharded import ShardedVerifier, contiguous_slice, slice_bounds  # noqa: E402

P = int(os.environ.get("P", 4))
B, G, V = 256 * P, 8, 128256
v = Verifier(0)
draft_f, target_f = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft_f, p, vocab=V)
svs, parts = [], []
for r in range(P):
    lo, n = slice_bounds(V, P, r)
    parts.append((lo, n, contiguous_slice(draft_f, lo, n), contiguous_slice(target_f, lo, n)))
    svs.append(ShardedVerifier(v))
del draft_f, target_f
p.window = 7
packed_all = torch.stack([svs[r].stats(d, t, tokens, p, V, lo, n) for r, (lo, n, d, t) in enumerate(parts)])
lo, n, d, t = parts[0]
for w in range(3):
    svs[0].merge(d, t, tokens, p, V, lo, n, packed_all)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for w in range(20):
    svs[0].merge(d, t, tokens, p, V, lo, n, packed_all)
e1.record()
torch.cuda.synchronize()
print(f"P={P} merge ms {e0.elapsed_time(e1) / 20:.4f}")
