"""One-process emulation of a P-rank sharded window (for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402
from paper_2511_11733_b200.sharded import shard_slices  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
v = Verifier(0)
B, G, V = 256 * P, 8, 128256
draft, target = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft, p, vocab=V)
for w in range(3):
    p.window = w
    shard_slices(v, draft, target, tokens, p, V, P)
torch.cuda.synchronize()
print("ok")
