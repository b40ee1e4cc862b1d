"""Quick device timing of dsdv_verify at a named shape (development aid)."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--gamma", type=int, default=8)
ap.add_argument("--V", type=int, default=128256)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--tau", type=float, default=0.2)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--top_m", type=int, default=10)
ap.add_argument("--none_key", action="store_true")
a = ap.parse_args()
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
v = Verifier(0)
draft, target = v.synth_logits(a.B, a.gamma, a.V, dt, logits_seed=42)
p = VerifyParams(gamma=a.gamma, tau=a.tau, seed=1, top_m=a.top_m)
if a.none_key:
    p.ratio_limit, p.gap_limit, p.overlap_floor = float("inf"), 1.0, 0.0
tokens = v.draft_sample(draft, p, vocab=a.V)
out = v.verify(draft, target, tokens, p, vocab=a.V, per_position=False)
v.sync(p, out, batch=a.B, vocab=a.V)
for w in range(3):
    p.window = w
    v.verify(draft, target, tokens, p, vocab=a.V, out=out)
torch.cuda.synchronize()
times = []
for i in range(a.iters):
    p.window = 100 + i
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    v.verify(draft, target, tokens, p, vocab=a.V, out=out)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
v.sync(p, out, batch=a.B, vocab=a.V)
es = draft.element_size()
nbytes = a.B * (2 * a.gamma + 1) * a.V * es
ms = sorted(times)[len(times) // 2]
k = out.accepted_count.float().mean().item()
print(json.dumps(dict(shape=vars(a), ms_median=ms, ms_min=min(times), GBps=nbytes / ms / 1e6,
                      frac_hbm=nbytes / ms / 1e6 / 6550.7, mean_k=k,
                      verified_tokens_per_s=a.B * a.gamma / ms * 1e3)))
