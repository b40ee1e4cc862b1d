"""Device time of dsdv_verify without status checks (development aid for
probe builds such as libdsdv_nofold.so, whose results are meaningless)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402

dt = torch.bfloat16 if (sys.argv[1] if len(sys.argv) > 1 else "bf16") == "bf16" else torch.float32
import os
B, G, V = (int(os.environ.get(k, d)) for k, d in (("B", 256), ("G", 8), ("V", 128256)))
v = Verifier(0)
draft, target = v.synth_logits(B, G, V, dt, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft, p, vocab=V)
out = v.verify(draft, target, tokens, p, vocab=V, per_position=False)
for w in range(3):
    p.window = w
    v.verify(draft, target, tokens, p, vocab=V, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for w in range(20):
    p.window = 100 + w
    v.verify(draft, target, tokens, p, vocab=V, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"{dt} ms {ms:.4f} GB/s {B * (2 * G + 1) * V * draft.element_size() / ms / 1e6:.0f}")
