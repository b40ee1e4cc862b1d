"""Stage timeline of CTA 0 (development aid; needs a -DDSDV_TRACE -DDSDV_TIMELINE build):
issue -> ready latency of each chunk's copies and the compute warps' pace."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200 import dsdv  # noqa: E402
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams, WindowResult  # noqa: E402

v = Verifier(0)
lib = dsdv.LIB
lib.dsdv_debug_trace.restype = C.c_int
lib.dsdv_debug_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
B, G, V = 256, 8, 128256
draft, target = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft, p, vocab=V)
out = WindowResult.allocate(B, G, draft.device, per_position=False)
for w in range(3):
    p.window = w
    v.verify(draft, target, tokens, p, vocab=V, out=out)
torch.cuda.synchronize()
buf = np.zeros((1024, 28), dtype=np.uint64)
lib.dsdv_debug_trace(v._h, buf.ctypes.data, 1024)  # clear
p.window = 77
v.verify(draft, target, tokens, p, vocab=V, out=out)
torch.cuda.synchronize()
lib.dsdv_debug_trace(v._h, buf.ctypes.data, 1024)
tl = buf.reshape(-1)[512 * 28: 512 * 28 + 4096].astype(np.int64)
n = int(min(tl[4094], tl[4095], 1000))
t = tl[:n * 4].reshape(n, 4)
issue, ready, waited, done = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
lat = ready - issue
print(f"chunks {n}")
print(f"compute per chunk (ready->done) median {np.median(done - ready):.0f} cycles")
print(f"waited per chunk median {np.median(waited):.0f}, mean {waited.mean():.0f}; chunks that waited >200: {(waited > 200).mean():.2f}")
print(f"issue->ready latency median {np.median(lat):.0f}, p10 {np.percentile(lat, 10):.0f}, p90 {np.percentile(lat, 90):.0f}")
S = 5
gap = issue[S:] - done[:-S]  # producer reissues stage k+S after the last release of k (warp 0's done ~ release)
print(f"issue(k+{S}) - done(k) median {np.median(gap):.0f}, p90 {np.percentile(gap, 90):.0f}")
print(f"chunk period (ready[k+1]-ready[k]) median {np.median(np.diff(ready)):.0f}")
for i in range(40, 60):
    print(i, issue[i] - issue[0], ready[i] - issue[0], waited[i], done[i] - issue[0], ready[i] - issue[i])
