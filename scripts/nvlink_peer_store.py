"""NVLink evidence for the fused peer exchange: one process drives GPU 0 and
GPU 1 (peer access, no IPC), and rank 0's stats pass of a P=2 vocabulary-sharded
C4 window (B=512, V=128256 bf16, this rank's 64128 ids) stores every item's
record and top lists into GPU 1's exchange buffer as items complete. Profile
the kernel on device 0 with NVLink counters (one process, so ncu may wrap it):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,nvltx__bytes.sum,\
nvltx__bytes_data_user.sum -k regex:fused_verify python scripts/nvlink_peer_store.py
Prints the algorithmic peer-store bytes per window for comparison."""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import LIB, Verifier, VerifyParams  # noqa: E402
from paper_2511_11733_b200.sharded import (PeerExchange, ShardedVerifier,  # noqa: E402
                                           contiguous_slice, slice_bounds)

assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
P, B, G, V = 2, 512, 8, 128256
v0, v1 = Verifier(0), Verifier(1)
v0._check(LIB.dsdv_enable_peer_access(v0._h, 1))
torch.cuda.set_device(0)
sv = ShardedVerifier(v0)
_, size = sv.exchange_layout(B, G, 10)
stride = -(-size // 256) * 256
nbytes = 2 * P * stride + 8 * P
b0, b1 = C.c_void_p(), C.c_void_p()
v0._check(LIB.dsdv_dev_alloc(v0._h, nbytes, C.byref(b0)))
v1._check(LIB.dsdv_dev_alloc(v1._h, nbytes, C.byref(b1)))
ex = PeerExchange(v0, P, 0, size, bases=[b0.value, b1.value])
draft_f, target_f = v0.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v0.draft_sample(draft_f, p, vocab=V)
lo, n = slice_bounds(V, P, 0)
draft, target = contiguous_slice(draft_f, lo, n), contiguous_slice(target_f, lo, n)
del draft_f, target_f
for w in range(4):
    p.window = w
    sv.stats_peers(ex, w + 1, draft, target, tokens, p, V, lo, n)
torch.cuda.synchronize(0)
# what one window stores into the peer's buffer (records [B][G+1][8] f64 + top
# lists [B][G][2][M] (f64 value + i32 id))
peer_bytes = B * (G + 1) * 8 * 8 + B * G * 2 * 10 * 12
print(json.dumps({"peer_store_bytes_per_window": peer_bytes, "batch": B, "vocab_slice": n,
                  "logit_bytes_per_window": B * (2 * G + 1) * n * 2}))
