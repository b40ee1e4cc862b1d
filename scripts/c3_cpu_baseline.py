"""The reference's CPU verifier on the C3 workload (C3 full batch,
or a stated subset with explicit extrapolation), beside the GPU window time.

C3: V=151936, gamma=16, B=1024, fp32 logits, tau=0.2, lambda=(2.0, 0.2, 0.5),
top_m=10. The host timing runs the reference sources compiled (oracle/_ref) over
the first NSUB sequences of the same device-synthesised window, on all host
threads; the full batch is extrapolated linearly in the sequence count (the
sequences are independent). The GPU time is dsdv_verify over the whole window.
    python scripts/c3_cpu_baseline.py [NSUB] > profiles/r2_c3_cpu_baseline.json"""
import json
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.oracle_lib import Oracle, RefOracle, window_uniforms  # noqa: E402
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams, WindowResult  # noqa: E402
from bench import cpu_model  # noqa: E402

NSUB = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B, G, V, TAU = 1024, 16, 151936, 0.2
v = Verifier(0)
draft, target = v.synth_logits(B, G, V, torch.float32, logits_seed=42)
p = VerifyParams(gamma=G, tau=TAU, seed=1)
tokens = v.draft_sample(draft, p, vocab=V)
out = WindowResult.allocate(B, G, draft.device, per_position=False)
for w in range(3):
    p.window = w
    v.verify(draft, target, tokens, p, vocab=V, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for w in range(10):
    p.window = 100 + w
    v.verify(draft, target, tokens, p, vocab=V, out=out)
e1.record()
torch.cuda.synchronize()
gpu_ms = e0.elapsed_time(e1) / 10
p.window = 109
gpu_k = out.accepted_count[:NSUB].cpu().numpy()

impl, kind = (RefOracle(), "reference") if RefOracle.available() else (Oracle(), "port")
crit = Oracle.crit(2.0, 0.2, 0.5, 10)
dh = draft[:NSUB].cpu().numpy()
th = target[:NSUB].cpu().numpy()
th_tok = tokens[:NSUB].cpu().numpy()
U = window_uniforms(1, 109, NSUB, G)
nthreads = os.cpu_count() or 1
t0 = time.perf_counter()
k, _, _ = impl.verify_batch_f32(dh, th, th_tok, TAU, crit, U, V, nthreads)
cpu_s = time.perf_counter() - t0
cpu_full_s = cpu_s * B / NSUB
print(json.dumps({
    "config": "C3: V=151936, gamma=16, B=1024, fp32 logits, tau=0.2, lambda=(2.0, 0.2, 0.5), "
              "top_m=10",
    "gpu_ms_per_window": gpu_ms, "gpu_verified_tokens_per_s": B * G / (gpu_ms * 1e-3),
    "cpu": {"kind": kind, "cores": nthreads, "cpu_model": cpu_model(), "sequences_timed": NSUB,
            "seconds": cpu_s, "extrapolated_full_batch_seconds": cpu_full_s,
            "verified_tokens_per_s": NSUB * G / cpu_s},
    "gpu_over_cpu": cpu_full_s / (gpu_ms * 1e-3),
    "same_k_on_the_subset": bool((k == gpu_k).all()),
    "note": "the CPU subset is the first NSUB sequences of the same window (window 109); the "
            "full-batch CPU time is extrapolated linearly in the sequence count"}, indent=1))
