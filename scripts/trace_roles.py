"""Per-role cycle accounting of the fused kernel (development aid).

Run with the tracing build:  python paper_2511_11733_b200/build.py --trace
    DSDV_LIB=paper_2511_11733_b200/libdsdv_trace.so python scripts/trace_roles.py
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200 import dsdv  # noqa: E402
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams, WindowResult  # noqa: E402

names = ["compute_wait_full", "compute_fold", "compute_sample", "compute_wait_slot",
         "compute_item_end", "epi_wait_full", "epi_merge", "epi_topm", "epi_decide", "epi_sample",
         "prod_wait_empty", "prod_drain", "prod_items", "prod_samples", "kernel", "epi_items",
         "topm_candidates", "topm_survivors", "topm_fallbacks", "max_survivors", "need_exact",
         "cap_calls", "cap_sorts", "compute_cap", "compute_loop", "compute_a", "compute_b"]
B = int(os.environ.get("B", 256))
V = int(os.environ.get("V", 128256))
G = int(os.environ.get("G", 8))
tau = float(os.environ.get("TAU", 0.2))
top_m = int(os.environ.get("TOPM", 10))
dt = torch.bfloat16 if os.environ.get("DT", "bf16") == "bf16" else torch.float32
v = Verifier(0)
lib = dsdv.LIB
lib.dsdv_debug_trace.restype = C.c_int
lib.dsdv_debug_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
draft, target = v.synth_logits(B, G, V, dt, logits_seed=42)
p = VerifyParams(gamma=G, tau=tau, top_m=top_m, seed=1)
if os.environ.get("NONEKEY"):
    p.ratio_limit, p.gap_limit, p.overlap_floor = float("inf"), 1.0, 0.0
tokens = v.draft_sample(draft, p, vocab=V)
out = WindowResult.allocate(B, G, draft.device, per_position=False)
SHARD = int(os.environ.get("SHARD", 0))  # >0: the partial stats pass of slice 0 of SHARD
if SHARD:
    from paper_2511_11733_b200.sharded import ShardedVerifier, contiguous_slice, slice_bounds
    sv = ShardedVerifier(v)
    lo, n = slice_bounds(V, SHARD, 0)
    ds, ts = contiguous_slice(draft, lo, n), contiguous_slice(target, lo, n)


def run_window():
    if SHARD:
        sv.stats(ds, ts, tokens, p, V, lo, n)
    else:
        v.verify(draft, target, tokens, p, vocab=V, out=out)


for w in range(3):
    p.window = w
    run_window()
torch.cuda.synchronize()
buf = np.zeros((1024, 28), dtype=np.uint64)
lib.dsdv_debug_trace(v._h, buf.ctypes.data, 1024)  # clear
reps = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for w in range(reps):
    p.window = 100 + w
    run_window()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
grid = lib.dsdv_debug_trace(v._h, buf.ctypes.data, 1024)
t = buf[:grid].astype(np.float64)
kern = t[:, 14].mean()
res = {"ms_per_window": ms, "grid": grid, "kernel_cycles_per_cta": kern / reps}
for i, n in enumerate(names):
    if n == "max_survivors":
        res[n] = float(t[:, i].max())
        continue
    if n in ("prod_items", "prod_samples", "epi_items", "kernel", "topm_candidates",
             "topm_survivors", "topm_fallbacks", "need_exact", "cap_calls", "cap_sorts"):
        res[n] = t[:, i].sum() / reps
        continue
    per = {"compute": 16, "epi": 2, "prod": 1}[n.split("_")[0]]
    res[n + "_frac"] = round(t[:, i].mean() / per / kern, 4)
kc = t[:, 14] / reps
res["kernel_cycles_min_med_max"] = [float(kc.min()), float(np.median(kc)), float(kc.max())]
fw = t[:, 1] / 16 / reps
res["fold_cycles_per_warp_min_med_max"] = [float(fw.min()), float(np.median(fw)), float(fw.max())]
print(json.dumps(res, indent=1))
