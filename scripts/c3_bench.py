"""C3 timing (V=151936, gamma=16, B=1024, fp32 logits, tau sweep
0-0.5): device time of dsdv_verify (full window) and dsdv_verify_early_exit per
tau, CUDA events over back-to-back windows, against the measured HBM peak.
The logits (20.5 GB per window) exceed L2 many times over, so no flush is needed.
    python scripts/c3_bench.py > profiles/r2_c3_bench.json
With C2=1: the C2 window (V=128256, gamma=8, B=256, bf16) over tau in {0, 0.2,
0.5, 1}; tau = 0 and 1 need no softened-mix sum (2 exponentials per pair).
    C2=1 python scripts/c3_bench.py > profiles/r2_c2_tau_sweep.json"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams, WindowResult  # noqa: E402
from bench import ClockSampler  # noqa: E402

import os  # noqa: E402

C2 = os.environ.get("C2") == "1"
B, G, V = (256, 8, 128256) if C2 else (1024, 16, 151936)
DT = torch.bfloat16 if C2 else torch.float32
TAUS = (0.0, 0.2, 0.5, 1.0) if C2 else (0.0, 0.1, 0.2, 0.3, 0.4, 0.5)
peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()
                  ).get("hbm_gbs", 6550.0) if (Path(__file__).resolve().parent.parent /
                                               "MEASURED_PEAKS.json").exists() else 6550.0
v = Verifier(0)
draft, target = v.synth_logits(B, G, V, DT, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = v.draft_sample(draft, p, vocab=V)
out = WindowResult.allocate(B, G, draft.device, per_position=False)
nbytes = B * (2 * G + 1) * V * (2 if C2 else 4)
rows = []
for tau in TAUS:
    p.tau = tau
    res = {"tau": tau}
    for mode in ("full", "early_exit"):
        ee = mode == "early_exit"
        for w in range(3):
            p.window = w
            v.verify(draft, target, tokens, p, vocab=V, out=out, early_exit=ee)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            e0.record()
            for w in range(20):
                p.window = 100 + w
                v.verify(draft, target, tokens, p, vocab=V, out=out, early_exit=ee)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        v.sync(p, out, batch=B, vocab=V)
        res[mode] = {"ms_per_window": ms, "verified_tokens_per_s": B * G / (ms * 1e-3),
                     "mean_accepted_k": float(out.accepted_count.float().mean()),
                     "clocks": clk.summary()}
        if not ee:
            res[mode]["GBps"] = nbytes / (ms * 1e-3) / 1e9
            res[mode]["frac_of_measured_hbm"] = res[mode]["GBps"] / peak
    rows.append(res)
cfg = ("C2: V=128256, gamma=8, B=256, bf16 logits" if C2 else
       "C3: V=151936, gamma=16, B=1024, fp32 logits")
print(json.dumps({"config": cfg + ", lambda=(2.0, 0.2, 0.5), top_m=10",
                  "algorithmic_bytes_per_window": nbytes,
                  "hbm_peak_gbs": peak, "rows": rows}, indent=1))
