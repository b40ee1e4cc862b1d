"""Timing probes of kernel variants (development aid)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams, WindowResult  # noqa: E402


def timeit(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


v = Verifier(0)
B, G, V = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 8, 128256
for dt in (torch.bfloat16, torch.float32):
    draft, target = v.synth_logits(B, G, V, dt, logits_seed=42)
    p = VerifyParams(gamma=G, tau=0.2, seed=1)
    tokens = v.draft_sample(draft, p, vocab=V)
    out = WindowResult.allocate(B, G, draft.device, per_position=True, records=True)
    nbytes = B * (2 * G + 1) * V * draft.element_size()
    res = {}
    for name, pp, stats in (("verify", p, False), ("stats_only", p, True),
                            ("tau0", VerifyParams(gamma=G, tau=0.0, seed=1), False),
                            ("top1", VerifyParams(gamma=G, tau=0.2, top_m=1, seed=1), False),
                            ("none_key_tau1", VerifyParams(gamma=G, tau=1.0, ratio_limit=float('inf'),
                                                           gap_limit=1.0, overlap_floor=0.0,
                                                           top_m=1, seed=1), False)):
        f = (lambda: v.window_stats(draft, target, tokens, pp, vocab=V, out=out)) if stats else \
            (lambda: v.verify(draft, target, tokens, pp, vocab=V, out=out))
        ms = timeit(f)
        res[name] = dict(ms=round(ms, 4), GBps=round(nbytes / ms / 1e6, 1))
    # copy bandwidth for reference
    x = torch.empty(nbytes // 2, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    ms = timeit(lambda: y.copy_(x))
    res["copy_rw_GBps"] = round(2 * x.numel() / ms / 1e6, 1)
    print(json.dumps({"dtype": str(dt), "B": B, **res}))
    del draft, target, x, y
