"""Benchmark of the fused B200 verifier on BASELINE.json's headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one verification window (dsdv_verify) over B=256 sequences of
gamma=8 drafted tokens with Llama-3 vocabulary V=128256 and bf16 logits
(configs[1] of BASELINE.json). The metric is verified draft
tokens/s = B*gamma/t_step (whole job, summed over ranks).

  value        device time of K back-to-back fused launches (CUDA events on the
               launching stream; inputs already in HBM; the 1.12 GB of logits per
               step exceed the 126 MB L2, so no flush is needed)
  e2e          the same metric through the public API with HOST buffers: pinned
               host logits/tokens are copied in and the round's results copied
               out inside the timed region, every step
  roofline     algorithmic bytes B*(2*gamma+1)*V*2 per launch / average launch
               time, against MEASURED_PEAKS.json's HBM copy bandwidth
  cpu_baseline the reference's own verifier (oracle/_ref, compiled from
               /root/reference) on the host cores, bounded sample

N > 1 (torchrun), default --parallel vocab: the vocabulary is
sharded over the N ranks (rank p holds ids [p*V/N, (p+1)*V/N) of every row, as
a tensor-parallel LM head produces them) and the batch grows to B*N sequences,
so every GPU streams the same 1.12 GB per window as at N=1 (weak scaling);
each window is dsdv_shard_stats -> NCCL all-gather -> dsdv_shard_merge ->
dsdv_shard_sample(MASS) -> all-gather -> dsdv_shard_sample(RESOLVE) ->
all-reduce (paper_2511_11733_b200/sharded.py). --parallel replicas runs N
independent copies of the N=1 window instead.

--impl reference times the reference's CPU verifier (oracle/_ref) on all host
threads on the same workload and prints the same JSON line with
"impl": "reference" (rank 0 only under torchrun).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

B, GAMMA, V = 256, 8, 128256
TAU, RATIO, GAP, OVERLAP, TOP_M = 0.2, 2.0, 0.2, 0.5, 10
LOGITS_SEED = 42
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
METRIC = "verified draft tokens/s & % HBM roofline (V=128k, γ=8, B=256) at 1/2/4/8 GPU"
UNIT = "verified draft tokens/s"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled by NVML every few
    milliseconds while the timed region runs (nvidia-smi as a fallback)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_s: float = 0.0005):
        self.index = index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return float(sm), float(mx), int(bits)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                              "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        sm, mx, act = [x.strip() for x in out.split(",")]
        return float(sm), float(mx), int(act, 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, _, bits in self.samples
                          for bit, name in self.REASONS.items() if bits & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def bf16_bits_to_f32(bits):
    import numpy as np
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def cpu_reference(draft_h, target_h, tokens_h, seed, window, nthreads=None):
    """Time the reference's CPU verifier (oracle/_ref, else the C restatement)
    on EVERY sequence of the window, all host threads. Returns a cpu_baseline
    dict plus the reference's k per sequence."""
    from oracle.oracle_lib import Oracle, RefOracle, window_uniforms
    nthreads = nthreads or os.cpu_count() or 1
    if RefOracle.available():
        impl, kind = RefOracle(), "reference"
    else:
        impl, kind = Oracle(), "port"
    crit = Oracle.crit(RATIO, GAP, OVERLAP, TOP_M)
    Bh = draft_h.shape[0]
    U = window_uniforms(seed, window, Bh, GAMMA)
    t0 = time.perf_counter()
    k, _, _ = impl.verify_batch_f32(draft_h, target_h, tokens_h, TAU, crit, U, V, nthreads)
    dt = time.perf_counter() - t0
    return {"value": Bh * GAMMA / dt, "unit": UNIT, "cores": nthreads, "kind": kind,
            "cpu_model": cpu_model(), "seconds": dt,
            "sample": f"all {Bh} sequences of the C2 window (V={V}, gamma={GAMMA}, bf16 logits "
                      f"widened to fp32), reference verify_round loop over Distribution rows "
                      f"({'oracle/_ref: the reference sources compiled' if kind == 'reference' else 'oracle C port'}), "
                      f"{nthreads} threads, {dt:.2f} s"}, k


def check_parity(ver, draft, target, tokens, p, timed_k):
    """Verify the timed window against the fp64 oracle on every sequence
    (per-position outputs of the same launch parameters; the window is
    deterministic, so k must equal the timed launch's)."""
    import numpy as np
    from oracle.oracle_lib import Oracle, window_uniforms
    from tests.parity_util import compare_batch, gpu_window, host_logits
    crit = Oracle.crit(RATIO, GAP, OVERLAP, TOP_M)
    gpu = gpu_window(ver, draft, target, tokens, V, TAU, crit, p.seed, p.window)
    ref = Oracle().verify_batch(host_logits(draft), host_logits(target), tokens.cpu().numpy(),
                                [(TAU, crit)], window_uniforms(p.seed, p.window, B, GAMMA), V,
                                all_positions=True)[0]
    rep = compare_batch(ref, gpu)
    return {"window": int(p.window), "sequences": rep.sequences,
            "positions_checked": rep.positions_checked, "mismatches": len(rep.mismatches),
            "eps_events": rep.eps_events,
            "device_near_threshold": int(gpu["near_threshold"].sum()),
            "timed_k_equal": bool(np.array_equal(gpu["accepted_count"].numpy(), timed_k)),
            "max_h_rel_err": rep.max_h_err, "max_p_rel_err": rep.max_p_rel_err,
            "checker": "oracle/dsd_oracle.c fp64 (Oracle.verify_batch), every sequence"}


def check_parity_sharded(ver, out, tokens, window, Bt, world, device):
    """A vocabulary-sharded window (every rank holds the same decisions) against
    the fp64 oracle over the whole rows, every sequence: the eps-band count of
    this P (the merge order of the slice sums differs from one GPU's)."""
    import torch
    from oracle.oracle_lib import Oracle, window_uniforms
    from tests.parity_util import compare_batch, host_logits
    crit = Oracle.crit(RATIO, GAP, OVERLAP, TOP_M)
    gpu = out.to_host()
    draft_f, target_f = ver.synth_logits(Bt, GAMMA, V, torch.bfloat16, logits_seed=LOGITS_SEED,
                                         device=device)
    dh, th = host_logits(draft_f), host_logits(target_f)
    del draft_f, target_f
    ref = Oracle().verify_batch(dh, th, tokens.cpu().numpy(), [(TAU, crit)],
                                window_uniforms(1, window, Bt, GAMMA), V, all_positions=True)[0]
    rep = compare_batch(ref, gpu)
    return {"window": int(window), "shards": world, "sequences": rep.sequences,
            "positions_checked": rep.positions_checked, "mismatches": len(rep.mismatches),
            "eps_events": rep.eps_events, "device_near_threshold": int(gpu["near_threshold"].sum()),
            "max_h_rel_err": rep.max_h_err, "max_p_rel_err": rep.max_p_rel_err,
            "checker": "oracle/dsd_oracle.c fp64 (Oracle.verify_batch) over the unsharded rows"}


def make_inputs(ver, device):
    import torch
    from paper_2511_11733_b200.dsdv import VerifyParams
    draft, target = ver.synth_logits(B, GAMMA, V, torch.bfloat16, logits_seed=LOGITS_SEED,
                                     device=device)
    p = VerifyParams(gamma=GAMMA, tau=TAU, ratio_limit=RATIO, gap_limit=GAP,
                     overlap_floor=OVERLAP, top_m=TOP_M, seed=1, window=0)
    tokens = ver.draft_sample(draft, p, vocab=V)  # draft_window's draws (verifier.cpp:93-110)
    torch.cuda.synchronize(device)
    return draft, target, tokens, p


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2511_11733_b200.dsdv import Verifier, WindowResult

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    ver = Verifier(local_rank)
    draft, target, tokens, p = make_inputs(ver, device)
    out = WindowResult.allocate(B, GAMMA, device, per_position=False)
    stream = torch.cuda.current_stream(device)

    def step(w):
        p.window = w
        ver.verify(draft, target, tokens, p, vocab=V, out=out, stream=stream)

    for w in range(args.warmup):
        step(10_000 + w)
    ver.sync(p, out, batch=B, vocab=V)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    launches0 = ver.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one more event after every window: the per-window times (SURVEY 8(d) asks
    # for the median); the total over the K windows gives `value`
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for k in range(args.steps):
            step(k)
            marks[k].record(stream)
        e1.record(stream)
        torch.cuda.synchronize(device)
    per_window = [e0.elapsed_time(marks[0])] + [marks[k - 1].elapsed_time(marks[k])
                                                  for k in range(1, args.steps)]
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    gpu_launches = ver.launches - launches0
    ms_t = torch.tensor([ms], device=device)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    ver.sync(p, out, batch=B, vocab=V)
    mean_k = float(out.accepted_count.float().mean().item())
    committed = float((out.accepted_count.float() + 1).sum().item())
    timed_k = out.accepted_count.cpu().numpy()

    # ---- early exit (dsdv_verify_early_exit): rows past each sequence's first
    # rejection are not streamed; same k / extra tokens. Its roofline counts the
    # rows the reference actually needs, never the full window's bytes.
    early = None
    if world == 1:
        def estep(w):
            p.window = w
            ver.verify(draft, target, tokens, p, vocab=V, out=out, stream=stream,
                       early_exit=True)
        for w in range(args.warmup):
            estep(10_000 + w)
        ver.sync(p, out, batch=B, vocab=V)
        ver.streamed_bytes(reset=True)
        torch.cuda.synchronize(device)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for k in range(args.steps):
            estep(k)
        g1.record(stream)
        torch.cuda.synchronize(device)
        ems = g0.elapsed_time(g1) / args.steps
        streamed = ver.streamed_bytes(reset=True) / args.steps
        # rows the reference needs, per timed window (k differs per window index)
        need_rows = 0
        ks = []
        for k in range(args.steps):
            estep(k)
            kk = out.accepted_count.cpu()
            ks.append(kk)
            need_rows += int(torch.where(kk < GAMMA, 2 * (kk + 1), 2 * GAMMA + 1).sum())
        need_bytes = need_rows * V * 2 / args.steps
        ek = torch.stack(ks)
        early = {"value": B * GAMMA / (ems * 1e-3), "unit": UNIT, "ms_per_step": ems,
                 "mean_accepted_k": float(ek.float().mean()),
                 "same_k_as_full_window": bool(torch.equal(ek[-1], out.accepted_count.cpu())),
                 "required_bytes_per_window": need_bytes, "streamed_bytes_per_window": streamed,
                 "roofline": {"bound": "hbm", "achieved": need_bytes / (ems * 1e-3) / 1e9,
                              "peak": measured_peaks().get("hbm_gbs", 6650.0), "unit": "GB/s",
                              "frac": need_bytes / (ems * 1e-3) / 1e9 /
                              measured_peaks().get("hbm_gbs", 6650.0),
                              "note": "required bytes = row pairs 0..k (k < gamma) or all gamma "
                                      "pairs + target row gamma (k = gamma), each read once "
                                      "(SPEC.md:244); streamed bytes include the extra-draw "
                                      "re-reads and rows in flight when a rejection landed"}}

    # ---- e2e: host buffers through the public API, copies inside the timed region
    draft_h = draft.cpu().pin_memory()
    target_h = target.cpu().pin_memory()
    tokens_h = tokens.cpu().pin_memory()
    res_h = {n: torch.empty(B, dtype=torch.int32).pin_memory()
             for n in ("accepted_count", "extra_token", "key_count", "status")}
    d_draft, d_target, d_tokens = (torch.empty_like(draft), torch.empty_like(target),
                                   torch.empty_like(tokens))
    h2d = draft_h.numel() * 2 + target_h.numel() * 2 + tokens_h.numel() * 4
    d2h = 4 * B * len(res_h)

    def e2e_step(w):
        d_draft.copy_(draft_h, non_blocking=True)
        d_target.copy_(target_h, non_blocking=True)
        d_tokens.copy_(tokens_h, non_blocking=True)
        p.window = w
        ver.verify(d_draft, d_target, d_tokens, p, vocab=V, out=out, stream=stream)
        for n, h in res_h.items():
            h.copy_(getattr(out, n), non_blocking=True)

    e2e_steps = max(3, min(args.steps, 10))
    for w in range(2):
        e2e_step(20_000 + w)
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for k in range(e2e_steps):
        e2e_step(30_000 + k)
    f1.record(stream)
    torch.cuda.synchronize(device)
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    et = torch.tensor([e2e_ms], device=device)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_ms = float(et.item())

    # ---- parity of the timed window and the CPU baseline (rank 0, N=1 only)
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        p.window = args.steps - 1  # the last timed window
        parity = check_parity(ver, draft, target, tokens, p, timed_k)
        d32 = draft_h.float().numpy()
        t32 = target_h.float().numpy()
        cpu, _ = cpu_reference(d32, t32, tokens_h.numpy(), p.seed, p.window)

    if rank != 0:
        return
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    alg_bytes = B * (2 * GAMMA + 1) * V * 2
    achieved = alg_bytes / (ms * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "traffic_c2.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    value = world * B * GAMMA / (ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: Philox-seeded Zipf/Gaussian logit-row families (SURVEY.md 8d), "
                "draft tokens sampled on device from P_d",
        "config": {"workload": "C2: dsdv_verify window, V=128256, gamma=8, B=256 per GPU, bf16 logits, "
                               "tau=0.2, lambda=(2.0, 0.2, 0.5), top_m=10",
                   "batch_per_gpu": B, "gamma": GAMMA, "vocab": V,
                   "parallelism": f"{world} independent ranks (sequence-parallel replicas)",
                   "l2": "no flush needed: 1.12 GB of logits per step > 126 MB L2",
                   "mean_accepted_k": mean_k, "committed_tokens_per_s": world * committed / (ms_max * 1e-3)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "frac_of_nominal_8tbs": achieved / 8000.0,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback",
                     "note": "bf16 at tau in (0,1) is compute-bound before HBM: 3 exponentials per element pair, all on MUFU; the fold alone, data in shared memory, runs at 5.9 TB/s equivalent (DESIGN.md section 3)"},
        "e2e": {"value": world * B * GAMMA / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "ms_per_window_median": statistics.median(per_window),
    }
    # the second bound: exponentials on the MUFU pipe (0.5 warp-instructions per
    # clock per SM measured, scripts/micro/pipes.cu) at the sampled SM clock
    exps = (3 * GAMMA + 1) * B * V  # t, d and the softened mix per pair; bonus row t
    mhz = line["clocks"].get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
    peak_exp = sms * 16 * mhz * 1e6 / 1e9
    line["roofline"]["exp_pipe"] = {
        "achieved": exps / (ms * 1e-3) / 1e9, "peak": peak_exp, "unit": "Gexp/s",
        "frac": exps / (ms * 1e-3) / 1e9 / peak_exp, "exps_per_launch": exps,
        "note": "algorithmic exponentials of the first pass (sample items add ~10%); "
                "peak = SMs x 16 MUFU.EX2 lanes per clock"}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if parity is not None:
        line["parity"] = parity
    if early is not None:
        line["early_exit"] = early
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, local_rank):
    """C4: vocabulary-sharded window over NCCL, B*world sequences."""
    import torch
    import torch.distributed as dist
    from paper_2511_11733_b200.dsdv import Verifier, VerifyParams
    from paper_2511_11733_b200.sharded import (ShardedVerifier, TorchComm, contiguous_slice,
                                               slice_bounds)

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    ver = Verifier(local_rank)
    comm = TorchComm()
    sv = ShardedVerifier(ver)
    Bt = B * world
    # identical full rows on every rank (same seed), then this rank's slice
    draft_f, target_f = ver.synth_logits(Bt, GAMMA, V, torch.bfloat16, logits_seed=LOGITS_SEED,
                                         device=device)
    p = VerifyParams(gamma=GAMMA, tau=TAU, ratio_limit=RATIO, gap_limit=GAP,
                     overlap_floor=OVERLAP, top_m=TOP_M, seed=1, window=0)
    tokens = ver.draft_sample(draft_f, p, vocab=V)
    lo, n = slice_bounds(V, world, rank)
    draft = contiguous_slice(draft_f, lo, n)
    target = contiguous_slice(target_f, lo, n)
    del draft_f, target_f
    torch.cuda.synchronize(device)
    stream = torch.cuda.current_stream(device)

    def step(w):
        p.window = w
        return sv.verify(draft, target, tokens, p, V, lo, n, comm, stream=stream,
                         exchange=args.exchange)

    for w in range(args.warmup):
        out = step(10_000 + w)
    dist.barrier()
    torch.cuda.synchronize(device)
    launches0 = ver.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        h0 = time.perf_counter()
        e0.record(stream)
        for k in range(args.steps):
            out = step(k)
        e1.record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # enqueue rate
        torch.cuda.synchronize(device)
    dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    gpu_launches = ver.launches - launches0
    timed_window = args.steps - 1  # `out` holds this window's results
    ms_t = torch.tensor([ms], device=device)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    mean_k = float(out.accepted_count.float().mean().item())
    committed = float((out.accepted_count.float() + 1).sum().item())
    bad = int((out.status != 0).sum().item())  # includes peer flag-round timeouts (DSDV_E_NCCL)

    # e2e: this rank's slice and the tokens from pinned host memory, results back
    draft_h, target_h, tokens_h = (draft.cpu().pin_memory(), target.cpu().pin_memory(),
                                   tokens.cpu().pin_memory())
    res_h = {k: torch.empty(Bt, dtype=torch.int32).pin_memory()
             for k in ("accepted_count", "extra_token", "key_count", "status")}
    d_draft, d_target, d_tokens = (torch.empty_like(draft), torch.empty_like(target),
                                   torch.empty_like(tokens))
    h2d = draft_h.numel() * 2 + target_h.numel() * 2 + tokens_h.numel() * 4
    d2h = 4 * Bt * len(res_h)

    def e2e_step(w):
        d_draft.copy_(draft_h, non_blocking=True)
        d_target.copy_(target_h, non_blocking=True)
        d_tokens.copy_(tokens_h, non_blocking=True)
        p.window = w
        o = sv.verify(d_draft, d_target, d_tokens, p, V, lo, n, comm, stream=stream,
                      exchange=args.exchange)
        for k, h in res_h.items():
            h.copy_(getattr(o, k), non_blocking=True)

    e2e_steps = max(3, min(args.steps, 10))
    for w in range(2):
        e2e_step(20_000 + w)
    torch.cuda.synchronize(device)
    dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for k in range(e2e_steps):
        e2e_step(30_000 + k)
    f1.record(stream)
    torch.cuda.synchronize(device)
    et = torch.tensor([f0.elapsed_time(f1) / e2e_steps], device=device)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_ms = float(et.item())
    if rank != 0:
        return
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    alg_bytes = Bt * (2 * GAMMA + 1) * n * 2  # this rank's slice of every row
    # peer stores per window (exchange="peer"): records [B][G+1][8] f64 + top lists
    # [B][G][2][M] (f64 value, i32 id) + [B] masses f64 + [B] tokens i32, into
    # each of the other ranks' buffers
    M = min(TOP_M, V)
    nvl_bytes = (world - 1) * (Bt * (GAMMA + 1) * 8 * 8 + Bt * GAMMA * 2 * M * 12 + Bt * 12)
    line = {
        "metric": METRIC, "value": Bt * GAMMA / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: Philox-seeded Zipf/Gaussian logit-row families (SURVEY.md 8d), "
                "draft tokens sampled on device from P_d",
        "config": {"workload": f"C4: vocabulary-sharded window, V=128256 over {world} ranks "
                               f"({n} ids on rank 0), B={Bt} (256 per GPU), gamma=8, bf16 logits, "
                               "tau=0.2, lambda=(2.0, 0.2, 0.5), top_m=10",
                   "batch_total": Bt, "gamma": GAMMA, "vocab": V, "vocab_per_rank": n,
                   "parallelism": (f"vocab-sharded tp{world} (no collective call per window: "
                                   "records, masses and tokens as the kernels' NVLink peer "
                                   "stores into IPC-mapped buffers + flag rounds)")
                   if args.exchange == "peer" else
                   (f"vocab-sharded tp{world} (NCCL: 2 all-gathers + 1 all-reduce "
                    "per window)"),
                   "exchange": ("nccl (peer mapping unavailable)"
                                if getattr(sv, "peer_fallback", False) else args.exchange),
                   "l2": "no flush needed: 1.12 GB of logits per GPU per step > 126 MB L2",
                   "mean_accepted_k": mean_k, "status_errors": bad,
                   "host_enqueue_ms_per_step": host_ms,
                   "committed_tokens_per_s": committed / (ms_max * 1e-3)},
        "roofline": {"bound": "hbm+nvlink", "achieved": alg_bytes / (ms_max * 1e-3) / 1e9,
                     "peak": hbm, "unit": "GB/s",
                     "frac": (alg_bytes / (hbm * 1e9) + nvl_bytes / (NVLINK_GBS * 1e9)) /
                             (ms_max * 1e-3),
                     "traffic": None, "algorithmic_bytes_per_launch": alg_bytes,
                     "nvlink_bytes_out_per_window": nvl_bytes, "nvlink_peak_gbs": NVLINK_GBS,
                     "roofline_us": (alg_bytes / (hbm * 1e9) + nvl_bytes / (NVLINK_GBS * 1e9)) * 1e6,
                     "note": "frac = (this rank's logit bytes / HBM peak + the bytes it stores "
                             "into its peers' exchange buffers / NVLink peer bandwidth) / window "
                             "time; NVLink peak: the measured peer copy of B200_PROFILING.md "
                             "(770 GB/s per direction)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback"},
        "e2e": {"value": Bt * GAMMA / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
    }
    # the last timed window against the fp64 oracle on the whole rows (rank 0,
    # after the timed regions; the other ranks are done)
    if not args.no_cpu:
        line["parity"] = check_parity_sharded(ver, out, tokens, timed_window, Bt, world, device)
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU verifier (oracle/_ref, the
    reference sources compiled) on all host threads, every sequence of the
    C2 window each step. Inputs never touch the GPU library: the window is
    generated on the host by oracle_synth_logits (bit-identical to the
    device's dsdv_synth_logits, tests/test_gpu_parity.py) and the draft
    tokens are drawn from P_d by the fp64 oracle with the same Philox draft
    slots as dsdv_draft_sample (equal except draws within 1e-5 of a CDF
    boundary)."""
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np
    from oracle.oracle_lib import Oracle, window_uniforms
    nthreads = os.cpu_count() or 1
    o = Oracle()
    t0 = time.perf_counter()
    dbits, tbits = o.synth_logits(B, GAMMA, V, True, logits_seed=LOGITS_SEED, nthreads=nthreads)
    d32, t32 = bf16_bits_to_f32(dbits), bf16_bits_to_f32(tbits)
    del dbits, tbits
    U = window_uniforms(1, 0, B, GAMMA)

    def draw(b):
        st, tok, _ = o.draft_tokens(d32[b, :, :V].astype(np.float64), U[b, :GAMMA])
        assert st == 0
        return tok

    with ThreadPoolExecutor(nthreads) as ex:
        tk = np.stack(list(ex.map(draw, range(B)))).astype(np.int32)
    prep_s = time.perf_counter() - t0
    samples = []
    for w in range(args.warmup + args.steps):
        r, _ = cpu_reference(d32, t32, tk, 1, w, nthreads)
        if w >= args.warmup:
            samples.append(r)
    total_s = sum(x["seconds"] for x in samples)
    v = B * GAMMA * len(samples) / total_s
    sample = samples[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s / len(samples) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the GPU arm's Philox Zipf/Gaussian window (SURVEY.md 8d) generated "
                "on the host (oracle_synth_logits, bit-identical to dsdv_synth_logits), draft "
                "tokens drawn from P_d on the host",
        "config": {"workload": "C2: dsdv_verify window, V=128256, gamma=8, B=256 per GPU, bf16 logits, "
                               "tau=0.2, lambda=(2.0, 0.2, 0.5), top_m=10",
                   "batch_per_gpu": B, "gamma": GAMMA, "vocab": V,
                   "implementation": "reference verify_round loop (oracle/_ref) on all host threads",
                   "input_prep_s": prep_s},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": sample["cores"], "kind": sample["kind"],
                         "cpu_model": sample["cpu_model"],
                         "sample": f"every step: {sample['sample']}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--parallel", choices=["vocab", "replicas"], default="vocab",
                    help="N>1: vocabulary-sharded window (C4) or independent replicas")
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                    help="vocab: partial records by the stats kernel's own NVLink stores into "
                         "every rank's buffer (CUDA IPC), or by an NCCL all-gather")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        elif world > 1 and args.parallel == "vocab":
            run_sharded(args, rank, world, local)
        else:
            run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
