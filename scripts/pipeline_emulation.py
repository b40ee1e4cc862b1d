"""C5: pipeline-sharded decoding emulation on the box's GPUs.

    python scripts/pipeline_emulation.py                     # 1 GPU, N=8 stages
    torchrun --nproc-per-node P scripts/pipeline_emulation.py  # stage s on GPU s mod P

k per round comes from the GPU verifier (dsdv_verify, C2 workload, gamma=8);
t0 is a device spin, t1 in {3, 5, 7, 10} t0 is injected before every hop.
Prints one JSON line per t1 (rank 0)."""
import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200 import metrics  # noqa: E402
from paper_2511_11733_b200 import pipeline as pl  # noqa: E402
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams  # noqa: E402


def verifier_ks(v: Verifier, rounds: int, seed: int = 1):
    """Accepted lengths and key counts of `rounds` verification windows of
    the C2 workload (one per sequence)."""
    B, G, V = 64, 8, 128256
    draft, target = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
    p = VerifyParams(gamma=G, tau=0.2, seed=seed)
    tokens = v.draft_sample(draft, p, vocab=V)
    ks, kcs = [], []
    for w in range(-(-rounds // B)):
        p.window = w
        out = v.verify(draft, target, tokens, p, vocab=V, per_position=False)
        v.sync(p, out, batch=B, vocab=V)
        ks += out.accepted_count.cpu().tolist()
        kcs += out.key_count.cpu().tolist()
    return ks[:rounds], kcs[:rounds]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=64)
    ap.add_argument("--t0-us", type=float, default=50.0)
    ap.add_argument("--csv-dir", default=None,
                    help="also write trace/summary CSVs in the reference schema (metrics.hpp)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
        from paper_2511_11733_b200.sharded import TorchComm
        comm = TorchComm()
    v = Verifier(local)
    ks, kcs = verifier_ks(v, args.rounds)
    if comm:  # every rank uses rank 0's k values
        t = torch.tensor(ks + kcs, dtype=torch.int32, device="cuda")
        comm.dist.broadcast(t, 0)
        allv = t.cpu().tolist()
        ks, kcs = allv[:len(ks)], allv[len(ks):]
    N, t0 = args.stages, int(args.t0_us * 1000)
    emu = pl.PipelineEmulator(v, N, comm)
    tokens = sum(k + 1 for k in ks)
    kbar = tokens / len(ks)
    emu.run(pl.standard_units(8, 0), 0)  # warm-up (NCCL P2P communicators)
    # per-unit transport overhead with zero injected latency (measured, reported)
    zero = emu.run(pl.standard_units(32, 0), 0) / 32
    trace, summary = [], []
    for mult in (3, 5, 7, 10):
        t1 = mult * t0
        t_std = emu.run(pl.standard_units(tokens, t0), t1)
        t_dsd = emu.run(pl.dsd_units(ks, t0), t1)
        if rank == 0 and args.csv_dir:
            run_id = f"c5_p{world}_t1x{mult}"
            st = metrics.compute_stats(ks, kcs, 8, total_ms=t_dsd)
            for i, (k, kc) in enumerate(zip(ks, kcs)):
                trace.append(metrics.TraceRow(run_id, i, 8, 0.2, N, t0 / 1e6, t1 / 1e6, k, kc,
                                              k * t0 / 1e6, (N - 1) * t1 / 1e6,
                                              (k * t0 + (N - 1) * t1) / 1e6, 1))
            summary.append(metrics.SummaryRow(
                run_id, st.rho, st.avg_accepted_len, st.total_tokens, st.sync_rounds,
                st.tokens_per_ms or 0.0, st.key_token_fraction,
                pl.analytic_speedup(st.rho, st.avg_accepted_len - 1.0, N, t0, t1),
                t_std / t_dsd))
        if rank == 0:
            des_std = pl.des_total(pl.standard_units(tokens, t0), N, t1) / 1e6
            des_dsd = pl.des_total(pl.dsd_units(ks, t0), N, t1) / 1e6
            print(json.dumps({
                "config": "C5", "stages": N, "gpus": world, "t0_ms": t0 / 1e6, "t1_ms": t1 / 1e6,
                "t1_over_t0": mult, "rounds": len(ks), "committed_tokens": tokens,
                "mean_committed_per_round": kbar, "mean_accepted_k": kbar - 1,
                "measured": {"standard_ms": t_std, "dsd_ms": t_dsd,
                             "R_comm": 1.0 - t_dsd / t_std, "speedup": t_std / t_dsd,
                             "sync_rounds_standard": tokens, "sync_rounds_dsd": len(ks)},
                "des": {"standard_ms": des_std, "dsd_ms": des_dsd, "R_comm": 1.0 - des_dsd / des_std},
                "analytic_R_comm_at_mean": pl.comm_reduction_ratio(kbar, N, t0, t1),
                "transport_overhead_per_unit_ms": zero,
            }), flush=True)
    if rank == 0 and args.csv_dir:
        d = Path(args.csv_dir)
        d.mkdir(parents=True, exist_ok=True)
        (d / f"c5_p{world}_trace.csv").write_text(metrics.render_trace_csv(trace))
        (d / f"c5_p{world}_summary.csv").write_text(metrics.render_summary_csv(summary))
    if comm:
        comm.dist.destroy_process_group()


if __name__ == "__main__":
    main()
