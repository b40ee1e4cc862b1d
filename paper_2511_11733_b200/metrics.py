"""Run statistics and the reference's trace / summary CSV schema for GPU
verifier and pipeline-emulation runs (reference:
proj/include/dsd/metrics.hpp:29-78, proj/src/metrics.cpp:29-142), so the
reference's analysis conventions (rho, avg_len, key fraction, sync rounds)
consume GPU runs unchanged."""
from __future__ import annotations

from dataclasses import dataclass, field

TRACE_HEADER = ("run_id,round_index,gamma,tau,n_nodes,t0_ms,t1_ms,k_accepted,key_count,"
                "compute_ms,comm_ms,total_ms,sync_rounds")
SUMMARY_HEADER = ("run_id,rho,avg_accepted_len,total_tokens,sync_rounds,tokens_per_ms,"
                  "key_token_fraction,analytic_speedup,measured_speedup")


def format_double(v: float) -> str:
    """Six significant digits, shortest general form (std::to_chars general, 6)."""
    return "%.6g" % v


@dataclass
class RunStats:
    rho: float
    avg_accepted_len: float
    total_tokens: int
    sync_rounds: int
    key_token_fraction: float
    tokens_per_ms: float | None = None


def compute_stats(ks: list[int], key_counts: list[int], gamma: int,
                  total_ms: float | None = None) -> RunStats:
    """compute_stats (metrics.cpp:29-59) over the rounds of one run: k per
    round and key tokens among its evaluated positions (the accepted ones plus
    the rejected one, or all gamma when the window passed)."""
    if not ks:
        raise ValueError("compute_stats needs at least one verification round")
    if gamma < 1:
        raise ValueError("compute_stats gamma must be >= 1")
    mean_k = sum(ks) / len(ks)
    decisions = sum(min(k + 1, gamma) for k in ks)
    tokens = sum(k + 1 for k in ks)
    st = RunStats(rho=mean_k / (gamma + 1), avg_accepted_len=mean_k + 1.0, total_tokens=tokens,
                  sync_rounds=len(ks),
                  key_token_fraction=(sum(key_counts) / decisions) if decisions else 0.0)
    if total_ms is not None and total_ms > 0.0:
        st.tokens_per_ms = tokens / total_ms
    return st


@dataclass
class TraceRow:
    run_id: str = ""
    round_index: int = 0
    gamma: int = 0
    tau: float = 0.0
    n_nodes: int = 0
    t0_ms: float = 0.0
    t1_ms: float = 0.0
    k_accepted: int = 0
    key_count: int = 0
    compute_ms: float = 0.0
    comm_ms: float = 0.0
    total_ms: float = 0.0
    sync_rounds: int = 0


@dataclass
class SummaryRow:
    run_id: str = ""
    rho: float = 0.0
    avg_accepted_len: float = 0.0
    total_tokens: float = 0.0
    sync_rounds: float = 0.0
    tokens_per_ms: float = 0.0
    key_token_fraction: float = 0.0
    analytic_speedup: float = 0.0
    measured_speedup: float = 0.0


def render_trace_csv(rows: list[TraceRow]) -> str:
    """Canonical order: round_index ascending, then run_id; LF endings."""
    out = [TRACE_HEADER]
    for r in sorted(rows, key=lambda r: (r.round_index, r.run_id)):
        out.append(",".join([r.run_id, str(r.round_index), str(r.gamma), format_double(r.tau),
                             str(r.n_nodes), format_double(r.t0_ms), format_double(r.t1_ms),
                             str(r.k_accepted), str(r.key_count), format_double(r.compute_ms),
                             format_double(r.comm_ms), format_double(r.total_ms),
                             str(r.sync_rounds)]))
    return "\n".join(out) + "\n"


def render_summary_csv(rows: list[SummaryRow]) -> str:
    """Ordered by run_id; counts are doubles (integral values render as integers)."""
    out = [SUMMARY_HEADER]
    for r in sorted(rows, key=lambda r: r.run_id):
        out.append(",".join([r.run_id, format_double(r.rho), format_double(r.avg_accepted_len),
                             format_double(r.total_tokens), format_double(r.sync_rounds),
                             format_double(r.tokens_per_ms), format_double(r.key_token_fraction),
                             format_double(r.analytic_speedup),
                             format_double(r.measured_speedup)]))
    return "\n".join(out) + "\n"


def window_trace_rows(accepted_count, key_count, gamma: int, tau: float, run_prefix: str = "seq",
                      window: int = 0) -> list[TraceRow]:
    """One trace row per sequence of a GPU verification window (each sequence's
    window is one round of its own run)."""
    return [TraceRow(run_id=f"{run_prefix}{b}", round_index=window, gamma=gamma, tau=tau,
                     n_nodes=1, k_accepted=int(k), key_count=int(kc), sync_rounds=1)
            for b, (k, kc) in enumerate(zip(list(accepted_count), list(key_count)))]
