"""Pipeline-sharded decoding emulation.

The reference models an N-node pipeline where every committed unit pays its
compute and then one synchronization round of N-1 sequential link hops
(`run_pipeline`, netsim.cpp:110-172; closed forms latency.cpp:63-86):

    standard decoding  one unit per token:       t0 + (N-1) t1
    DSD                one unit per window:      k t0 + (N-1) t1, commits k + 1

This module measures the same thing on GPUs: stage s of the N logical stages
lives on GPU s mod P; a unit is a device spin of its compute time on the GPU of
stage 0, then for every link an injected device spin of t1 followed by a
send/recv of the committed token ids to the next stage's GPU (NCCL when the
stages sit on different GPUs), and finally the commit returns to stage 0
(the next unit's input). The k values come from the GPU verifier. Reported:
measured R_comm = 1 - T_dsd / T_std over equal committed tokens, the
analytic comm_reduction_ratio at the mean committed length, the reference's
deterministic DES totals and the synchronization-round counts.
"""
from __future__ import annotations

from dataclasses import dataclass


# ---- closed forms (latency.cpp:63-86) -------------------------------------
def sync_cost(n_nodes: int, t1: float) -> float:
    return (n_nodes - 1) * t1


def standard_decode_time(tokens: float, n_nodes: int, t0: float, t1: float) -> float:
    return tokens * (t0 + sync_cost(n_nodes, t1))


def dsd_round_time(tokens: float, n_nodes: int, t0: float, t1: float) -> float:
    return tokens * t0 + sync_cost(n_nodes, t1)


def comm_reduction_ratio(tokens: float, n_nodes: int, t0: float, t1: float) -> float:
    return sync_cost(n_nodes, t1) * (tokens - 1.0) / (tokens * (t0 + sync_cost(n_nodes, t1)))


def expected_speedup(rho: float, mean_accepted: float, n_nodes: int, t0: float,
                     t1: float) -> float:
    """latency.cpp:88-95: (t0 + sync) / (t0 / rho + sync / mean_accepted)."""
    sync = sync_cost(n_nodes, t1)
    return (t0 + sync) / (t0 / rho + sync / mean_accepted)


def analytic_speedup(rho: float, mean_accepted: float, n_nodes: int, t0: float,
                     t1: float) -> float:
    """commands.cpp:64-71: the closed form, or 0 for degenerate runs."""
    if rho > 0.0 and mean_accepted >= 1.0:
        return expected_speedup(rho, mean_accepted, n_nodes, t0, t1)
    return 0.0


# ---- the reference's pipeline with constant link latency ------------------
@dataclass
class Unit:
    compute: float  # time units
    tokens: int     # committed by the unit


def standard_units(n_tokens: int, t0: float) -> list[Unit]:
    """simulate_standard (netsim.cpp:176-185): one unit per token."""
    return [Unit(t0, 1) for _ in range(n_tokens)]


def dsd_units(ks: list[int], t0: float) -> list[Unit]:
    """simulate_dsd (netsim.cpp:187-202): compute k t0, commit k + 1."""
    return [Unit(k * t0, k + 1) for k in ks]


def des_total(units: list[Unit], n_nodes: int, t1: float) -> float:
    """run_pipeline with a constant link sampler: units strictly sequential,
    each computes then crosses the N-1 links one after another."""
    now = 0.0
    for u in units:
        now += u.compute
        for _ in range(n_nodes - 1):
            now += t1
    return now


# ---- the device emulation --------------------------------------------------
class PipelineEmulator:
    """Runs units over N logical stages on the `comm` ranks (stage s on rank
    s mod P). The whole unit loop of a run is enqueued by one C-ABI call
    (dsdv_pipeline_run): device spins for the compute and the injected link
    latency, and across GPUs the hops are NVLink peer stores of the committed
    tokens into the next rank's CUDA-IPC-mapped buffer plus a per-source
    counter the receiver's stream waits on — no collective and no host round
    trip per hop. `comm` is a torch.distributed wrapper (None for one GPU)."""

    def __init__(self, verifier, n_stages: int, comm=None):
        import torch
        self.torch = torch
        self.v = verifier
        self.N = n_stages
        self.comm = comm
        self.P = comm.size if comm else 1
        self.rank = comm.rank if comm else 0
        self.dev = torch.device("cuda", verifier.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.ex = None
        if self.P > 1:
            from .sharded import PeerExchange
            self.ex = PeerExchange(verifier, self.P, self.rank, 64, comm=comm)
            if not self.ex.ok:
                raise RuntimeError("pipeline emulation: peer buffers could not be mapped")
        self.runs = 0

    def owner(self, s: int) -> int:
        return s % self.P

    def run(self, units: list[Unit], t1_ns: int) -> float:
        """Executes the units (compute in ns); returns elapsed device
        milliseconds (max over ranks when distributed)."""
        import ctypes as C
        from .dsdv import LIB
        torch = self.torch
        if self.comm:
            self.comm.dist.barrier()
        torch.cuda.synchronize(self.dev)
        self.runs += 1
        compute = (C.c_uint64 * max(1, len(units)))(*[int(u.compute) for u in units])
        bases = (C.c_void_p * self.P)(*(self.ex.bases if self.ex else [None]))
        stream = torch.cuda.current_stream(self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        self.v._check(LIB.dsdv_pipeline_run(
            self.v._h, self.N, self.P, self.rank, bases, self.ex.stride if self.ex else 0, compute,
            len(units), int(t1_ns), self.runs, int(60e9), self.status.data_ptr(),
            stream.cuda_stream))
        e1.record(stream)
        torch.cuda.synchronize(self.dev)
        if int(self.status.item()) != 0:
            raise RuntimeError("pipeline emulation: a hop timed out")
        ms = e0.elapsed_time(e1)
        if self.comm:
            t = torch.tensor([ms], device=self.dev)
            self.comm.all_reduce_max(t)
            ms = float(t.item())
        return ms
