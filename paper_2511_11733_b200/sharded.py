"""Vocabulary-sharded verification window.

Rank p of P holds the contiguous id slice [offset_p, offset_p + V_p) of every
draft / target row — the layout a tensor-parallel LM head produces. A window
is three device steps of libdsdv (csrc/shard.cu) around three small
collectives:

    dsdv_shard_stats  -> all_gather(records [B][G+1][8], top lists [B][G][2][m])
    dsdv_shard_merge  (every rank, identical: k, key flags, accept draws)
    dsdv_shard_sample(MASS) -> all_gather(masses [B])
    dsdv_shard_sample(RESOLVE) -> all_reduce_max(tokens [B])

Per window that is 392 B per position + 12 B per sequence per rank, the
"one sync per window" of DSD plus two [B]-sized exchanges for the emitted
token. `Comm` abstracts the collectives: `TorchComm` is torch.distributed
(NCCL on GPUs, gloo on CPU); `shard_slices` runs all P ranks of one window in
one process on one device (tests and single-GPU emulation).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import replace

import torch

from . import dsdv
from .dsdv import LIB, VerifyParams, Verifier, WindowResult

SHARD_MASS, SHARD_RESOLVE = 0, 1


def slice_bounds(vocab: int, nranks: int, rank: int, align: int = 8) -> tuple[int, int]:
    """Contiguous slice of rank `rank`: boundaries rounded to `align` ids so
    every slice starts on a 16-byte boundary of a bf16 / fp32 / fp64 row."""
    step = -(-vocab // nranks)
    step = -(-step // align) * align
    lo = min(vocab, rank * step)
    hi = min(vocab, lo + step)
    return lo, hi - lo


class TorchComm:
    """Collectives over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """[size, *t.shape]: every rank's tensor in rank (= shard) order."""
        flat = t.contiguous().reshape(-1)
        out = torch.empty(self.size * flat.numel(), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, flat, group=self.group)
        return out.view(self.size, *t.shape)

    def all_reduce_max(self, t: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t


class ShardedVerifier:
    """One rank of the vocabulary-sharded verifier."""

    def __init__(self, verifier: Verifier):
        self.v = verifier

    def _cp(self, p: VerifyParams, draft, target, tokens, vocab, offset, local):
        q = replace(p, vocab_offset=offset, vocab_local=local)
        return self.v.params(q, draft, target, tokens, vocab)

    # ---- the three device steps -------------------------------------------
    def stats(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
              stream=None):
        B, G, _ = draft.shape
        M = min(p.top_m, vocab)
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        rec = torch.empty((B, G + 1, dsdv.RECORD_WORDS), dtype=torch.float64, device=draft.device)
        topv = torch.empty((B, G, 2, M), dtype=torch.float64, device=draft.device)
        topi = torch.empty((B, G, 2, M), dtype=torch.int32, device=draft.device)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self.v._check(LIB.dsdv_shard_stats(self.v._h, C.byref(cp), draft.data_ptr(),
                                           target.data_ptr(), tokens.data_ptr(), rec.data_ptr(),
                                           topv.data_ptr(), topi.data_ptr(), s))
        return rec, topv, topi

    def merge(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
              rec_all, topv_all, topi_all, out: WindowResult | None = None, stream=None):
        B, G, _ = draft.shape
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        if out is None:
            out = WindowResult.allocate(B, G, draft.device, True, records=True)
        position = torch.empty(B, dtype=torch.int32, device=draft.device)
        u = torch.empty(B, dtype=torch.float64, device=draft.device)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self.v._check(LIB.dsdv_shard_merge(self.v._h, C.byref(cp), rec_all.shape[0],
                                           rec_all.data_ptr(), topv_all.data_ptr(),
                                           topi_all.data_ptr(), tokens.data_ptr(),
                                           C.byref(out._c), position.data_ptr(), u.data_ptr(), s))
        return out, position, u

    def sample(self, mode, rank, nranks, draft, target, tokens, p: VerifyParams, vocab: int,
               offset: int, local: int, out: WindowResult, position, u, masses_all=None,
               stream=None):
        B = draft.shape[0]
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        mass = torch.zeros(B, dtype=torch.float64, device=draft.device)
        tok = torch.full((B,), -1, dtype=torch.int32, device=draft.device)
        self.v._check(LIB.dsdv_shard_sample(
            self.v._h, C.byref(cp), mode, rank, nranks, draft.data_ptr(), target.data_ptr(),
            out.records.data_ptr(), position.data_ptr(), u.data_ptr(),
            masses_all.data_ptr() if masses_all is not None else None, mass.data_ptr(),
            tok.data_ptr(), out.status.data_ptr(), s))
        return mass if mode == SHARD_MASS else tok

    # ---- one window on this rank --------------------------------------------
    def verify(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
               comm: TorchComm, out: WindowResult | None = None, stream=None) -> WindowResult:
        rec, topv, topi = self.stats(draft, target, tokens, p, vocab, offset, local, stream)
        rec_all, topv_all, topi_all = comm.all_gather(rec), comm.all_gather(topv), comm.all_gather(topi)
        out, position, u = self.merge(draft, target, tokens, p, vocab, offset, local, rec_all,
                                      topv_all, topi_all, out, stream)
        mass = self.sample(SHARD_MASS, comm.rank, comm.size, draft, target, tokens, p, vocab,
                           offset, local, out, position, u, stream=stream)
        masses = comm.all_gather(mass)
        tok = self.sample(SHARD_RESOLVE, comm.rank, comm.size, draft, target, tokens, p, vocab,
                          offset, local, out, position, u, masses, stream=stream)
        out.extra_token.copy_(comm.all_reduce_max(tok))
        return out


def contiguous_slice(rows: torch.Tensor, lo: int, n: int) -> torch.Tensor:
    """Rows [.., lo:lo+n] as a 16-byte-aligned contiguous tensor (stride padded)."""
    vec = 16 // rows.element_size()
    stride = -(-n // vec) * vec
    out = torch.full((*rows.shape[:-1], stride), float("-inf"), dtype=rows.dtype,
                     device=rows.device)
    out[..., :n] = rows[..., lo:lo + n]
    return out


def shard_slices(verifier: Verifier, draft: torch.Tensor, target: torch.Tensor,
                 tokens: torch.Tensor, p: VerifyParams, vocab: int, nranks: int) -> WindowResult:
    """All `nranks` ranks of one sharded window in one process on one device:
    the same device steps, with the collectives done by stacking."""
    sv = ShardedVerifier(verifier)
    parts = []
    for r in range(nranks):
        lo, n = slice_bounds(vocab, nranks, r)
        parts.append((lo, n, contiguous_slice(draft, lo, n), contiguous_slice(target, lo, n)))
    stats = [sv.stats(d, t, tokens, p, vocab, lo, n) for lo, n, d, t in parts]
    rec_all = torch.stack([s[0] for s in stats])
    topv_all = torch.stack([s[1] for s in stats])
    topi_all = torch.stack([s[2] for s in stats])
    merged = [sv.merge(d, t, tokens, p, vocab, lo, n, rec_all, topv_all, topi_all)
              for lo, n, d, t in parts]
    masses = torch.stack([sv.sample(SHARD_MASS, r, nranks, d, t, tokens, p, vocab, lo, n,
                                    *merged[r]) for r, (lo, n, d, t) in enumerate(parts)])
    toks = torch.stack([sv.sample(SHARD_RESOLVE, r, nranks, d, t, tokens, p, vocab, lo, n,
                                  *merged[r], masses) for r, (lo, n, d, t) in enumerate(parts)])
    out = merged[0][0]
    out.extra_token.copy_(toks.max(dim=0).values)
    # every rank computed the same decisions; keep rank 0's
    return out
