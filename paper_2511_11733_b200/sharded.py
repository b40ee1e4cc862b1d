"""Vocabulary-sharded verification window.

Rank p of P holds the contiguous id slice [offset_p, offset_p + V_p) of every
draft / target row — the layout a tensor-parallel LM head produces. A window
is three device steps of libdsdv (csrc/shard.cu) around three small
collectives:

    dsdv_shard_stats  -> all_gather(packed records [B][G+1][8] + top lists [B][G][2][m])
    dsdv_shard_merge  (every rank, identical: k, key flags, accept draws; this
                      slice's mass of the extra-draw row) -> all_gather(masses [B])
    dsdv_shard_sample(RESOLVE) -> all_reduce_max(tokens [B])

Per window that is one all-gather of a packed buffer (392 B per position at
m=10), the "one sync per window" of DSD, plus two [B]-sized exchanges for the
emitted token. `Comm` abstracts the collectives: `TorchComm` is torch.distributed
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
TILE_WORDS = 514  # DSDV_SHARD_TILE_WORDS


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
    @staticmethod
    def packed_layout(B: int, G: int, M: int):
        """Byte offsets of (records, top values, top ids) in one rank's packed
        exchange buffer, and its size (a multiple of 8)."""
        n_rec = B * (G + 1) * dsdv.RECORD_WORDS * 8
        n_tv = B * G * 2 * M * 8
        n_ti = B * G * 2 * M * 4
        size = -(-(n_rec + n_tv + n_ti) // 8) * 8
        return (0, n_rec, n_rec + n_tv), size

    def stats(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
              stream=None) -> torch.Tensor:
        """dsdv_shard_stats into one packed uint8 buffer (one all-gather)."""
        B, G, _ = draft.shape
        M = min(p.top_m, vocab)
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        (o_rec, o_tv, o_ti), size = self.packed_layout(B, G, M)
        buf = torch.empty(size, dtype=torch.uint8, device=draft.device)
        base = buf.data_ptr()
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self.v._check(LIB.dsdv_shard_stats(self.v._h, C.byref(cp), draft.data_ptr(),
                                           target.data_ptr(), tokens.data_ptr(), base + o_rec,
                                           base + o_tv, base + o_ti, s))
        return buf

    def merge(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
              packed_all: torch.Tensor, out: WindowResult | None = None, stream=None):
        """dsdv_shard_merge over the gathered packed buffers [P][size]."""
        B, G, _ = draft.shape
        M = min(p.top_m, vocab)
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        if out is None:
            out = WindowResult.allocate(B, G, draft.device, True, records=True)
        position = torch.empty(B, dtype=torch.int32, device=draft.device)
        u = torch.empty(B, dtype=torch.float64, device=draft.device)
        mass = torch.empty(B, dtype=torch.float64, device=draft.device)
        # tile sums of each extra-draw row, reused by the owner's RESOLVE
        self._tiles = torch.empty((B, TILE_WORDS), dtype=torch.float64, device=draft.device)
        (o_rec, o_tv, o_ti), size = self.packed_layout(B, G, M)
        assert packed_all.is_contiguous() and packed_all.shape[-1] == size
        base = packed_all.data_ptr()
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self.v._check(LIB.dsdv_shard_merge(self.v._h, C.byref(cp), packed_all.shape[0],
                                           base + o_rec, base + o_tv, base + o_ti, size,
                                           draft.data_ptr(), target.data_ptr(), tokens.data_ptr(),
                                           C.byref(out._c), position.data_ptr(), u.data_ptr(),
                                           mass.data_ptr(), self._tiles.data_ptr(), s))
        return out, position, u, mass

    def sample(self, mode, rank, nranks, draft, target, tokens, p: VerifyParams, vocab: int,
               offset: int, local: int, out: WindowResult, position, u, masses_all=None,
               stream=None, tiles=None):
        B = draft.shape[0]
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        mass = torch.zeros(B, dtype=torch.float64, device=draft.device)
        tok = torch.full((B,), -1, dtype=torch.int32, device=draft.device)
        self.v._check(LIB.dsdv_shard_sample(
            self.v._h, C.byref(cp), mode, rank, nranks, draft.data_ptr(), target.data_ptr(),
            out.records.data_ptr(), position.data_ptr(), u.data_ptr(),
            masses_all.data_ptr() if masses_all is not None else None, mass.data_ptr(),
            tok.data_ptr(), out.status.data_ptr(),
            tiles.data_ptr() if tiles is not None else None, s))
        return mass if mode == SHARD_MASS else tok

    # ---- one window on this rank --------------------------------------------
    def verify(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
               comm: TorchComm, out: WindowResult | None = None, stream=None) -> WindowResult:
        packed = self.stats(draft, target, tokens, p, vocab, offset, local, stream)
        out, position, u, mass = self.merge(draft, target, tokens, p, vocab, offset, local,
                                            comm.all_gather(packed), out, stream)
        masses = comm.all_gather(mass)
        tok = self.sample(SHARD_RESOLVE, comm.rank, comm.size, draft, target, tokens, p, vocab,
                          offset, local, out, position, u, masses, stream=stream,
                          tiles=self._tiles)
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
    svs = [ShardedVerifier(verifier) for _ in range(nranks)]  # one per rank (tile caches)
    parts = []
    for r in range(nranks):
        lo, n = slice_bounds(vocab, nranks, r)
        parts.append((lo, n, contiguous_slice(draft, lo, n), contiguous_slice(target, lo, n)))
    packed_all = torch.stack([svs[r].stats(d, t, tokens, p, vocab, lo, n)
                              for r, (lo, n, d, t) in enumerate(parts)])
    merged = [svs[r].merge(d, t, tokens, p, vocab, lo, n, packed_all)
              for r, (lo, n, d, t) in enumerate(parts)]
    masses = torch.stack([m[3] for m in merged])
    toks = torch.stack([svs[r].sample(SHARD_RESOLVE, r, nranks, d, t, tokens, p, vocab, lo, n,
                                      *merged[r][:3], masses, tiles=svs[r]._tiles)
                        for r, (lo, n, d, t) in enumerate(parts)])
    out = merged[0][0]
    out.extra_token.copy_(toks.max(dim=0).values)
    # every rank computed the same decisions; keep rank 0's
    return out
