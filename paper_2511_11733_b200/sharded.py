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

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)


class PeerExchange:
    """Exchange buffers of all ranks mapped into this process (CUDA IPC over
    NVLink): the stats kernel of every rank stores its packed records straight
    into slot `rank` of each rank's buffer (dsdv_shard_stats_peers), then a
    flag per rank (dsdv_peer_signal / dsdv_peer_wait) replaces the record
    all-gather. Two buffer sets alternate by window (the next window's stores
    never touch the set a slower peer may still be merging).

    `bases` may also be given directly: P virtual ranks in one process on one
    device (tests), where no IPC mapping is needed."""

    def __init__(self, verifier: Verifier, nranks: int, rank: int, size: int,
                 comm: "TorchComm | None" = None, bases: list[int] | None = None):
        self.v, self.P, self.rank = verifier, nranks, rank
        self.stride = -(-size // 256) * 256
        self.set_bytes = self.P * self.stride
        self.bytes = 2 * self.set_bytes + 8 * self.P  # two sets, then the flags
        self._owned, self._opened = [], []
        self.comm = comm
        self.ok = True
        if bases is not None:
            self.bases = list(bases)
            return
        # Every rank runs the same collectives whatever fails locally, so a
        # failure on one rank can never leave the others in a mismatched
        # collective: (1) local allocation and export, (2) all-gather of
        # (ok, handle), (3) open the peers, (4) all-gather of ok. On any
        # failure every rank releases what it holds (close()) and self.ok is
        # False on all of them.
        handle = (C.c_uint8 * 64)()
        ok = 1
        ptr = C.c_void_p()
        try:
            self.v._check(LIB.dsdv_dev_alloc(self.v._h, self.bytes, C.byref(ptr)))
            self._owned.append(ptr.value)
            self.v._check(LIB.dsdv_ipc_handle(self.v._h, ptr, handle))
        except Exception:  # noqa: BLE001  (reported through the collective flag)
            ok = 0
        mine = torch.tensor([ok] + list(bytearray(handle)), dtype=torch.uint8,
                            device=verifier.device)
        allh = comm.all_gather(mine).cpu()
        ok = int(allh[:, 0].min().item())
        self.bases = []
        if ok:
            try:
                for q in range(self.P):
                    if q == rank:
                        self.bases.append(ptr.value)
                        continue
                    h = (C.c_uint8 * 64)(*allh[q, 1:].tolist())
                    peer = C.c_void_p()
                    self.v._check(LIB.dsdv_ipc_open(self.v._h, h, C.byref(peer)))
                    self._opened.append(peer.value)
                    self.bases.append(peer.value)
            except Exception:  # noqa: BLE001
                ok = 0
        flags = comm.all_gather(torch.tensor([ok], dtype=torch.int32, device=verifier.device))
        self.ok = int(flags.min().item()) == 1
        if not self.ok:
            self.close()

    @staticmethod
    def allocate_local(verifier: Verifier, nranks: int, size: int) -> list[int]:
        """P exchange buffers on this device (the single-process emulation)."""
        stride = -(-size // 256) * 256
        out = []
        for _ in range(nranks):
            ptr = C.c_void_p()
            verifier._check(LIB.dsdv_dev_alloc(verifier._h, 2 * nranks * stride + 8 * nranks,
                                               C.byref(ptr)))
            out.append(ptr.value)
        return out

    def set_bases(self, epoch: int) -> list[int]:
        off = (epoch & 1) * self.set_bytes
        return [b + off for b in self.bases]

    def flag_bases(self) -> list[int]:
        """Bases whose [P * stride] offset is the flag array (signal / wait)."""
        return [b + 2 * self.set_bytes - self.P * self.stride for b in self.bases]

    def close(self):
        """Unmap the peers' buffers, wait until every rank has done the same
        (freeing an exported allocation while importers still map it is
        undefined), then free our own. Collective when a comm is attached."""
        for ptr in self._opened:
            LIB.dsdv_ipc_close(self.v._h, C.c_void_p(ptr))
        self._opened = []
        if self.comm is not None:
            torch.cuda.synchronize(self.v.device)
            self.comm.barrier()
        for ptr in self._owned:
            LIB.dsdv_dev_free(self.v._h, C.c_void_p(ptr))
        self._owned = []


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

    @staticmethod
    def exchange_layout(B: int, G: int, M: int):
        """One rank's slot in a peer-exchange set: the packed records, then its
        [B] slice masses and [B] RESOLVE tokens. Returns (offsets, size)."""
        (o_rec, o_tv, o_ti), size = ShardedVerifier.packed_layout(B, G, M)
        o_mass = -(-size // 8) * 8
        o_tok = o_mass + 8 * B
        return (o_rec, o_tv, o_ti, o_mass, o_tok), o_tok + 4 * B

    def signal_peers(self, ex: PeerExchange, value: int, stream=None, device=None):
        s = (stream or torch.cuda.current_stream(device)).cuda_stream
        flags = (C.c_void_p * ex.P)(*ex.flag_bases())
        self.v._check(LIB.dsdv_peer_signal(self.v._h, ex.P, ex.rank, flags, ex.stride, value, s))

    def stats_peers(self, ex: PeerExchange, epoch: int, draft, target, tokens,
                    p: VerifyParams, vocab: int, offset: int, local: int, stream=None,
                    flag: int | None = None):
        """dsdv_shard_stats_peers: this rank's records into every rank's buffer
        set `epoch & 1`, then its arrival flag (`flag`, default epoch) in every
        rank's buffer."""
        B, G, _ = draft.shape
        M = min(p.top_m, vocab)
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        (o_rec, o_tv, o_ti), size = self.packed_layout(B, G, M)
        assert ex.stride >= size
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        bases = (C.c_void_p * ex.P)(*ex.set_bases(epoch))
        self.v._check(LIB.dsdv_shard_stats_peers(
            self.v._h, C.byref(cp), draft.data_ptr(), target.data_ptr(), tokens.data_ptr(), ex.P,
            ex.rank, bases, ex.stride, o_rec, o_tv, o_ti, s))
        self.signal_peers(ex, epoch if flag is None else flag, stream, draft.device)

    def merge_peers(self, ex: PeerExchange, epoch: int, draft, target, tokens, p: VerifyParams,
                    vocab: int, offset: int, local: int, out: WindowResult | None = None,
                    stream=None):
        """dsdv_shard_merge_peers: records from this rank's buffer set, the slice
        masses stored into every rank's set. Returns (out, position, u)."""
        B, G, _ = draft.shape
        M = min(p.top_m, vocab)
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        if out is None:
            out = WindowResult.allocate(B, G, draft.device, True, records=True)
        position = torch.empty(B, dtype=torch.int32, device=draft.device)
        u = torch.empty(B, dtype=torch.float64, device=draft.device)
        self._tiles = torch.empty((B, TILE_WORDS), dtype=torch.float64, device=draft.device)
        (o_rec, o_tv, o_ti, o_mass, _), _ = self.exchange_layout(B, G, M)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        bases = (C.c_void_p * ex.P)(*ex.set_bases(epoch))
        self.v._check(LIB.dsdv_shard_merge_peers(
            self.v._h, C.byref(cp), ex.P, ex.rank, bases, ex.stride, o_rec, o_tv, o_ti, o_mass,
            draft.data_ptr(), target.data_ptr(), tokens.data_ptr(), C.byref(out._c),
            position.data_ptr(), u.data_ptr(), self._tiles.data_ptr(), s))
        return out, position, u

    def resolve_peers(self, ex: PeerExchange, epoch: int, draft, target, tokens,
                      p: VerifyParams, vocab: int, offset: int, local: int, out: WindowResult,
                      position, u, stream=None):
        """dsdv_shard_resolve_peers: masses from this rank's set, tokens into
        every rank's set."""
        B, G, _ = draft.shape
        cp = self._cp(p, draft, target, tokens, vocab, offset, local)
        (_, _, _, o_mass, o_tok), _ = self.exchange_layout(B, G, min(p.top_m, vocab))
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        bases = (C.c_void_p * ex.P)(*ex.set_bases(epoch))
        self.v._check(LIB.dsdv_shard_resolve_peers(
            self.v._h, C.byref(cp), ex.P, ex.rank, bases, ex.stride, o_mass, o_tok,
            draft.data_ptr(), target.data_ptr(), out.records.data_ptr(), position.data_ptr(),
            u.data_ptr(), out.status.data_ptr(), self._tiles.data_ptr(), s))

    def tokens_max_peers(self, ex: PeerExchange, epoch: int, B: int, G: int, M: int,
                         token_out: torch.Tensor, stream=None):
        (_, _, _, _, o_tok), _ = self.exchange_layout(B, G, M)
        s = (stream or torch.cuda.current_stream(token_out.device)).cuda_stream
        local = ex.set_bases(epoch)[ex.rank]
        self.v._check(LIB.dsdv_peer_tokens_max(self.v._h, ex.P, C.c_void_p(local), ex.stride,
                                               o_tok, B, token_out.data_ptr(), s))

    def wait_peers(self, ex: PeerExchange, epoch: int, status: torch.Tensor, stream=None,
                   timeout_s: float = 10.0):
        """Hold the stream until every rank's records of `epoch` have landed."""
        s = (stream or torch.cuda.current_stream(status.device)).cuda_stream
        local = ex.flag_bases()[ex.rank]
        self.v._check(LIB.dsdv_peer_wait(self.v._h, ex.P, C.c_void_p(local), ex.stride, epoch,
                                         int(timeout_s * 1e9), status.data_ptr(), s))

    def merge(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
              packed_all: torch.Tensor | tuple, out: WindowResult | None = None, stream=None):
        """dsdv_shard_merge over the gathered packed buffers [P][size], or over
        (base pointer, P, stride) of a peer-exchange buffer set."""
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
        if isinstance(packed_all, tuple):
            base, nranks, stride = packed_all
        else:
            assert packed_all.is_contiguous() and packed_all.shape[-1] == size
            base, nranks, stride = packed_all.data_ptr(), packed_all.shape[0], size
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self.v._check(LIB.dsdv_shard_merge(self.v._h, C.byref(cp), nranks,
                                           base + o_rec, base + o_tv, base + o_ti, stride,
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

    def _peer_failed(self) -> bool:
        """Did a flag round of an earlier window time out? Read without a sync:
        the status of the last window's first sequence (a timeout fails every
        sequence with DSDV_E_NCCL) is checked once it has landed."""
        ev = getattr(self, "_peer_event", None)
        if ev is None or not ev.query():
            return False
        return int(self._peer_status_host.item()) == dsdv.E_NCCL

    # ---- one window on this rank --------------------------------------------
    def verify(self, draft, target, tokens, p: VerifyParams, vocab: int, offset: int, local: int,
               comm: TorchComm, out: WindowResult | None = None, stream=None,
               exchange: str = "nccl") -> WindowResult:
        """One window on this rank. exchange="peer": the records travel by the
        stats kernel's own NVLink stores (PeerExchange) instead of an all-gather."""
        if exchange == "peer" and getattr(self, "peer_fallback", False):
            exchange = "nccl"
        if exchange == "peer":
            # no collective call: three flag rounds over the mapped buffers
            B, G, _ = draft.shape
            M = min(p.top_m, vocab)
            _, size = self.exchange_layout(B, G, M)
            ex = getattr(self, "_ex", None)
            if ex is not None and self._peer_failed():
                # a flag round of an earlier window timed out (a peer stalled or
                # died): that window already reported DSDV_E_NCCL in its statuses.
                # Fatal for the exchange: the buffer sets may hold stale records and
                # a peer may still write into them, so they are never reused.
                self._ex = None
                raise dsdv.DsdvError(dsdv.E_NCCL, "peer exchange: a flag round timed out in an "
                                     "earlier window; the exchange is unusable")
            if ex is None or ex.stride < size:
                if ex is not None:  # a larger window: remap (every rank does the same)
                    ex.close()
                    self._ex = None
                # collective setup; if any rank cannot map its peers (no CUDA IPC
                # / peer access), every rank falls back to the NCCL exchange
                ex = PeerExchange(self.v, comm.size, comm.rank, size, comm=comm)
                if not ex.ok:
                    self.peer_fallback = True
                    return self.verify(draft, target, tokens, p, vocab, offset, local, comm, out,
                                       stream, exchange="nccl")
                self._ex = ex
                self._epoch = 0
                self._peer_status = torch.zeros(1, dtype=torch.int32, device=draft.device)
                self._peer_status_host = torch.zeros(1, dtype=torch.int32).pin_memory()
                self._peer_event = None
            self._epoch += 1
            if out is None:
                out = WindowResult.allocate(B, G, draft.device, True, records=True)
            # the whole window in one C-ABI call: stats with peer stores, merge,
            # RESOLVE, tokens max, three flag rounds, timeout -> statuses
            cp = self._cp(p, draft, target, tokens, vocab, offset, local)
            cs = stream or torch.cuda.current_stream(draft.device)
            bases = (C.c_void_p * ex.P)(*ex.bases)
            self.v._check(LIB.dsdv_shard_verify_peers(
                self.v._h, C.byref(cp), draft.data_ptr(), target.data_ptr(), tokens.data_ptr(),
                ex.P, ex.rank, bases, ex.stride, self._epoch, int(10e9), C.byref(out._c),
                cs.cuda_stream))
            with torch.cuda.stream(cs):
                self._peer_status_host.copy_(out.status[:1], non_blocking=True)
                self._peer_event = torch.cuda.Event()
                self._peer_event.record(cs)
            return out
        else:
            packed = self.stats(draft, target, tokens, p, vocab, offset, local, stream)
            merged_in = comm.all_gather(packed)
        out, position, u, mass = self.merge(draft, target, tokens, p, vocab, offset, local,
                                            merged_in, out, stream)
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


def shard_slices_peer(verifier: Verifier, draft: torch.Tensor, target: torch.Tensor,
                      tokens: torch.Tensor, p: VerifyParams, vocab: int, nranks: int,
                      epoch: int = 1) -> WindowResult:
    """shard_slices with the peer exchange (the collective-free window of
    ShardedVerifier.verify(exchange="peer")): every virtual rank stores into all
    P exchange buffers — plain device buffers of this process instead of IPC
    mappings — with the same three flag rounds."""
    B, G, _ = draft.shape
    M = min(p.top_m, vocab)
    _, size = ShardedVerifier.exchange_layout(B, G, M)
    bases = PeerExchange.allocate_local(verifier, nranks, size)
    exs = [PeerExchange(verifier, nranks, r, size, bases=bases) for r in range(nranks)]
    svs = [ShardedVerifier(verifier) for _ in range(nranks)]
    parts = []
    for r in range(nranks):
        lo, n = slice_bounds(vocab, nranks, r)
        parts.append((lo, n, contiguous_slice(draft, lo, n), contiguous_slice(target, lo, n)))
    status = torch.zeros(1, dtype=torch.int32, device=draft.device)
    f = 3 * epoch
    for r, (lo, n, d, t) in enumerate(parts):
        svs[r].stats_peers(exs[r], epoch, d, t, tokens, p, vocab, lo, n, flag=f)
    merged = []
    for r, (lo, n, d, t) in enumerate(parts):
        svs[r].wait_peers(exs[r], f, status, timeout_s=2.0)
        merged.append(svs[r].merge_peers(exs[r], epoch, d, t, tokens, p, vocab, lo, n))
        svs[r].signal_peers(exs[r], f + 1, device=draft.device)
    for r, (lo, n, d, t) in enumerate(parts):
        svs[r].wait_peers(exs[r], f + 1, status, timeout_s=2.0)
        out, position, u = merged[r]
        svs[r].resolve_peers(exs[r], epoch, d, t, tokens, p, vocab, lo, n, out, position, u)
        svs[r].signal_peers(exs[r], f + 2, device=draft.device)
    for r in range(nranks):
        svs[r].wait_peers(exs[r], f + 2, status, timeout_s=2.0)
        svs[r].tokens_max_peers(exs[r], epoch, B, G, M, merged[r][0].extra_token)
    torch.cuda.synchronize(draft.device)
    assert int(status.item()) == 0, "peer wait timed out"
    for r in range(1, nranks):  # every rank holds the same window
        for k in ("accepted_count", "extra_token", "key_count", "status"):
            assert torch.equal(getattr(merged[r][0], k), getattr(merged[0][0], k)), k
    for b in bases:
        LIB.dsdv_dev_free(verifier._h, C.c_void_p(b))
    return merged[0][0]


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
