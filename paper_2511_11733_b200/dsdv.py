"""ctypes binding of the dsdv C-ABI (include/dsdv/dsdv.h).

PyTorch is used only for device memory and streams; every byte of verifier
arithmetic runs in libdsdv.so. There is no CPU fallback: if the library is
missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
# DSDV_LIB selects an alternate build of the same ABI (e.g. libdsdv_trace.so)
LIB_PATH = Path(os.environ["DSDV_LIB"]) if os.environ.get("DSDV_LIB") else _PKG / "libdsdv.so"

OK, E_INVARIANT, E_DEGENERATE_MIXTURE, E_DRAFTING_CONTRACT, E_EMPTY_RESIDUAL, E_CUDA, E_NCCL, \
    E_UNSUPPORTED = range(8)
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2
EXTRA_BONUS, EXTRA_RESIDUAL = 0, 1
RECORD_WORDS = 8

_TORCH_DTYPE = {DTYPE_F32: torch.float32, DTYPE_BF16: torch.bfloat16, DTYPE_F64: torch.float64}
_CODE_OF = {torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16, torch.float64: DTYPE_F64}


class DsdvError(RuntimeError):
    """Raised for a non-OK dsdv_status; `.status` carries the code."""

    def __init__(self, status: int, message: str):
        super().__init__(f"[dsdv status {status}] {message}")
        self.status = status


class _Params(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("gamma", C.c_int32), ("vocab", C.c_int32),
        ("row_stride", C.c_int32), ("dtype", C.c_int32), ("top_m", C.c_int32),
        ("tau", C.c_double), ("ratio_limit", C.c_double), ("gap_limit", C.c_double),
        ("overlap_floor", C.c_double), ("seed", C.c_uint64), ("window", C.c_uint64),
        ("sequence_offset", C.c_uint32), ("vocab_offset", C.c_int32),
        ("vocab_local", C.c_int32), ("eps_u", C.c_double), ("eps_lambda", C.c_double),
    ]


_OUT_FIELDS = [
    ("accepted_count", C.c_void_p), ("extra_token", C.c_void_p), ("extra_source", C.c_void_p),
    ("key_count", C.c_void_p), ("status", C.c_void_p), ("near_threshold", C.c_void_p),
    ("key_mask", C.c_void_p), ("accepted", C.c_void_p), ("accept_prob", C.c_void_p),
    ("h_target", C.c_void_p), ("h_draft", C.c_void_p), ("p_target_y", C.c_void_p),
    ("p_draft_y", C.c_void_p), ("norm_match", C.c_void_p), ("p_effective_y", C.c_void_p),
    ("uniform", C.c_void_p), ("records", C.c_void_p),
]


class _Outputs(C.Structure):
    _fields_ = _OUT_FIELDS


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    vp, st = C.c_void_p, C.c_int
    sigs = {
        "dsdv_create": (st, [C.c_int, C.POINTER(vp)]),
        "dsdv_destroy": (st, [vp]),
        "dsdv_last_error": (C.c_char_p, [vp]),
        "dsdv_abi_version": (C.c_int, []),
        "dsdv_validate": (st, [vp, C.POINTER(_Params)]),
        "dsdv_verify": (st, [vp, C.POINTER(_Params), vp, vp, vp, C.POINTER(_Outputs), vp]),
        "dsdv_verify_early_exit": (st, [vp, C.POINTER(_Params), vp, vp, vp, C.POINTER(_Outputs),
                                        vp]),
        "dsdv_streamed_bytes": (st, [vp, C.c_int, C.POINTER(C.c_uint64)]),
        "dsdv_shard_exchange_bytes": (C.c_uint64, [C.c_int32, C.c_int32, C.c_int32]),
        "dsdv_shard_verify_peers": (st, [vp, C.POINTER(_Params), vp, vp, vp, C.c_int32, C.c_int32,
                                         vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                         C.POINTER(_Outputs), vp]),
        "dsdv_pipeline_run": (st, [vp, C.c_int32, C.c_int32, C.c_int32, vp, C.c_uint64, vp,
                                   C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp]),
        "dsdv_log_rows": (st, [vp, vp, C.c_uint64, vp]),
        "dsdv_enable_peer_access": (st, [vp, C.c_int32]),
        "dsdv_calibrate": (st, [vp, vp, C.c_int32, vp, C.c_int64, vp, C.c_int32, C.c_double,
                                C.c_int32, C.c_double, vp]),
        "dsdv_window_stats_nm": (st, [vp, C.POINTER(_Params), vp, vp, vp, vp,
                                      C.POINTER(_Outputs), vp]),
        "dsdv_norm_match_scratch_bytes": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
        "dsdv_norm_match_rows": (st, [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      vp, C.c_size_t, vp, vp]),
        "dsdv_window_stats": (st, [vp, C.POINTER(_Params), vp, vp, vp, C.POINTER(_Outputs), vp]),
        "dsdv_sample_extra": (st, [vp, C.POINTER(_Params), vp, vp, vp, vp, vp, vp, vp, vp]),
        "dsdv_draft_sample": (st, [vp, C.POINTER(_Params), vp, vp, vp]),
        "dsdv_sync": (st, [vp, C.POINTER(_Params), vp, vp]),
        "dsdv_uniform": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]),
        "dsdv_synth_logits": (st, [vp, C.POINTER(_Params), C.c_uint64, vp, vp, vp]),
        "dsdv_launch_count": (C.c_uint64, [vp]),
        "dsdv_shard_stats": (st, [vp, C.POINTER(_Params), vp, vp, vp, vp, vp, vp, vp]),
        "dsdv_shard_merge": (st, [vp, C.POINTER(_Params), C.c_int32, vp, vp, vp, C.c_uint64, vp,
                                  vp, vp, C.POINTER(_Outputs), vp, vp, vp, vp, vp]),
        "dsdv_shard_sample": (st, [vp, C.POINTER(_Params), C.c_int32, C.c_int32, C.c_int32, vp,
                                   vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "dsdv_mix_rows": (st, [vp, C.c_int32, C.c_int32, vp, vp, C.c_double, vp, vp, vp]),
        "dsdv_spin": (st, [vp, C.c_uint64, vp]),
        "dsdv_draft_sample_temperature": (st, [vp, C.POINTER(_Params), C.c_double, vp, vp, vp]),
        "dsdv_dev_alloc": (st, [vp, C.c_uint64, C.POINTER(vp)]),
        "dsdv_dev_free": (st, [vp, vp]),
        "dsdv_ipc_handle": (st, [vp, vp, vp]),
        "dsdv_ipc_open": (st, [vp, vp, C.POINTER(vp)]),
        "dsdv_ipc_close": (st, [vp, vp]),
        "dsdv_shard_stats_peers": (st, [vp, C.POINTER(_Params), vp, vp, vp, C.c_int32, C.c_int32,
                                        vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp]),
        "dsdv_peer_signal": (st, [vp, C.c_int32, C.c_int32, vp, C.c_uint64, C.c_uint64, vp]),
        "dsdv_peer_wait": (st, [vp, C.c_int32, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp]),
        "dsdv_shard_merge_peers": (st, [vp, C.POINTER(_Params), C.c_int32, C.c_int32, vp,
                                        C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64, vp, vp, vp, C.POINTER(_Outputs), vp, vp, vp,
                                        vp]),
        "dsdv_shard_resolve_peers": (st, [vp, C.POINTER(_Params), C.c_int32, C.c_int32, vp,
                                          C.c_uint64, C.c_uint64, C.c_uint64, vp, vp, vp, vp, vp,
                                          vp, vp, vp]),
        "dsdv_peer_tokens_max": (st, [vp, C.c_int32, vp, C.c_uint64, C.c_uint64, C.c_int32, vp,
                                      vp]),
    }
    for name, (res, args) in sigs.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if LIB_PATH.name == "libdsdv.so":
                raise  # the product library must export the whole ABI
            continue  # an older development build (DSDV_LIB)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
EXPORTED = ("dsdv_create", "dsdv_destroy", "dsdv_last_error", "dsdv_abi_version", "dsdv_validate",
            "dsdv_verify", "dsdv_verify_early_exit", "dsdv_streamed_bytes",
            "dsdv_shard_exchange_bytes", "dsdv_shard_verify_peers", "dsdv_calibrate",
            "dsdv_pipeline_run", "dsdv_log_rows", "dsdv_enable_peer_access",
            "dsdv_window_stats_nm", "dsdv_norm_match_scratch_bytes", "dsdv_norm_match_rows", "dsdv_window_stats", "dsdv_sample_extra", "dsdv_draft_sample",
            "dsdv_sync", "dsdv_uniform", "dsdv_synth_logits", "dsdv_launch_count",
            "dsdv_shard_stats", "dsdv_shard_merge", "dsdv_shard_sample", "dsdv_mix_rows",
            "dsdv_spin", "dsdv_draft_sample_temperature", "dsdv_dev_alloc", "dsdv_dev_free",
            "dsdv_ipc_handle", "dsdv_ipc_open", "dsdv_ipc_close", "dsdv_shard_stats_peers",
            "dsdv_peer_signal", "dsdv_peer_wait", "dsdv_shard_merge_peers",
            "dsdv_shard_resolve_peers", "dsdv_peer_tokens_max")


def uniform(seed: int, window: int, sequence: int, slot: int) -> float:
    """The Philox draw the kernels use for (seed, window, sequence, slot)."""
    return LIB.dsdv_uniform(seed, window, sequence, slot)


@dataclass
class VerifyParams:
    """Mirror of dsd::VerifyParams + KeyCriteria (verifier.hpp:32-43, :86-92)
    plus the window-level fields of dsdv_params."""
    gamma: int = 8
    tau: float = 0.2
    ratio_limit: float = 2.0
    gap_limit: float = 0.2
    overlap_floor: float = 0.5
    top_m: int = 10
    seed: int = 1
    window: int = 0
    sequence_offset: int = 0
    vocab_offset: int = 0
    vocab_local: int | None = None
    eps_u: float = 1e-5
    eps_lambda: float = 1e-5

    def to_c(self, batch: int, vocab: int, row_stride: int, dtype: int) -> _Params:
        return _Params(batch, self.gamma, vocab, row_stride, dtype, self.top_m, self.tau,
                       self.ratio_limit, self.gap_limit, self.overlap_floor, self.seed,
                       self.window, self.sequence_offset, self.vocab_offset,
                       vocab if self.vocab_local is None else self.vocab_local, self.eps_u,
                       self.eps_lambda)


@dataclass
class WindowResult:
    """Device tensors written by one verification window."""
    accepted_count: torch.Tensor
    extra_token: torch.Tensor
    extra_source: torch.Tensor
    key_count: torch.Tensor
    status: torch.Tensor
    near_threshold: torch.Tensor
    key_mask: torch.Tensor | None = None
    accepted: torch.Tensor | None = None
    accept_prob: torch.Tensor | None = None
    h_target: torch.Tensor | None = None
    h_draft: torch.Tensor | None = None
    p_target_y: torch.Tensor | None = None
    p_draft_y: torch.Tensor | None = None
    norm_match: torch.Tensor | None = None
    p_effective_y: torch.Tensor | None = None
    uniform: torch.Tensor | None = None
    records: torch.Tensor | None = None
    _c: _Outputs = field(default=None, repr=False)

    @staticmethod
    def allocate(batch: int, gamma: int, device, per_position: bool = True,
                 records: bool = False) -> "WindowResult":
        """Zeroed outputs carved from one buffer (one fill launch, not one per field)."""
        f64 = (["accept_prob", "h_target", "h_draft", "p_target_y", "p_draft_y", "norm_match",
                "p_effective_y", "uniform"] if per_position else [])
        plan = [(n, torch.float64, (batch, gamma)) for n in f64]
        if records:
            plan.append(("records", torch.float64, (batch, gamma + 1, RECORD_WORDS)))
        plan += [(n, torch.int32, (batch,)) for n in
                 ("accepted_count", "extra_token", "key_count", "status", "near_threshold")]
        plan.append(("extra_source", torch.uint8, (batch,)))
        if per_position:
            plan += [("key_mask", torch.uint8, (batch, gamma)), ("accepted", torch.uint8, (batch, gamma))]
        sizes = []
        for _, dt, shp in plan:
            n = 1
            for d in shp:
                n *= d
            sizes.append(n * torch.empty((), dtype=dt).element_size())
        buf = torch.zeros(sum(-(-x // 8) * 8 for x in sizes), dtype=torch.uint8, device=device)
        r = WindowResult(*[None] * 6)
        off = 0
        for (name, dt, shp), nbytes in zip(plan, sizes):
            setattr(r, name, buf[off:off + nbytes].view(dt).view(shp))
            off += -(-nbytes // 8) * 8
        r._buf = buf
        r._c = _Outputs(*[(getattr(r, n).data_ptr() if getattr(r, n) is not None else None)
                          for n, _ in _OUT_FIELDS])
        return r

    def to_host(self) -> dict:
        return {n: getattr(self, n).cpu() for n, _ in _OUT_FIELDS if getattr(self, n) is not None}


class Verifier:
    """One dsdv context on one device (dsdv_create / dsdv_destroy)."""

    def __init__(self, device: int | torch.device = 0):
        if isinstance(device, torch.device):
            device = device.index or 0
        self.device = int(device)
        h = C.c_void_p()
        st = LIB.dsdv_create(self.device, C.byref(h))
        if st != OK:
            raise DsdvError(st, f"dsdv_create({self.device}) failed (no usable CUDA device?)")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            LIB.dsdv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(LIB.dsdv_launch_count(self._h))

    def _check(self, st: int):
        if st != OK:
            raise DsdvError(st, LIB.dsdv_last_error(self._h).decode())

    @staticmethod
    def _shape(draft: torch.Tensor, target: torch.Tensor, tokens: torch.Tensor):
        if draft.dim() != 3 or target.dim() != 3:
            raise ValueError("draft [B][gamma][stride], target [B][gamma+1][stride]")
        B, G, stride = draft.shape
        if tuple(target.shape) != (B, G + 1, stride):
            raise ValueError(f"target shape {tuple(target.shape)} != {(B, G + 1, stride)}")
        if tuple(tokens.shape) != (B, G) or tokens.dtype != torch.int32:
            raise ValueError("draft tokens must be int32 [B][gamma]")
        if draft.dtype != target.dtype or draft.dtype not in _CODE_OF:
            raise ValueError("logits must share one of f32/bf16/f64")
        for t in (draft, target, tokens):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("inputs must be contiguous CUDA tensors")
        return B, G, stride, _CODE_OF[draft.dtype]

    def params(self, p: VerifyParams, draft, target, tokens, vocab: int) -> _Params:
        B, G, stride, code = self._shape(draft, target, tokens)
        if G != p.gamma:
            raise ValueError(f"gamma {p.gamma} != draft rows {G}")
        return p.to_c(B, vocab, stride, code)

    def verify(self, draft: torch.Tensor, target: torch.Tensor, tokens: torch.Tensor,
               p: VerifyParams, vocab: int | None = None, out: WindowResult | None = None,
               stream: torch.cuda.Stream | None = None, per_position: bool = True,
               early_exit: bool = False) -> WindowResult:
        """dsdv_verify (or dsdv_verify_early_exit): one fused window for every
        sequence (asynchronous)."""
        vocab = draft.shape[-1] if vocab is None else vocab
        cp = self.params(p, draft, target, tokens, vocab)
        if out is None:
            out = WindowResult.allocate(cp.batch, cp.gamma, draft.device, per_position)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        fn = LIB.dsdv_verify_early_exit if early_exit else LIB.dsdv_verify
        self._check(fn(self._h, C.byref(cp), draft.data_ptr(), target.data_ptr(),
                       tokens.data_ptr(), C.byref(out._c), s))
        return out

    def streamed_bytes(self, reset: bool = False) -> int:
        """dsdv_streamed_bytes: logit bytes copied by the fused kernel (syncs)."""
        v = C.c_uint64(0)
        self._check(LIB.dsdv_streamed_bytes(self._h, 1 if reset else 0, C.byref(v)))
        return int(v.value)

    def window_stats(self, draft, target, tokens, p: VerifyParams, vocab: int | None = None,
                     out: WindowResult | None = None, stream=None) -> WindowResult:
        vocab = draft.shape[-1] if vocab is None else vocab
        cp = self.params(p, draft, target, tokens, vocab)
        if out is None:
            out = WindowResult.allocate(cp.batch, cp.gamma, draft.device, True, records=True)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self._check(LIB.dsdv_window_stats(self._h, C.byref(cp), draft.data_ptr(),
                                          target.data_ptr(), tokens.data_ptr(), C.byref(out._c), s))
        return out

    def sample_extra(self, draft, target, tokens, p: VerifyParams, records: torch.Tensor,
                     position: torch.Tensor, u: torch.Tensor, vocab: int | None = None,
                     stream=None):
        vocab = draft.shape[-1] if vocab is None else vocab
        cp = self.params(p, draft, target, tokens, vocab)
        tok = torch.empty(cp.batch, dtype=torch.int32, device=draft.device)
        st = torch.empty(cp.batch, dtype=torch.int32, device=draft.device)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self._check(LIB.dsdv_sample_extra(self._h, C.byref(cp), draft.data_ptr(),
                                          target.data_ptr(), records.data_ptr(),
                                          position.data_ptr(), u.data_ptr(), tok.data_ptr(),
                                          st.data_ptr(), s))
        return tok, st

    def draft_sample(self, draft: torch.Tensor, p: VerifyParams, vocab: int | None = None,
                     stream=None, temperature: float = 1.0) -> torch.Tensor:
        """dsdv_draft_sample(_temperature): tokens[b][j] ~ softmax(draft row / T)."""
        B, G, stride = draft.shape
        vocab = stride if vocab is None else vocab
        cp = p.to_c(B, vocab, stride, _CODE_OF[draft.dtype])
        tokens = torch.empty((B, G), dtype=torch.int32, device=draft.device)
        s = (stream or torch.cuda.current_stream(draft.device)).cuda_stream
        self._check(LIB.dsdv_draft_sample_temperature(self._h, C.byref(cp), float(temperature),
                                                      draft.data_ptr(), tokens.data_ptr(), s))
        return tokens

    def synth_logits(self, batch: int, gamma: int, vocab: int, dtype: torch.dtype,
                     logits_seed: int = 42, device=None, stride: int | None = None):
        device = device or torch.device("cuda", self.device)
        code = _CODE_OF[dtype]
        vec = 16 // torch.empty((), dtype=dtype).element_size()
        stride = stride or (vocab + vec - 1) // vec * vec
        draft = torch.empty((batch, gamma, stride), dtype=dtype, device=device)
        target = torch.empty((batch, gamma + 1, stride), dtype=dtype, device=device)
        cp = VerifyParams(gamma=gamma).to_c(batch, vocab, stride, code)
        s = torch.cuda.current_stream(device).cuda_stream
        self._check(LIB.dsdv_synth_logits(self._h, C.byref(cp), logits_seed, draft.data_ptr(),
                                          target.data_ptr(), s))
        return draft, target

    def spin(self, nanoseconds: int, stream=None) -> None:
        """dsdv_spin: hold the stream for `nanoseconds` of device time."""
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(LIB.dsdv_spin(self._h, int(nanoseconds), s))

    def sync(self, p: VerifyParams | None = None, out: WindowResult | None = None,
             batch: int = 0, vocab: int = 2, stream=None):
        """dsdv_sync: wait, then raise the first failing sequence's error."""
        s = (stream or torch.cuda.current_stream(torch.device("cuda", self.device))).cuda_stream
        if out is None:
            self._check(LIB.dsdv_sync(self._h, None, None, s))
            return
        cp = (p or VerifyParams()).to_c(batch or out.status.numel(), vocab, 8, 0)
        self._check(LIB.dsdv_sync(self._h, C.byref(cp), out.status.data_ptr(), s))


def validate(p: VerifyParams, batch: int = 1, vocab: int = 16, row_stride: int = 16,
             dtype: int = DTYPE_F32) -> None:
    """Host-only dsdv_validate (no device needed); raises DsdvError with the
    reference's message (verifier.cpp:55-91)."""
    cp = p.to_c(batch, vocab, row_stride, dtype)
    st = LIB.dsdv_validate(None, C.byref(cp))
    if st != OK:
        raise DsdvError(st, LIB.dsdv_last_error(None).decode())


def row_stride_for(vocab: int, dtype: torch.dtype) -> int:
    vec = 16 // torch.empty((), dtype=dtype).element_size()
    return int(math.ceil(vocab / vec) * vec)
