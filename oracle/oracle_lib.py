"""Python access to the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker (never as the measured or
shipped path).

  Oracle    the plain-C restatement (oracle/dsd_oracle.c -> oracle/liboracle.so)
  RefOracle the reference's own sources compiled in place (oracle/_ref/libdsdref.so)
  philox_uniforms  an independent numpy restatement of include/dsdv/philox.h
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_ORACLE = HERE / "liboracle.so"
LIB_REF = HERE / "_ref" / "libdsdref.so"

OK, E_INVARIANT, E_DEGENERATE_MIXTURE, E_DRAFTING_CONTRACT, E_EMPTY_RESIDUAL = range(5)

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """make -C oracle (restatement always; _ref only where /root/reference exists)."""
    cmd = ["make", "-s", "-C", str(HERE)]
    if force:
        subprocess.run(["make", "-s", "-C", str(HERE), "clean"], check=True)
    subprocess.run(cmd, check=True)


# ----------------------------------------------------------------- Philox
_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox_bits(seed: int, window: int, sequence, slot) -> np.ndarray:
    """Philox4x32-10 words 0,1 as uint64 for counters (slot, sequence, window)."""
    slot = np.asarray(slot, dtype=np.uint64)
    sequence = np.asarray(sequence, dtype=np.uint64)
    c0, c1 = np.broadcast_arrays(slot & _MASK, sequence & _MASK)
    c0 = c0.astype(np.uint64)
    c1 = c1.astype(np.uint64)
    c2 = np.full_like(c0, window & 0xFFFFFFFF)
    c3 = np.full_like(c0, (window >> 32) & 0xFFFFFFFF)
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & _MASK, lo1, (hi0 ^ c3 ^ k1) & _MASK, lo0
        k0 = (k0 + np.uint64(_W0)) & _MASK
        k1 = (k1 + np.uint64(_W1)) & _MASK
    return (c1 << np.uint64(32)) | c0


def philox_uniforms(seed: int, window: int, sequence, slot) -> np.ndarray:
    bits = philox_bits(seed, window, sequence, slot)
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def window_uniforms(seed: int, window: int, batch: int, gamma: int, sequence_offset: int = 0):
    """[batch][2*gamma+1] slot-indexed draws (draft slots, accept slots, extra)."""
    seq = np.arange(batch, dtype=np.uint64)[:, None] + np.uint64(sequence_offset)
    slot = np.arange(2 * gamma + 1, dtype=np.uint64)[None, :]
    return np.ascontiguousarray(philox_uniforms(seed, window, seq, slot))


# ----------------------------------------------------------------- restatement
class _Crit(C.Structure):
    _fields_ = [("ratio_limit", C.c_double), ("gap_limit", C.c_double),
                ("overlap_floor", C.c_double), ("top_m", C.c_int)]


class _Result(C.Structure):
    _fields_ = [("accepted_count", C.c_int), ("extra_token", C.c_int), ("extra_source", C.c_int),
                ("key_count", C.c_int), ("status", C.c_int), ("evaluated", C.c_int),
                ("key", C.c_void_p), ("accepted", C.c_void_p), ("accept_prob", C.c_void_p),
                ("h_target", C.c_void_p), ("h_draft", C.c_void_p), ("p_target_y", C.c_void_p),
                ("p_draft_y", C.c_void_p), ("norm_match", C.c_void_p), ("p_eff_y", C.c_void_p),
                ("uniform", C.c_void_p), ("margin_u", C.c_void_p), ("margin_key", C.c_void_p),
                ("margin_extra", C.c_double)]


class _BatchOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "k", "extra_token", "extra_source", "key_count", "status", "evaluated", "margin_extra",
        "key", "accepted", "accept_prob", "h_target", "h_draft", "p_target_y", "p_draft_y",
        "norm_match", "p_eff_y", "margin_u", "margin_key")]


_BATCH_SEQ_I32 = ("k", "extra_token", "extra_source", "key_count", "status", "evaluated")
_BATCH_POS_F64 = ("accept_prob", "h_target", "h_draft", "p_target_y", "p_draft_y", "norm_match",
                  "p_eff_y", "margin_u", "margin_key")

_PER_POS_U8 = ("key", "accepted")
_PER_POS_F64 = ("accept_prob", "h_target", "h_draft", "p_target_y", "p_draft_y", "norm_match",
                "p_eff_y", "uniform", "margin_u", "margin_key")


class Oracle:
    """The plain-C restatement (oracle/dsd_oracle.c)."""

    def __init__(self, path: Path = LIB_ORACLE):
        if not path.exists():
            build()
        L = C.CDLL(str(path))
        L.oracle_softmax.argtypes = [_dp, C.c_int, _dp]
        L.oracle_cross_entropy.argtypes = [_dp, C.c_int, C.c_int]
        L.oracle_cross_entropy.restype = C.c_double
        L.oracle_norm_match.argtypes = [_dp, _dp, C.c_int, C.c_int]
        L.oracle_norm_match.restype = C.c_double
        L.oracle_is_key.argtypes = [_dp, _dp, C.c_int, C.c_int, C.POINTER(_Crit), C.c_void_p]
        L.oracle_soften.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp]
        L.oracle_accept_prob.argtypes = [_dp, _dp, C.c_int, C.POINTER(C.c_int)]
        L.oracle_accept_prob.restype = C.c_double
        L.oracle_residual.argtypes = [_dp, _dp, C.c_int, _dp]
        L.oracle_sample_with_uniform.argtypes = [_dp, C.c_int, C.c_double, C.c_void_p]
        L.oracle_verify_window_logits.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip, C.c_double,
                                                  C.POINTER(_Crit), _dp, C.POINTER(_Result)]
        L.oracle_draft_tokens.argtypes = [_dp, C.c_int, C.c_int, _dp, _ip, _dp]
        L.oracle_generate_iid.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double,
                                          C.POINTER(_Crit), C.c_int, C.c_uint64, _ip, C.c_int]
        L.oracle_verify_batch_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _fp, _fp, _ip,
                                              C.c_double, C.POINTER(_Crit), _dp, C.c_int, _ip,
                                              _ip, _ip]
        L.oracle_verify_batch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p, _ip, C.c_int, _dp, C.c_void_p, _dp, C.c_int,
                                          C.c_int, C.c_void_p]
        L.oracle_synth_logits.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_int]
        self.L = L

    def synth_logits(self, batch: int, gamma: int, vocab: int, bf16: bool, logits_seed: int = 42,
                     stride: int | None = None, nthreads=None):
        """The device's dsdv_synth_logits window on the host, bit for bit:
        (draft [B][gamma][stride], target [B][gamma+1][stride]) as fp32, or
        as raw bf16 bits (uint16) when bf16."""
        vec = 8 if bf16 else 4
        stride = stride or (vocab + vec - 1) // vec * vec
        dt = np.uint16 if bf16 else np.float32
        draft = np.empty((batch, gamma, stride), dt)
        target = np.empty((batch, gamma + 1, stride), dt)
        self.L.oracle_synth_logits(batch, gamma, vocab, stride, logits_seed, 1 if bf16 else 0,
                                   draft.ctypes.data, target.ctypes.data,
                                   nthreads or os.cpu_count() or 1)
        return draft, target

    @staticmethod
    def crit(ratio_limit=2.0, gap_limit=0.2, overlap_floor=0.5, top_m=10) -> _Crit:
        return _Crit(ratio_limit, gap_limit, overlap_floor, top_m)

    def softmax(self, logits) -> tuple[int, np.ndarray]:
        l = np.ascontiguousarray(logits, dtype=np.float64)
        p = np.empty_like(l)
        return self.L.oracle_softmax(l, l.size, p), p

    def cross_entropy(self, p, y) -> float:
        p = np.ascontiguousarray(p, dtype=np.float64)
        return self.L.oracle_cross_entropy(p, p.size, y)

    def norm_match(self, pt, pd, m) -> float:
        pt = np.ascontiguousarray(pt, dtype=np.float64)
        pd = np.ascontiguousarray(pd, dtype=np.float64)
        return self.L.oracle_norm_match(pt, pd, pt.size, m)

    def is_key(self, pt, pd, y, crit: _Crit) -> bool:
        pt = np.ascontiguousarray(pt, dtype=np.float64)
        pd = np.ascontiguousarray(pd, dtype=np.float64)
        return bool(self.L.oracle_is_key(pt, pd, pt.size, y, C.byref(crit), None))

    def soften(self, pt, pd, tau) -> tuple[int, np.ndarray]:
        pt = np.ascontiguousarray(pt, dtype=np.float64)
        pd = np.ascontiguousarray(pd, dtype=np.float64)
        out = np.empty_like(pt)
        return self.L.oracle_soften(pt, pd, pt.size, tau, out), out

    def accept_prob(self, eff, pd, y) -> tuple[int, float]:
        eff = np.ascontiguousarray(eff, dtype=np.float64)
        pd = np.ascontiguousarray(pd, dtype=np.float64)
        err = C.c_int(0)
        a = self.L.oracle_accept_prob(eff, pd, y, C.byref(err))
        return err.value, a

    def residual(self, eff, pd) -> tuple[int, np.ndarray]:
        eff = np.ascontiguousarray(eff, dtype=np.float64)
        pd = np.ascontiguousarray(pd, dtype=np.float64)
        out = np.empty_like(eff)
        return self.L.oracle_residual(eff, pd, eff.size, out), out

    def sample_with_uniform(self, p, u) -> int:
        p = np.ascontiguousarray(p, dtype=np.float64)
        return self.L.oracle_sample_with_uniform(p, p.size, u, None)

    def sample_with_margin(self, p, u) -> tuple[int, float]:
        """sample_with_uniform plus the CDF margin |u - nearest boundary|."""
        p = np.ascontiguousarray(p, dtype=np.float64)
        m = C.c_double(0.0)
        return self.L.oracle_sample_with_uniform(p, p.size, u, C.byref(m)), m.value

    def verify_window(self, draft_logits, target_logits, tokens, tau, crit: _Crit,
                      uniforms) -> dict:
        """One sequence: draft [gamma][V], target [gamma+1][V] (fp64 copies)."""
        dl = np.ascontiguousarray(draft_logits, dtype=np.float64)
        tl = np.ascontiguousarray(target_logits, dtype=np.float64)
        G, V = dl.shape
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        bufs = {n: np.zeros(G, dtype=np.uint8) for n in _PER_POS_U8}
        bufs.update({n: np.full(G, np.nan) for n in _PER_POS_F64})
        r = _Result()
        for n, arr in bufs.items():
            setattr(r, n, arr.ctypes.data)
        self.L.oracle_verify_window_logits(G, V, dl, tl, tok, tau, C.byref(crit), u, C.byref(r))
        out = {n: getattr(r, n) for n in ("accepted_count", "extra_token", "extra_source",
                                           "key_count", "status", "evaluated", "margin_extra")}
        out.update(bufs)
        return out

    def draft_tokens(self, draft_logits, uniforms) -> tuple[int, np.ndarray, np.ndarray]:
        dl = np.ascontiguousarray(draft_logits, dtype=np.float64)
        G, V = dl.shape
        tok = np.zeros(G, dtype=np.int32)
        margins = np.zeros(G, dtype=np.float64)
        st = self.L.oracle_draft_tokens(dl, G, V, np.ascontiguousarray(uniforms, np.float64), tok,
                                        margins)
        return st, tok, margins

    def generate_iid(self, pd, pt, gamma, tau, crit: _Crit, max_new, seed) -> list[int]:
        pd = np.ascontiguousarray(pd, dtype=np.float64)
        pt = np.ascontiguousarray(pt, dtype=np.float64)
        ks = np.zeros(max_new + 1, dtype=np.int32)
        n = self.L.oracle_generate_iid(pd, pt, pd.size, gamma, tau, C.byref(crit), max_new, seed,
                                       ks, ks.size)
        if n < 0:
            raise RuntimeError(f"oracle_generate_iid failed with status {-n}")
        return ks[:n].tolist()

    def verify_batch(self, draft, target, tokens, configs, uniforms, V, all_positions=False,
                     nthreads=None) -> list[dict]:
        """Parity checker over a whole batch: draft [B][gamma][stride],
        target [B][gamma+1][stride] as fp32 or raw bf16 bits (uint16);
        configs = [(tau, crit), ...] share the softmaxed rows. Returns one dict
        of numpy arrays per configuration (per sequence [B], per position
        [B][gamma]; NaN / 0 where the reference never evaluates)."""
        if draft.dtype == np.uint16:
            dtype = 1
        else:
            draft = draft.astype(np.float32, copy=False)
            target = target.astype(np.float32, copy=False)
            dtype = 0
        draft = np.ascontiguousarray(draft)
        target = np.ascontiguousarray(target)
        B, G, stride = draft.shape
        assert target.shape == (B, G + 1, stride)
        tok = np.ascontiguousarray(tokens, dtype=np.int32).reshape(B, G)
        U = np.ascontiguousarray(uniforms, dtype=np.float64).reshape(B, 2 * G + 1)
        n = len(configs)
        taus = np.ascontiguousarray([float(t) for t, _ in configs], dtype=np.float64)
        crits = (_Crit * n)(*[c for _, c in configs])
        res, outs = [], (_BatchOut * n)()
        for i in range(n):
            d = {k: np.zeros(B, np.int32) for k in _BATCH_SEQ_I32}
            d["margin_extra"] = np.full(B, np.inf)
            d["key"] = np.zeros((B, G), np.uint8)
            d["accepted"] = np.zeros((B, G), np.uint8)
            d.update({k: np.full((B, G), np.nan) for k in _BATCH_POS_F64})
            for k, a in d.items():
                setattr(outs[i], k, a.ctypes.data)
            res.append(d)
        self.L.oracle_verify_batch(B, G, V, stride, dtype, draft.ctypes.data, target.ctypes.data,
                                   tok, n, taus, C.cast(crits, C.c_void_p), U,
                                   1 if all_positions else 0, nthreads or os.cpu_count() or 1,
                                   C.cast(outs, C.c_void_p))
        return res

    def verify_batch_f32(self, draft, target, tokens, tau, crit: _Crit, uniforms, V,
                         nthreads=None):
        draft = np.ascontiguousarray(draft, dtype=np.float32)
        target = np.ascontiguousarray(target, dtype=np.float32)
        B, G, stride = draft.shape
        k = np.zeros(B, np.int32)
        e = np.zeros(B, np.int32)
        s = np.zeros(B, np.int32)
        self.L.oracle_verify_batch_f32(B, G, V, stride, draft, target,
                                       np.ascontiguousarray(tokens, np.int32), tau, C.byref(crit),
                                       np.ascontiguousarray(uniforms, np.float64),
                                       nthreads or os.cpu_count(), k, e, s)
        return k, e, s


# ----------------------------------------------------------------- reference
class RefOracle:
    """The reference's own verifier sources (oracle/_ref/libdsdref.so)."""

    @staticmethod
    def available() -> bool:
        return LIB_REF.exists()

    def __init__(self, path: Path = LIB_REF):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference; `make -C oracle`)")
        L = C.CDLL(str(path))
        L.ref_cross_entropy.argtypes = [_dp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_norm_match.argtypes = [_dp, _dp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_is_key.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.c_int, C.POINTER(C.c_int)]
        L.ref_soften.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp]
        L.ref_accept_prob.argtypes = [_dp, _dp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_residual.argtypes = [_dp, _dp, C.c_int, _dp]
        L.ref_sample_with_uniform.argtypes = [_dp, C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.ref_temperature_scale.argtypes = [_dp, C.c_int, C.c_double, _dp]
        L.ref_enumerate_first.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_double, C.c_double, C.c_int, _dp,
                                          C.POINTER(C.c_double)]
        L.ref_softmax.argtypes = [_dp, C.c_int, _dp]
        L.ref_seeded_uniform.argtypes = [C.c_uint64, C.c_int]
        L.ref_seeded_uniform.restype = C.c_double
        L.ref_verify_round_iid.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.c_int, C.c_uint64,
                                           C.c_uint64, C.c_uint32, _ip, _up, _up, _dp, _ip]
        L.ref_verify_window_logits.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip, C.c_double,
                                               C.c_double, C.c_double, C.c_double, C.c_int, _dp,
                                               _up, _up, _dp, _ip]
        L.ref_verify_batch_f32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _fp, _fp, _ip,
                                           C.c_double, C.c_double, C.c_double, C.c_double,
                                           C.c_int, _dp, C.c_int, _ip, _ip, _ip]
        L.ref_calibrate_c8.argtypes = [C.c_double, _dp, _dp, C.c_int]
        L.ref_generate_iid.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int, C.c_int, C.c_uint64, _ip,
                                       C.c_int]
        self.L = L

    @staticmethod
    def _a(x):
        return np.ascontiguousarray(x, dtype=np.float64)

    def softmax(self, logits):
        l = self._a(logits)
        p = np.empty_like(l)
        return self.L.ref_softmax(l, l.size, p), p

    def cross_entropy(self, p, y):
        p = self._a(p)
        out = C.c_double()
        st = self.L.ref_cross_entropy(p, p.size, y, C.byref(out))
        return st, out.value

    def norm_match(self, pt, pd, m):
        pt, pd = self._a(pt), self._a(pd)
        out = C.c_double()
        st = self.L.ref_norm_match(pt, pd, pt.size, m, C.byref(out))
        return st, out.value

    def is_key(self, pt, pd, y, ratio_limit, gap_limit, overlap_floor, top_m):
        pt, pd = self._a(pt), self._a(pd)
        out = C.c_int()
        st = self.L.ref_is_key(pt, pd, pt.size, y, ratio_limit, gap_limit, overlap_floor, top_m,
                               C.byref(out))
        return st, bool(out.value)

    def soften(self, pt, pd, tau):
        pt, pd = self._a(pt), self._a(pd)
        out = np.empty_like(pt)
        return self.L.ref_soften(pt, pd, pt.size, tau, out), out

    def accept_prob(self, eff, pd, y):
        eff, pd = self._a(eff), self._a(pd)
        out = C.c_double()
        st = self.L.ref_accept_prob(eff, pd, eff.size, y, C.byref(out))
        return st, out.value

    def residual(self, eff, pd):
        eff, pd = self._a(eff), self._a(pd)
        out = np.empty_like(eff)
        return self.L.ref_residual(eff, pd, eff.size, out), out

    def sample_with_uniform(self, p, u):
        p = self._a(p)
        out = C.c_int()
        st = self.L.ref_sample_with_uniform(p, p.size, u, C.byref(out))
        return st, out.value

    def seeded_uniform(self, seed, index):
        return self.L.ref_seeded_uniform(seed, index)

    def verify_round_iid(self, pd, pt, gamma, tau, crit, seed, window, seq):
        pd, pt = self._a(pd), self._a(pt)
        tok = np.zeros(gamma, np.int32)
        key = np.zeros(gamma, np.uint8)
        acc = np.zeros(gamma, np.uint8)
        ap = np.zeros(gamma, np.float64)
        res = np.zeros(5, np.int32)
        st = self.L.ref_verify_round_iid(pd, pt, pd.size, gamma, tau, crit.ratio_limit,
                                         crit.gap_limit, crit.overlap_floor, crit.top_m, seed,
                                         window, seq, tok, key, acc, ap, res)
        n = int(res[4])
        return dict(status=st, tokens=tok, key=key[:n], accepted=acc[:n], accept_prob=ap[:n],
                    accepted_count=int(res[0]), extra_token=int(res[1]),
                    extra_source=int(res[2]), key_count=int(res[3]))

    def verify_window(self, draft_logits, target_logits, tokens, tau, crit, uniforms):
        dl, tl = self._a(draft_logits), self._a(target_logits)
        G, V = dl.shape
        key = np.zeros(G, np.uint8)
        acc = np.zeros(G, np.uint8)
        ap = np.full(G, np.nan)
        res = np.zeros(6, np.int32)
        self.L.ref_verify_window_logits(G, V, dl, tl, np.ascontiguousarray(tokens, np.int32), tau,
                                        crit.ratio_limit, crit.gap_limit, crit.overlap_floor,
                                        crit.top_m, self._a(uniforms), key, acc, ap, res)
        return dict(accepted_count=int(res[0]), extra_token=int(res[1]), extra_source=int(res[2]),
                    key_count=int(res[3]), status=int(res[4]), evaluated=int(res[5]), key=key,
                    accepted=acc, accept_prob=ap)

    def verify_batch_f32(self, draft, target, tokens, tau, crit, uniforms, V, nthreads=None):
        draft = np.ascontiguousarray(draft, dtype=np.float32)
        target = np.ascontiguousarray(target, dtype=np.float32)
        B, G, stride = draft.shape
        k = np.zeros(B, np.int32)
        e = np.zeros(B, np.int32)
        s = np.zeros(B, np.int32)
        self.L.ref_verify_batch_f32(B, G, V, stride, draft, target,
                                    np.ascontiguousarray(tokens, np.int32), tau, crit.ratio_limit,
                                    crit.gap_limit, crit.overlap_floor, crit.top_m,
                                    self._a(uniforms), nthreads or os.cpu_count(), k, e, s)
        return k, e, s

    def calibrate_c8(self, budget):
        """Acceptance criterion 8 through the reference's calibrate_thresholds:
        (winner [len, divergence, ratio, gap, overlap], grid log [n][6])."""
        best = np.zeros(5)
        log = np.zeros((64, 6))
        n = self.L.ref_calibrate_c8(budget, best, log, 64)
        if n < 0:
            raise RuntimeError("ref_calibrate_c8 failed")
        return best, log[:n]

    def temperature_scale(self, p, T):
        p = self._a(p)
        out = np.zeros(p.size, np.float64)
        st = self.L.ref_temperature_scale(p, p.size, T, out)
        if st != 0:
            raise RuntimeError(f"ref_temperature_scale failed with status {-st}")
        return out

    def enumerate_first(self, pd, pt, gamma, tau, crit):
        """Exact distribution of the first committed token and E[accepted] of
        one round (enumerate_output_distribution / expected_accepted_count)."""
        pd, pt = self._a(pd), self._a(pt)
        out = np.zeros(pd.size, np.float64)
        ek = C.c_double()
        st = self.L.ref_enumerate_first(pd, pt, pd.size, gamma, tau, crit.ratio_limit,
                                        crit.gap_limit, crit.overlap_floor, crit.top_m, out,
                                        C.byref(ek))
        if st != 0:
            raise RuntimeError(f"ref_enumerate_first failed with status {-st}")
        return out, ek.value

    def generate_iid(self, pd, pt, gamma, tau, crit, max_new, seed):
        pd, pt = self._a(pd), self._a(pt)
        ks = np.zeros(max_new + 1, np.int32)
        n = self.L.ref_generate_iid(pd, pt, pd.size, gamma, tau, crit.ratio_limit, crit.gap_limit,
                                    crit.overlap_floor, crit.top_m, max_new, seed, ks, ks.size)
        if n < 0:
            raise RuntimeError(f"ref_generate_iid failed with status {-n}")
        return ks[:n].tolist()
