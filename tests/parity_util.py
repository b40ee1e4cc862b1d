"""GPU-vs-oracle parity harness shared by the -m gpu tests, smoke() and bench.

Semantics contract (north_star / SURVEY.md §8(a)):
  * key masks, accept decisions, accepted lengths k, extra sources and emitted
    tokens are bit-exact with the fp64 oracle, EXCEPT where the oracle's own
    draw or clause sits within eps of its threshold; such "epsilon events" are
    counted and reported, never silently compared;
  * surprisals H and probabilities at y match within 1e-5 relative in fp32
    (with an absolute floor for surprisals near 0, where H = LSE - l_y cancels:
    |dH| <= 1e-5 |H| + 2e-6);
  * NormMatch is exact (a multiple of 1/m).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from oracle.oracle_lib import Oracle, philox_uniforms, window_uniforms

EPS_U = 1e-5        # |u - a_ref| band for accept draws
EPS_LAMBDA = 1e-5   # |clause - lambda| / max(1, lambda) band for key clauses
EPS_CDF = 1e-5      # normalised CDF margin of the extra draw
H_REL, H_ABS = 1e-5, 2e-6
P_REL, P_ABS = 1e-5, 1e-9


@dataclass
class ParityReport:
    sequences: int = 0
    positions_checked: int = 0
    eps_events: int = 0
    mismatches: list = field(default_factory=list)
    max_h_err: float = 0.0
    max_p_rel_err: float = 0.0
    ks: list = field(default_factory=list)

    def ok(self) -> bool:
        return not self.mismatches


def host_rows(t: torch.Tensor, V: int) -> np.ndarray:
    """fp64 copy of device logit rows (bf16/f32 values are exact in fp64)."""
    return t[..., :V].to(torch.float64).cpu().numpy()


def oracle_draft_tokens(oracle: Oracle, draft64: np.ndarray, seed: int, window: int,
                        sequence_offset: int = 0) -> np.ndarray:
    """Draft tokens sampled by the fp64 oracle with the Philox draft slots 0..gamma-1."""
    B, G, V = draft64.shape
    U = window_uniforms(seed, window, B, G, sequence_offset)
    toks = np.zeros((B, G), dtype=np.int32)
    for b in range(B):
        st, tok, _ = oracle.draft_tokens(draft64[b], U[b, :G])
        assert st == 0
        toks[b] = tok
    return toks


def position_stats(oracle: Oracle, dl: np.ndarray, tl: np.ndarray, y: int, tau: float, crit):
    """Reference per-position quantities at one (draft row, target row) pair."""
    _, pt = oracle.softmax(tl)
    _, pd = oracle.softmax(dl)
    key = oracle.is_key(pt, pd, y, crit)
    if key:
        eff = pt
    else:
        st, eff = oracle.soften(pt, pd, tau)
        if st != 0:
            return None
    _, a = oracle.accept_prob(eff, pd, y)
    m = min(crit.top_m, pt.size)
    return dict(h_target=oracle.cross_entropy(pt, y), h_draft=oracle.cross_entropy(pd, y),
                p_target_y=pt[y], p_draft_y=pd[y], norm_match=oracle.norm_match(pt, pd, m),
                key=key, p_eff_y=eff[y], accept_prob=a)


def _close(g, r, rel, ab):
    if np.isinf(r) or np.isinf(g):
        return np.isinf(r) and np.isinf(g)
    return abs(g - r) <= rel * abs(r) + ab


def compare_window(oracle: Oracle, draft64, target64, tokens, gpu: dict, tau: float, crit,
                   seed: int, window: int, sequence_offset: int = 0,
                   all_positions: bool = True) -> ParityReport:
    """Compare one dsdv_verify window (host copies in `gpu`) with the oracle."""
    B, G, V = draft64.shape
    U = window_uniforms(seed, window, B, G, sequence_offset)
    rep = ParityReport(sequences=B)
    for b in range(B):
        ref = oracle.verify_window(draft64[b], target64[b], tokens[b], tau, crit, U[b])
        rep.ks.append(ref["accepted_count"])
        g_status = int(gpu["status"][b])
        if ref["status"] != 0 or g_status != 0:
            if ref["status"] != g_status:
                rep.mismatches.append((b, "status", g_status, ref["status"]))
            continue
        # per-position numerics (evaluated positions via the window oracle,
        # the rest via the primitives)
        npos = G if all_positions else ref["evaluated"]
        for j in range(npos):
            if j < ref["evaluated"]:
                r = {k: ref[k][j] for k in ("h_target", "h_draft", "p_target_y", "p_draft_y",
                                            "norm_match", "p_eff_y", "accept_prob")}
                r["key"] = bool(ref["key"][j])
            else:
                r = position_stats(oracle, draft64[b, j], target64[b, j], int(tokens[b, j]), tau,
                                   crit)
                if r is None:
                    continue
            rep.positions_checked += 1
            for name, gname in (("h_target", "h_target"), ("h_draft", "h_draft")):
                g, rv = float(gpu[gname][b, j]), float(r[name])
                if not _close(g, rv, H_REL, H_ABS):
                    rep.mismatches.append((b, j, name, g, rv))
                elif np.isfinite(rv):
                    rep.max_h_err = max(rep.max_h_err, abs(g - rv) / (abs(rv) + 1e-12))
            for name, gname in (("p_target_y", "p_target_y"), ("p_draft_y", "p_draft_y")):
                g, rv = float(gpu[gname][b, j]), float(r[name])
                if not _close(g, rv, P_REL, P_ABS):
                    rep.mismatches.append((b, j, name, g, rv))
                else:
                    rep.max_p_rel_err = max(rep.max_p_rel_err, abs(g - rv) / (abs(rv) + 1e-300))
            if float(gpu["norm_match"][b, j]) != float(r["norm_match"]):
                rep.mismatches.append((b, j, "norm_match", float(gpu["norm_match"][b, j]),
                                       r["norm_match"]))
            gkey = bool(gpu["key_mask"][b, j])
            if gkey == r["key"]:
                # same effective distribution -> p_eff and a must agree numerically
                for name, gname in (("p_eff_y", "p_effective_y"), ("accept_prob", "accept_prob")):
                    g, rv = float(gpu[gname][b, j]), float(r[name])
                    if not _close(g, rv, P_REL, P_ABS):
                        rep.mismatches.append((b, j, name, g, rv))
        # decisions: bit-exact unless an epsilon event explains the divergence
        div = None
        for j in range(ref["evaluated"]):
            if bool(gpu["key_mask"][b, j]) != bool(ref["key"][j]):
                div = ("key", j, ref["margin_key"][j] < EPS_LAMBDA)
                break
            if bool(gpu["accepted"][b, j]) != bool(ref["accepted"][j]):
                div = ("accepted", j, ref["margin_u"][j] < EPS_U)
                break
        if div is None:
            same = (int(gpu["accepted_count"][b]) == ref["accepted_count"]
                    and int(gpu["extra_source"][b]) == ref["extra_source"]
                    and int(gpu["key_count"][b]) == ref["key_count"])
            if not same:
                rep.mismatches.append((b, "round", int(gpu["accepted_count"][b]),
                                       ref["accepted_count"]))
            elif int(gpu["extra_token"][b]) != ref["extra_token"]:
                if ref["margin_extra"] < EPS_CDF:
                    rep.eps_events += 1
                else:
                    rep.mismatches.append((b, "extra_token", int(gpu["extra_token"][b]),
                                           ref["extra_token"], ref["margin_extra"]))
        else:
            what, j, excused = div
            if excused:
                rep.eps_events += 1
            else:
                rep.mismatches.append((b, j, "decision:" + what))
    return rep


def _close_arr(g, r, rel, ab):
    """Elementwise _close over arrays (inf only matches inf)."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    inf = np.isinf(g) | np.isinf(r)
    with np.errstate(invalid="ignore"):
        fin = np.abs(g - r) <= rel * np.abs(r) + ab
    return np.where(inf, np.isinf(g) & np.isinf(r) & (np.sign(g) == np.sign(r)), fin)


def _to_np(x):
    return x.numpy() if hasattr(x, "numpy") else np.asarray(x)


def compare_batch(ref: dict, gpu: dict, all_positions: bool = True,
                  max_report: int = 50) -> ParityReport:
    """compare_window over a whole batch against Oracle.verify_batch output
    (one configuration). Same contract: numerics within tolerance at every
    position the oracle evaluated (and at the later ones when it supplied
    them), decisions bit-exact up to the first divergence, which must be an
    epsilon event (oracle margin inside the band) to be excused."""
    g = {k: _to_np(v) for k, v in gpu.items()}
    B, G = ref["key"].shape
    rep = ParityReport(sequences=B)
    rep.ks = ref["k"].tolist()
    rs, gs = ref["status"], g["status"].astype(np.int64)
    bad_status = rs != gs
    for b in np.nonzero(bad_status)[0][:max_report]:
        rep.mismatches.append((int(b), "status", int(gs[b]), int(rs[b])))
    ok_seq = (rs == 0) & (gs == 0)
    ev = ref["evaluated"]
    jj = np.arange(G)[None, :]
    # positions with oracle numerics: evaluated ones (+ later ones with a finite h)
    has = (jj < ev[:, None]) | (all_positions & ~np.isnan(ref["h_target"]))
    has &= ok_seq[:, None]
    rep.positions_checked = int(has.sum())

    def check(name, gname, rel, ab, mask=None):
        m = has if mask is None else (has & mask)
        okv = _close_arr(g[gname], ref[name], rel, ab) | ~m
        for b, j in zip(*np.nonzero(~okv)):
            if len(rep.mismatches) < max_report:
                rep.mismatches.append((int(b), int(j), name, float(g[gname][b, j]),
                                       float(ref[name][b, j])))
        return okv

    check("h_target", "h_target", H_REL, H_ABS)
    check("h_draft", "h_draft", H_REL, H_ABS)
    check("p_target_y", "p_target_y", P_REL, P_ABS)
    check("p_draft_y", "p_draft_y", P_REL, P_ABS)
    nm_bad = has & (g["norm_match"] != ref["norm_match"])
    for b, j in zip(*np.nonzero(nm_bad)):
        if len(rep.mismatches) < max_report:
            rep.mismatches.append((int(b), int(j), "norm_match", float(g["norm_match"][b, j]),
                                   float(ref["norm_match"][b, j])))
    same_key = g["key_mask"].astype(bool) == ref["key"].astype(bool)
    check("p_eff_y", "p_effective_y", P_REL, P_ABS, same_key)
    check("accept_prob", "accept_prob", P_REL, P_ABS, same_key)
    with np.errstate(invalid="ignore"):
        h_err = np.abs(g["h_target"] - ref["h_target"]) / (np.abs(ref["h_target"]) + 1e-12)
        p_err = np.abs(g["p_target_y"] - ref["p_target_y"]) / (np.abs(ref["p_target_y"]) + 1e-300)
    fin = has & np.isfinite(ref["h_target"]) & np.isfinite(h_err)
    if fin.any():
        rep.max_h_err = float(h_err[fin].max())
        rep.max_p_rel_err = float(p_err[fin & np.isfinite(p_err)].max())
    # decisions
    gk, ga = g["key_mask"].astype(bool), g["accepted"].astype(bool)
    rk, ra = ref["key"].astype(bool), ref["accepted"].astype(bool)
    for b in np.nonzero(ok_seq)[0]:
        n = int(ev[b])
        div = None
        for j in range(n):
            if gk[b, j] != rk[b, j]:
                div = ("key", j, ref["margin_key"][b, j] < EPS_LAMBDA)
                break
            if ga[b, j] != ra[b, j]:
                div = ("accepted", j, ref["margin_u"][b, j] < EPS_U)
                break
        if div is None:
            same = (int(g["accepted_count"][b]) == int(ref["k"][b])
                    and int(g["extra_source"][b]) == int(ref["extra_source"][b])
                    and int(g["key_count"][b]) == int(ref["key_count"][b]))
            if not same:
                rep.mismatches.append((int(b), "round", int(g["accepted_count"][b]),
                                       int(ref["k"][b])))
            elif int(g["extra_token"][b]) != int(ref["extra_token"][b]):
                if ref["margin_extra"][b] < EPS_CDF:
                    rep.eps_events += 1
                else:
                    rep.mismatches.append((int(b), "extra_token", int(g["extra_token"][b]),
                                           int(ref["extra_token"][b]),
                                           float(ref["margin_extra"][b])))
        else:
            what, j, excused = div
            if excused:
                rep.eps_events += 1
            else:
                rep.mismatches.append((int(b), j, "decision:" + what))
    return rep


def gpu_window(verifier, draft, target, tokens, V: int, tau: float, crit, seed: int,
               window: int = 0, out=None, raise_on_status: bool = True):
    """One dsdv_verify launch with per-position outputs; host dict of results."""
    from paper_2511_11733_b200.dsdv import VerifyParams
    p = VerifyParams(gamma=tokens.shape[1], tau=tau, ratio_limit=crit.ratio_limit,
                     gap_limit=crit.gap_limit, overlap_floor=crit.overlap_floor,
                     top_m=crit.top_m, seed=seed, window=window)
    o = verifier.verify(draft, target, tokens, p, vocab=V, out=out)
    if raise_on_status:
        verifier.sync(p, o, batch=tokens.shape[0], vocab=V)
    else:
        torch.cuda.synchronize()
    return o.to_host()


def host_logits(t: torch.Tensor) -> np.ndarray:
    """Host copy for Oracle.verify_batch: fp32 as is, bf16 as raw bits."""
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.float().cpu().numpy()


def run_gpu_window(verifier, dtype: torch.dtype, B: int, G: int, V: int, tau: float, crit,
                   seed: int = 1, window: int = 0, logits_seed: int = 42, stride=None,
                   oracle: Oracle | None = None):
    """Synthesise logits on the device, draw drafts with the oracle, verify on
    the GPU. Returns (draft64, target64, tokens, gpu_host_dict)."""
    from paper_2511_11733_b200.dsdv import VerifyParams
    oracle = oracle or Oracle()
    draft, target = verifier.synth_logits(B, G, V, dtype, logits_seed=logits_seed, stride=stride)
    torch.cuda.synchronize()
    d64, t64 = host_rows(draft, V), host_rows(target, V)
    toks = oracle_draft_tokens(oracle, d64, seed, window)
    tokens = torch.from_numpy(toks).to(draft.device)
    p = VerifyParams(gamma=G, tau=tau, ratio_limit=crit.ratio_limit, gap_limit=crit.gap_limit,
                     overlap_floor=crit.overlap_floor, top_m=crit.top_m, seed=seed, window=window)
    out = verifier.verify(draft, target, tokens, p, vocab=V)
    verifier.sync(p, out, batch=B, vocab=V)
    return d64, t64, toks, out.to_host(), (draft, target, tokens, p)
