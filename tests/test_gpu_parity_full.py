"""Parity of the fused verifier at the configurations it is benchmarked on.

Every sequence of full windows is compared with the fp64 oracle
(Oracle.verify_batch, all host threads): C2 exactly as bench.py times it
(B=256, gamma=8, V=128256, bf16: 2,304 items, ~15.6 per CTA, so slot reuse,
both epilogue warps, queued sample requests and ring carry-over across items
of different kinds are all exercised), C3 at B=1024 (gamma=16, V=151936,
fp32: 17,408 items), the C3 tau x lambda grid of calibrate.cpp:25-31 at
B=160 (2,720 items per launch), and the batched error statuses of
verifier.cpp:32-37, :181-184, :188-196. Draft tokens are drawn on the device
(dsdv_draft_sample) as in the bench; the oracle takes them as given.

Contract (tests/parity_util.py): numerics within the stated tolerances at
every position, decisions bit-exact except where the oracle's own value is
within eps of its threshold (counted as eps events, which must stay rare).
"""
import itertools

import numpy as np
import pytest
import torch

from oracle.oracle_lib import (E_DEGENERATE_MIXTURE, E_DRAFTING_CONTRACT, E_INVARIANT, Oracle,
                               window_uniforms)
from tests.parity_util import compare_batch, gpu_window, host_logits

pytestmark = pytest.mark.gpu


def _window(verifier, dtype, B, G, V, logits_seed, draft_seed, window):
    from paper_2511_11733_b200.dsdv import VerifyParams
    draft, target = verifier.synth_logits(B, G, V, dtype, logits_seed=logits_seed)
    tokens = verifier.draft_sample(draft, VerifyParams(gamma=G, seed=draft_seed, window=window),
                                   vocab=V)
    torch.cuda.synchronize()
    return draft, target, tokens


def _report(rep, tag):
    print(f"[{tag}] sequences={rep.sequences} positions={rep.positions_checked} "
          f"eps_events={rep.eps_events} mismatches={len(rep.mismatches)} "
          f"max_h_rel={rep.max_h_err:.2e} max_p_rel={rep.max_p_rel_err:.2e}")


@pytest.mark.parametrize("seed,window", [(1, 0), (2, 7), (3, 12345)])
def test_c2_full_window_every_sequence(verifier, oracle, seed, window):
    """The benchmarked window itself: B=256, gamma=8, V=128256, bf16."""
    B, G, V = 256, 8, 128256
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    draft, target, tokens = _window(verifier, torch.bfloat16, B, G, V, 41 + seed, seed, window)
    gpu = gpu_window(verifier, draft, target, tokens, V, 0.2, crit, seed, window)
    ref = oracle.verify_batch(host_logits(draft), host_logits(target), tokens.cpu().numpy(),
                              [(0.2, crit)], window_uniforms(seed, window, B, G), V,
                              all_positions=True)[0]
    rep = compare_batch(ref, gpu)
    _report(rep, f"C2 seed={seed} window={window}")
    assert rep.ok(), rep.mismatches[:10]
    assert rep.eps_events <= 3, rep.eps_events
    assert rep.positions_checked == B * G
    # the decisions the bench reports (k, extra token) equal the oracle's
    # everywhere outside the eps events
    same_k = (gpu["accepted_count"].numpy() == ref["k"]).sum()
    assert same_k >= B - rep.eps_events


@pytest.mark.parametrize("tau,crit_args", [(0.0, (2.0, 0.2, 0.5, 10)),
                                           (0.5, (1.2, 0.05, 0.8, 4)),
                                           (1.0, (2.0, 0.2, 0.5, 10)),
                                           (0.2, (float("inf"), 1.0, 0.0, 32))])
def test_c2_window_tau_and_criteria(verifier, oracle, tau, crit_args):
    """The C2 window at the tau endpoints (no mix sum), a key-heavy criterion
    set, and no key criterion at all with the widest warp selection (m = 32)."""
    B, G, V = 256, 8, 128256
    crit = Oracle.crit(*crit_args)
    draft, target, tokens = _window(verifier, torch.bfloat16, B, G, V, 77, 4, 2)
    gpu = gpu_window(verifier, draft, target, tokens, V, tau, crit, 4, 2)
    ref = oracle.verify_batch(host_logits(draft), host_logits(target), tokens.cpu().numpy(),
                              [(tau, crit)], window_uniforms(4, 2, B, G), V,
                              all_positions=True)[0]
    rep = compare_batch(ref, gpu)
    _report(rep, f"C2 tau={tau} crit={crit_args}")
    assert rep.ok(), rep.mismatches[:10]
    assert rep.eps_events <= 3, rep.eps_events


def test_c3_full_batch_every_sequence(verifier, oracle):
    """C3 at full size: B=1024, gamma=16, V=151936, fp32 (20.5 GB per window)."""
    B, G, V = 1024, 16, 151936
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    draft, target, tokens = _window(verifier, torch.float32, B, G, V, 42, 5, 3)
    gpu = gpu_window(verifier, draft, target, tokens, V, 0.3, crit, 5, 3)
    d, t = host_logits(draft), host_logits(target)
    del draft, target
    torch.cuda.empty_cache()
    ref = oracle.verify_batch(d, t, tokens.cpu().numpy(), [(0.3, crit)],
                              window_uniforms(5, 3, B, G), V, all_positions=False)[0]
    rep = compare_batch(ref, gpu, all_positions=False)
    _report(rep, "C3 B=1024")
    assert rep.ok(), rep.mismatches[:10]
    assert rep.eps_events <= 10, rep.eps_events


TAUS = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5]
LAMBDAS = list(itertools.product([1.2, 2.0, 3.0], [0.05, 0.2], [0.3, 0.5, 0.8]))  # calibrate.cpp:25-31


def test_c3_tau_lambda_grid(verifier, oracle):
    """Every (tau, lambda1, lambda2, lambda3) point of the C3 sweep, B=160."""
    B, G, V = 160, 16, 151936
    draft, target, tokens = _window(verifier, torch.float32, B, G, V, 7, 9, 1)
    configs = [(tau, Oracle.crit(l1, l2, l3, 10)) for tau in TAUS for (l1, l2, l3) in LAMBDAS]
    from paper_2511_11733_b200.dsdv import WindowResult
    out = WindowResult.allocate(B, G, draft.device)
    gpus = []
    for tau, c in configs:
        gpus.append(gpu_window(verifier, draft, target, tokens, V, tau, c, 9, 1, out=out))
    refs = oracle.verify_batch(host_logits(draft), host_logits(target), tokens.cpu().numpy(),
                               configs, window_uniforms(9, 1, B, G), V, all_positions=False)
    eps = 0
    keys = 0
    for (tau, c), g, r in zip(configs, gpus, refs):
        rep = compare_batch(r, g, all_positions=False)
        assert rep.ok(), (tau, c.ratio_limit, c.gap_limit, c.overlap_floor, rep.mismatches[:5])
        eps += rep.eps_events
        keys += int(r["key_count"].sum())
    print(f"[C3 grid] {len(configs)} points x {B} sequences, eps_events={eps}, key tokens={keys}")
    assert eps <= len(configs) * B // 200
    assert keys > 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_batched_error_statuses(verifier, oracle, dtype):
    """Per-sequence statuses of a window, as the reference raises them:
    a token outside the vocabulary -> InvariantError (verifier.cpp:32-37),
    p_d(y) = 0 from a -inf draft logit -> DraftingContractError (:188-196),
    disjoint supports under KeyCriteria::none -> DegenerateMixtureError
    (:181-184); the other sequences of the window stay parity-green."""
    B, G, V = 12, 4, 5000
    draft, target, tokens = _window(verifier, dtype, B, G, V, 31, 4, 0)
    ninf = float("-inf")
    tokens[1, 0] = V + 7                           # out of vocabulary at position 0
    draft[2, 0, int(tokens[2, 0])] = ninf          # p_d(y) = 0 at position 0
    # disjoint supports at position 0 of sequence 3: target on even ids, draft on
    # odd ids, y odd (p_t(y) = 0: not key under none(), soften has no mass)
    target[3, 0, 1:V:2] = ninf
    draft[3, 0, 0:V:2] = ninf
    if int(tokens[3, 0]) % 2 == 0:
        tokens[3, 0] = int(tokens[3, 0]) + 1 if int(tokens[3, 0]) + 1 < V else 1
    torch.cuda.synchronize()
    crit = Oracle.crit(float("inf"), 1.0, 0.0, 1)  # KeyCriteria::none()
    gpu = gpu_window(verifier, draft, target, tokens, V, 0.5, crit, 4, 0, raise_on_status=False)
    ref = oracle.verify_batch(host_logits(draft), host_logits(target), tokens.cpu().numpy(),
                              [(0.5, crit)], window_uniforms(4, 0, B, G), V,
                              all_positions=False)[0]
    st = gpu["status"].numpy()
    assert ref["status"][1] == E_INVARIANT and st[1] == E_INVARIANT
    assert ref["status"][2] == E_DRAFTING_CONTRACT and st[2] == E_DRAFTING_CONTRACT
    assert ref["status"][3] == E_DEGENERATE_MIXTURE and st[3] == E_DEGENERATE_MIXTURE
    assert (st[4:] == 0).all() and st[0] == 0
    rep = compare_batch(ref, gpu, all_positions=False)
    assert rep.ok(), rep.mismatches[:10]
    # the drop-in's sync raises the first failing sequence's error class
    from paper_2511_11733_b200.dsdv import DsdvError, VerifyParams
    p = VerifyParams(gamma=G, tau=0.5, ratio_limit=float("inf"), gap_limit=1.0,
                     overlap_floor=0.0, top_m=1, seed=4)
    o = verifier.verify(draft, target, tokens, p, vocab=V)
    with pytest.raises(DsdvError) as ei:
        verifier.sync(p, o, batch=B, vocab=V)
    assert ei.value.status == E_INVARIANT


@pytest.mark.parametrize("dtype,B,G,V,tau", [(torch.bfloat16, 256, 8, 128256, 0.2),
                                             (torch.float32, 160, 16, 151936, 0.3)])
def test_early_exit_matches_oracle(verifier, oracle, dtype, B, G, V, tau):
    """dsdv_verify_early_exit: rows past a sequence's first rejection are not
    streamed, the round's results are the reference's."""
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    draft, target, tokens = _window(verifier, dtype, B, G, V, 44, 6, 2)
    from paper_2511_11733_b200.dsdv import VerifyParams
    p = VerifyParams(gamma=G, tau=tau, ratio_limit=2.0, gap_limit=0.2, overlap_floor=0.5,
                     top_m=10, seed=6, window=2)
    verifier.streamed_bytes(reset=True)
    full = verifier.verify(draft, target, tokens, p, vocab=V)
    verifier.sync(p, full, batch=B, vocab=V)
    full_bytes = verifier.streamed_bytes(reset=True)
    early = verifier.verify(draft, target, tokens, p, vocab=V, early_exit=True)
    verifier.sync(p, early, batch=B, vocab=V)
    early_bytes = verifier.streamed_bytes(reset=True)
    g = early.to_host()
    ref = oracle.verify_batch(host_logits(draft), host_logits(target), tokens.cpu().numpy(),
                              [(tau, crit)], window_uniforms(6, 2, B, G), V,
                              all_positions=False)[0]
    rep = compare_batch(ref, g, all_positions=False)
    _report(rep, f"early exit {dtype} B={B}")
    assert rep.ok(), rep.mismatches[:10]
    assert rep.eps_events <= 3
    f = full.to_host()
    for k in ("accepted_count", "extra_token", "extra_source", "key_count", "status"):
        assert torch.equal(f[k], g[k]), k
    print(f"[early exit] streamed {early_bytes / 1e9:.3f} GB vs {full_bytes / 1e9:.3f} GB full")
    assert early_bytes < 0.8 * full_bytes
