"""CPU tests of the oracle (no GPU): the plain-C restatement is pinned against

  * the reference's own known-answer tests (proj/tests/test_verifier.cpp,
    proj/tests/test_distribution.cpp), replayed value for value;
  * acceptance criterion 6 (proj/tests/acceptance.cpp:257-288), whose recorded
    output is proj/test_output.txt:50 — this pins the whole RNG consumption
    order through generate();
  * the reference sources themselves (oracle/_ref, when built here), bit for
    bit on random windows.
"""
import math

import numpy as np
import pytest

from oracle.oracle_lib import (E_DEGENERATE_MIXTURE, E_DRAFTING_CONTRACT, E_EMPTY_RESIDUAL,
                               E_INVARIANT, philox_uniforms, window_uniforms)

INF = float("inf")
DIVERGENT_DRAFT = [0.15, 0.2, 0.25, 0.2, 0.1, 0.1]    # support/generators.hpp:77-85
DIVERGENT_TARGET = [0.45, 0.3, 0.1, 0.08, 0.04, 0.03]


# ---------------------------------------------------------------- test_verifier.cpp
def test_cross_entropy_kat(oracle):
    # test_verifier.cpp:80-87
    assert oracle.cross_entropy([1.0, 0.0], 0) == 0.0
    e = math.exp(-1.0)
    assert abs(oracle.cross_entropy([e, 1 - e], 0) - 1.0) <= 1e-12
    assert math.isinf(oracle.cross_entropy([1.0, 0.0], 1))


def test_norm_match_kat(oracle):
    # test_verifier.cpp:89-103
    p = [0.5, 0.3, 0.1, 0.1]
    assert oracle.norm_match(p, p, 2) == 1.0
    assert oracle.norm_match(p, p, 4) == 1.0
    assert oracle.norm_match([0.4, 0.4, 0.1, 0.1], [0.1, 0.1, 0.4, 0.4], 2) == 0.0
    assert oracle.norm_match([0.5, 0.3, 0.1, 0.1], [0.05, 0.5, 0.4, 0.05], 2) == 0.5
    assert oracle.norm_match([0.25] * 4, [0.25] * 4, 2) == 1.0
    assert math.isnan(oracle.norm_match(p, p, 5))


def test_is_key_clauses_kat(oracle):
    # test_verifier.cpp:105-137
    c = oracle.crit
    p = [0.7, 0.3]
    assert not oracle.is_key(p, p, 0, c(1.0, 0.5, 0.5, 2))
    assert oracle.is_key(p, p, 0, c(0.99, 1.0, 0.0, 2))
    assert oracle.is_key([0.9, 0.1], [0.3, 0.7], 0, c(INF, 0.5, 0.0, 2))
    assert not oracle.is_key([0.9, 0.1], [0.3, 0.7], 0, c(INF, 0.65, 0.0, 2))
    assert oracle.is_key([0.9, 0.1], [0.5, 0.5], 0, c(2.0, 1.0, 0.0, 2))
    assert oracle.is_key([0.9, 0.1], [0.1, 0.9], 1, c(INF, 1.0, 0.5, 1))
    assert not oracle.is_key(p, p, 0, c(INF, 1.0, 0.0, 1))
    # certain target guard
    assert oracle.is_key([1.0, 0.0], [0.9, 0.1], 0, c(INF, 1.0, 0.0, 2))
    assert not oracle.is_key([1.0, 0.0], [1.0, 0.0], 0, c(INF, 1.0, 0.0, 2))


def test_soften_kat(oracle):
    # test_verifier.cpp:170-191
    t, d = [0.9, 0.1], [0.5, 0.5]
    assert oracle.soften(t, d, 0.0)[1].tolist() == t
    assert oracle.soften(t, d, 1.0)[1].tolist() == d
    st, m = oracle.soften(t, d, 0.5)
    assert st == 0 and abs(m[0] - 0.75) <= 1e-12 and abs(m[1] - 0.25) <= 1e-12
    st, _ = oracle.soften([1.0, 0.0], [0.0, 1.0], 0.5)
    assert st == E_DEGENERATE_MIXTURE
    assert oracle.soften([1.0, 0.0], [0.0, 1.0], 0.0)[1].tolist() == [1.0, 0.0]


def test_accept_prob_and_residual_kat(oracle):
    # test_verifier.cpp:210-231
    d = [0.5, 0.5]
    assert oracle.accept_prob([0.9, 0.1], d, 0) == (0, 1.0)
    err, a = oracle.accept_prob([0.1, 0.9], d, 0)
    assert err == 0 and abs(a - 0.2) <= 1e-12
    assert oracle.accept_prob(d, d, 1) == (0, 1.0)
    assert oracle.accept_prob(d, [1.0, 0.0], 1)[0] == E_DRAFTING_CONTRACT
    assert oracle.residual([0.9, 0.1], d)[1].tolist() == [1.0, 0.0]
    assert oracle.residual([0.2, 0.3, 0.5], [0.5, 0.3, 0.2])[1].tolist() == [0.0, 0.0, 1.0]
    assert oracle.residual([1.0, 0.0], d)[1].tolist() == [1.0, 0.0]
    assert oracle.residual(d, d)[0] == E_EMPTY_RESIDUAL


def test_sample_with_uniform_kat(oracle):
    # test_distribution.cpp:96-109: boundary goes up
    half = [0.5, 0.5]
    assert oracle.sample_with_uniform(half, 0.3) == 0
    assert oracle.sample_with_uniform(half, 0.5) == 1
    assert oracle.sample_with_uniform(half, 0.9999) == 1
    assert oracle.sample_with_uniform([0.0, 1.0, 0.0], 0.7) == 1


# ---------------------------------------------------------------- acceptance criterion 6
def test_criterion6_tau_sweep_mean_lengths(oracle):
    """acceptance.cpp:257-288 recorded as test_output.txt:50:
    mean lengths [ 2.50364 3.02053 3.81058 5.06016 6.77729 ]."""
    c = oracle.crit(2.0, 0.2, 0.5, 6)
    out = []
    for tau in (0.0, 0.2, 0.4, 0.6, 0.8):
        total = rounds = 0
        for seed in range(1, 13):
            ks = oracle.generate_iid(DIVERGENT_DRAFT, DIVERGENT_TARGET, 8, tau, c, 256, seed)
            total += sum(k + 1 for k in ks)
            rounds += len(ks)
        out.append(float(f"{total / rounds:.6g}"))
    assert out == [2.50364, 3.02053, 3.81058, 5.06016, 6.77729]


def test_generate_matches_reference_round_by_round(oracle, ref_oracle):
    c = oracle.crit(2.0, 0.2, 0.5, 6)
    for tau in (0.0, 0.3, 1.0):
        for seed in (1, 7, 99):
            a = oracle.generate_iid(DIVERGENT_DRAFT, DIVERGENT_TARGET, 4, tau, c, 64, seed)
            b = ref_oracle.generate_iid(DIVERGENT_DRAFT, DIVERGENT_TARGET, 4, tau, c, 64, seed)
            assert a == b


# ---------------------------------------------------------------- Philox
def test_philox_numpy_matches_c_abi():
    from paper_2511_11733_b200 import dsdv
    for seed, window, seq, slot in [(1, 0, 0, 0), (42, 7, 3, 9), (2**40 + 5, 2**33 + 1, 255, 16)]:
        assert philox_uniforms(seed, window, seq, slot) == dsdv.uniform(seed, window, seq, slot)


def test_philox_uniforms_are_53_bit_in_unit_interval():
    u = window_uniforms(3, 1, 64, 8)
    assert u.shape == (64, 17)
    assert (u >= 0).all() and (u < 1).all()
    assert np.all((u * 2.0**53) == np.floor(u * 2.0**53))


# ---------------------------------------------------------------- restatement vs reference
def _random_window(rng, G, V, scale=3.0):
    """Correlated draft/target logit rows (target row G feeds the bonus draw)."""
    dl = rng.normal(size=(G, V)) * scale
    tl = rng.normal(size=(G + 1, V)) * scale
    tl[:G] = 0.6 * tl[:G] + 0.4 * dl
    return dl, tl


@pytest.mark.parametrize("V", [2, 6, 50, 1000])
@pytest.mark.parametrize("tau", [0.0, 0.2, 0.5, 1.0])
def test_restatement_bit_exact_vs_reference(oracle, ref_oracle, V, tau):
    rng = np.random.default_rng(V * 10 + int(tau * 10))
    G = 4
    for trial in range(6):
        dl, tl = _random_window(rng, G, V)
        U = window_uniforms(11 + trial, trial, 1, G)[0]
        st, tok, _ = oracle.draft_tokens(dl, U[:G])
        assert st == 0
        c = oracle.crit(1.5, 0.2, 0.5, min(6, V))
        a = oracle.verify_window(dl, tl, tok, tau, c, U)
        b = ref_oracle.verify_window(dl, tl, tok, tau, c, U)
        for k in ("accepted_count", "extra_token", "extra_source", "key_count", "status",
                  "evaluated"):
            assert a[k] == b[k], (k, a[k], b[k])
        n = a["evaluated"]
        assert (a["key"][:n] == b["key"][:n]).all()
        assert (a["accepted"][:n] == b["accepted"][:n]).all()
        assert (a["accept_prob"][:n] == b["accept_prob"][:n]).all()  # bit-exact fp64


def test_softmax_bit_exact_vs_reference(oracle, ref_oracle):
    rng = np.random.default_rng(5)
    for V in (2, 17, 4096):
        l = rng.normal(size=V) * 7
        l[rng.integers(0, V)] = -np.inf
        assert (oracle.softmax(l)[1] == ref_oracle.softmax(l)[1]).all()


def test_oracle_a_matches_oracle_b_on_iid_rows(oracle, ref_oracle):
    """verify_round unchanged (Oracle-A, categorical models + Philox stream) equals
    the restated per-position loop fed the same rows."""
    from oracle.oracle_lib import Oracle  # noqa: F401
    rng = np.random.default_rng(9)
    V, G = 40, 5
    for trial in range(10):
        ld = rng.normal(size=V) * 2
        lt = 0.5 * ld + rng.normal(size=V)
        _, pd = oracle.softmax(ld)
        _, pt = oracle.softmax(lt)
        c = oracle.crit(2.0, 0.2, 0.5, 6)
        A = ref_oracle.verify_round_iid(pd, pt, G, 0.3, c, seed=trial + 1, window=2, seq=trial)
        U = philox_uniforms(trial + 1, 2, trial, np.arange(2 * G + 1))
        # feed identical iid rows as "logits" = log p so that softmax returns p
        dl = np.tile(np.log(pd), (G, 1))
        tl = np.tile(np.log(pt), (G + 1, 1))
        B = oracle.verify_window(dl, tl, A["tokens"], 0.3, c, U)
        assert B["accepted_count"] == A["accepted_count"]
        assert B["extra_token"] == A["extra_token"]
        assert B["key_count"] == A["key_count"]


def test_errors_follow_the_reference_taxonomy(oracle):
    c = oracle.crit(2.0, 0.2, 0.5, 2)
    G, V = 2, 4
    U = window_uniforms(1, 0, 1, G)[0]
    dl = np.zeros((G, V))
    tl = np.zeros((G + 1, V))
    # token outside the vocabulary -> InvariantError
    r = oracle.verify_window(dl, tl, [V, 0], 0.2, c, U)
    assert r["status"] == E_INVARIANT
    # drafted token with zero draft probability -> DraftingContractError
    dl2 = dl.copy()
    dl2[0, 1] = -np.inf
    r = oracle.verify_window(dl2, tl, [1, 0], 0.0, c, U)
    assert r["status"] == E_DRAFTING_CONTRACT
    # a row without mass -> InvariantError
    tl2 = tl.copy()
    tl2[0, :] = -np.inf
    r = oracle.verify_window(dl, tl2, [0, 0], 0.2, c, U)
    assert r["status"] == E_INVARIANT


# ---------------------------------------------------------------- batched checker
@pytest.mark.parametrize("as_bf16", [False, True])
def test_verify_batch_matches_per_window_oracle(oracle, as_bf16):
    """Oracle.verify_batch (the checker of the full-window GPU tests) equals the
    per-sequence restatement on every field, for several configurations that
    share the softmaxed rows, with strided rows and bf16 bit inputs."""
    import torch
    from tests.parity_util import compare_batch, position_stats
    rng = np.random.default_rng(21 + as_bf16)
    B, G, V, stride = 7, 4, 1500, 1504
    d = np.zeros((B, G, stride), np.float32)
    t = np.zeros((B, G + 1, stride), np.float32)
    for b in range(B):
        dl, tl = _random_window(rng, G, V, scale=2.0 + b)
        d[b, :, :V], t[b, :, :V] = dl, tl
    if as_bf16:
        d = torch.from_numpy(d).bfloat16().float().numpy()
        t = torch.from_numpy(t).bfloat16().float().numpy()
    U = window_uniforms(5, 3, B, G)
    tok = np.zeros((B, G), np.int32)
    for b in range(B):
        tok[b] = oracle.draft_tokens(d[b, :, :V].astype(np.float64), U[b, :G])[1]
    tok[2, 1] = V + 3  # an out-of-vocabulary token -> InvariantError for that sequence
    cfgs = [(0.2, oracle.crit(2.0, 0.2, 0.5, 10)), (0.0, oracle.crit(1.2, 0.05, 0.8, 4)),
            (0.5, oracle.crit(float("inf"), 1.0, 0.0, 1))]
    if as_bf16:
        dd = torch.from_numpy(d).bfloat16().view(torch.int16).numpy().view(np.uint16)
        tt = torch.from_numpy(t).bfloat16().view(torch.int16).numpy().view(np.uint16)
    else:
        dd, tt = d, t
    res = oracle.verify_batch(dd, tt, tok, cfgs, U, V, all_positions=True, nthreads=3)
    for (tau, c), r in zip(cfgs, res):
        for b in range(B):
            w = oracle.verify_window(d[b, :, :V].astype(np.float64),
                                     t[b, :, :V].astype(np.float64), tok[b], tau, c, U[b])
            assert r["k"][b] == w["accepted_count"]
            assert r["extra_token"][b] == w["extra_token"]
            assert r["status"][b] == w["status"]
            assert r["evaluated"][b] == w["evaluated"]
            n = w["evaluated"]
            assert (r["key"][b, :n] == w["key"][:n]).all()
            assert (r["accepted"][b, :n] == w["accepted"][:n]).all()
            assert np.array_equal(r["accept_prob"][b, :n], w["accept_prob"][:n])
            assert np.array_equal(r["h_target"][b, :n], w["h_target"][:n])
            if w["status"] != 0:
                continue
            for j in range(n, G):
                if not 0 <= tok[b, j] < V:
                    assert np.isnan(r["h_target"][b, j])
                    continue
                ps = position_stats(oracle, d[b, j, :V].astype(np.float64),
                                    t[b, j, :V].astype(np.float64), int(tok[b, j]), tau, c)
                assert ps is not None
                assert r["h_draft"][b, j] == ps["h_draft"]
                assert r["norm_match"][b, j] == ps["norm_match"]
                assert bool(r["key"][b, j]) == ps["key"]
                assert r["accept_prob"][b, j] == ps["accept_prob"]
        # the checker accepts the oracle's own answers as a "GPU" result
        gpu = {"status": r["status"], "accepted_count": r["k"], "extra_token": r["extra_token"],
               "extra_source": r["extra_source"], "key_count": r["key_count"],
               "key_mask": r["key"], "accepted": r["accepted"], "accept_prob": r["accept_prob"],
               "h_target": r["h_target"], "h_draft": r["h_draft"],
               "p_target_y": r["p_target_y"], "p_draft_y": r["p_draft_y"],
               "norm_match": r["norm_match"], "p_effective_y": r["p_eff_y"]}
        rep = compare_batch(r, gpu)
        assert rep.ok(), rep.mismatches[:5]
        assert rep.eps_events == 0
        # and flags a flipped decision outside the epsilon band
        bad = {k: np.array(v, copy=True) for k, v in gpu.items()}
        b0 = int(np.nonzero(r["status"] == 0)[0][0])
        bad["accepted_count"][b0] += 1
        assert not compare_batch(r, bad).ok()
