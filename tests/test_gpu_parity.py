"""Parity of the fused sm_100a verifier (dsdv_verify) with the fp64 oracle.

Runs through the C-ABI on the GPU. Inputs are the seeded synthetic row
families of SURVEY.md §8(d) (Zipf and Gaussian, b mod 4), generated on the
device and copied back; draft tokens are drawn by the oracle with the Philox
draft slots, exactly as verify_round's draft_window would (verifier.cpp:93-110).
"""
import numpy as np
import pytest
import torch

from tests.parity_util import compare_window, run_gpu_window

pytestmark = pytest.mark.gpu


def _crit(oracle, r=2.0, g=0.2, o=0.5, m=10):
    return oracle.crit(r, g, o, m)


def _check(rep, max_eps_frac=0.05):
    assert rep.ok(), rep.mismatches[:10]
    assert rep.eps_events <= max(1, int(max_eps_frac * rep.sequences)), rep.eps_events


def test_c1_shape_fp32(verifier, oracle):
    """C1: V=32000, gamma=4, tau=0.2, fp32 (batch 16 instead of 1 for coverage)."""
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.float32, 16, 4, 32000, 0.2,
                                       _crit(oracle), seed=1, oracle=oracle)
    rep = compare_window(oracle, d, t, tok, gpu, 0.2, _crit(oracle), seed=1, window=0)
    _check(rep)
    assert rep.positions_checked == 16 * 4


def test_c2_vocab_bf16(verifier, oracle):
    """C2 shape per sequence: V=128256, gamma=8, bf16 logits."""
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.bfloat16, 8, 8, 128256, 0.2,
                                       _crit(oracle), seed=2, oracle=oracle)
    rep = compare_window(oracle, d, t, tok, gpu, 0.2, _crit(oracle), seed=2, window=0)
    _check(rep)


@pytest.mark.parametrize("tau", [0.1, 0.3, 0.5])
def test_c3_shape_fp32(verifier, oracle, tau):
    """C3 per sequence: V=151936 (Qwen), gamma=16, fp32, tau in the C3 sweep."""
    crit = _crit(oracle, 2.5, 0.15, 0.4, 10)
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.float32, 4, 16, 151936, tau, crit,
                                       seed=3, oracle=oracle)
    rep = compare_window(oracle, d, t, tok, gpu, tau, crit, seed=3, window=0)
    _check(rep)


@pytest.mark.parametrize("tau", [0.0, 0.5, 1.0])
def test_tau_endpoints_and_mid(verifier, oracle, tau):
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.float32, 12, 6, 5000, tau,
                                       _crit(oracle), seed=3, oracle=oracle)
    rep = compare_window(oracle, d, t, tok, gpu, tau, _crit(oracle), seed=3, window=0)
    _check(rep)


@pytest.mark.parametrize("V,tau", [(32000, 0.2), (5001, 0.5), (151936, 1.0)])
def test_fp64_logits_full_window(verifier, oracle, V, tau):
    """fp64 logit rows through the batched dsdv_verify (the drop-in's row type):
    fp64 accumulation in the fold, the fp64 sample items, ragged 2-id vectors."""
    from paper_2511_11733_b200.dsdv import VerifyParams
    from tests.parity_util import host_rows, oracle_draft_tokens
    B, G = 12, 4
    crit = _crit(oracle)
    d32, t32 = verifier.synth_logits(B, G, V, torch.float32, logits_seed=17)
    stride = -(-V // 2) * 2  # 16-byte rows of fp64
    draft = torch.full((B, G, stride), float("-inf"), dtype=torch.float64, device=d32.device)
    target = torch.full((B, G + 1, stride), float("-inf"), dtype=torch.float64, device=d32.device)
    draft[..., :V] = d32[..., :V].double()
    target[..., :V] = t32[..., :V].double()
    d64, t64 = host_rows(draft, V), host_rows(target, V)
    toks = oracle_draft_tokens(oracle, d64, 6, 1)
    tokens = torch.from_numpy(toks).to(draft.device)
    p = VerifyParams(gamma=G, tau=tau, ratio_limit=crit.ratio_limit, gap_limit=crit.gap_limit,
                     overlap_floor=crit.overlap_floor, top_m=crit.top_m, seed=6, window=1)
    out = verifier.verify(draft, target, tokens, p, vocab=V)
    verifier.sync(p, out, batch=B, vocab=V)
    rep = compare_window(oracle, d64, t64, toks, out.to_host(), tau, crit, seed=6, window=1)
    _check(rep)


def test_sequence_offset_selects_the_philox_streams(verifier, oracle):
    """A replica's window (sequence_offset = its first global sequence id) draws
    the uniforms of those global sequences (the replicas mode of bench.py)."""
    from paper_2511_11733_b200.dsdv import VerifyParams
    from tests.parity_util import host_rows, oracle_draft_tokens
    B, G, V, off = 8, 4, 6000, 1000
    crit = _crit(oracle)
    draft, target = verifier.synth_logits(B, G, V, torch.float32, logits_seed=23)
    d64, t64 = host_rows(draft, V), host_rows(target, V)
    toks = oracle_draft_tokens(oracle, d64, 9, 2, sequence_offset=off)
    tokens = torch.from_numpy(toks).to(draft.device)
    p = VerifyParams(gamma=G, tau=0.3, ratio_limit=crit.ratio_limit, gap_limit=crit.gap_limit,
                     overlap_floor=crit.overlap_floor, top_m=crit.top_m, seed=9, window=2,
                     sequence_offset=off)
    out = verifier.verify(draft, target, tokens, p, vocab=V)
    verifier.sync(p, out, batch=B, vocab=V)
    gpu = out.to_host()
    rep = compare_window(oracle, d64, t64, toks, gpu, 0.3, crit, seed=9, window=2,
                         sequence_offset=off)
    _check(rep)
    # the accept uniforms it used are those of the offset sequences
    from oracle.oracle_lib import window_uniforms
    U_off = window_uniforms(9, 2, B, G, off)
    U_0 = window_uniforms(9, 2, B, G, 0)
    assert not np.array_equal(U_off, U_0)
    np.testing.assert_array_equal(gpu["uniform"].reshape(B, G), U_off[:, G:2 * G])


@pytest.mark.parametrize("V", [2, 7, 1000, 4099])
def test_ragged_vocab(verifier, oracle, V):
    """Vocabularies that are not a multiple of the vector / chunk width."""
    m = min(10, V)
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.float32, 8, 3, V, 0.3,
                                       _crit(oracle, m=m), seed=4, oracle=oracle)
    rep = compare_window(oracle, d, t, tok, gpu, 0.3, _crit(oracle, m=m), seed=4, window=0)
    _check(rep)


def test_all_key_thresholds(verifier, oracle):
    """gap_limit 0 and ratio 1e-9 mark everything key (acceptance.cpp:204)."""
    c = _crit(oracle, r=1e-9, g=0.0, o=1.0, m=1)
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.float32, 8, 4, 3000, 0.9, c, seed=5,
                                       oracle=oracle)
    rep = compare_window(oracle, d, t, tok, gpu, 0.9, c, seed=5, window=0)
    _check(rep)
    assert gpu["key_mask"].all()


def test_no_key_tau_one_accepts_everything(verifier, oracle):
    """KeyCriteria::none() + tau=1: every window is accepted (test_verifier.cpp:245-254)."""
    c = _crit(oracle, r=float("inf"), g=1.0, o=0.0, m=1)
    d, t, tok, gpu, _ = run_gpu_window(verifier, torch.float32, 16, 4, 2000, 1.0, c, seed=6,
                                       oracle=oracle)
    assert (gpu["accepted_count"] == 4).all()
    assert (gpu["extra_source"] == 0).all()
    assert not gpu["key_mask"].any()


def test_identical_rows_accept_whole_window(verifier, oracle):
    """Identical draft/target rows: a == 1 everywhere (test_verifier.cpp:233-243)."""
    from paper_2511_11733_b200.dsdv import VerifyParams
    B, G, V = 8, 5, 3001
    draft, target = verifier.synth_logits(B, G, V, torch.float32, logits_seed=9)
    target[:, :G].copy_(draft)
    tokens = torch.randint(0, V, (B, G), dtype=torch.int32, device=draft.device)
    p = VerifyParams(gamma=G, tau=0.0, ratio_limit=float("inf"), gap_limit=1.0,
                     overlap_floor=0.0, top_m=1, seed=7)
    out = verifier.verify(draft, target, tokens, p, vocab=V)
    verifier.sync(p, out, batch=B, vocab=V)
    h = out.to_host()
    assert (h["accepted_count"] == G).all()
    assert (h["accept_prob"] == 1.0).all()


def test_windows_are_independent_of_launch_history(verifier, oracle):
    """Same inputs, same seed/window -> bit-identical results across launches
    (test_verifier.cpp:306-324); a different window index changes the draws."""
    d, t, tok, gpu1, (draft, target, tokens, p) = run_gpu_window(
        verifier, torch.bfloat16, 16, 8, 20000, 0.2, _crit(oracle), seed=11, oracle=oracle)
    outs = []
    for _ in range(3):
        o = verifier.verify(draft, target, tokens, p, vocab=20000)
        verifier.sync(p, o, batch=16, vocab=20000)
        outs.append(o.to_host())
    for o in outs:
        for k in ("accepted_count", "extra_token", "extra_source", "key_mask", "accept_prob"):
            assert torch.equal(o[k], gpu1[k]), k


def test_draft_sample_matches_oracle(verifier, oracle):
    """Draft-side step (draft_window, verifier.cpp:93-110) on the device."""
    from paper_2511_11733_b200.dsdv import VerifyParams
    from tests.parity_util import host_rows, oracle_draft_tokens
    B, G, V = 16, 4, 32000
    draft, _ = verifier.synth_logits(B, G, V, torch.float32, logits_seed=13)
    p = VerifyParams(gamma=G, seed=21, window=3)
    tok = verifier.draft_sample(draft, p, vocab=V).cpu().numpy()
    torch.cuda.synchronize()
    from oracle.oracle_lib import window_uniforms
    from tests.parity_util import EPS_CDF
    rows = host_rows(draft, V)
    U = window_uniforms(21, 3, B, G)
    eps = 0
    for b in range(B):
        st, ref, margins = oracle.draft_tokens(rows[b], U[b, :G])
        assert st == 0
        for j in range(G):
            if tok[b, j] != ref[j]:
                # only a draw within eps of a CDF boundary may land on the neighbour
                assert margins[j] < EPS_CDF, (b, j, tok[b, j], ref[j], margins[j])
                eps += 1
    assert eps <= 2, eps


@pytest.mark.parametrize("T", [0.0, 0.5, 1.7])
def test_draft_sample_under_temperature(verifier, ref_oracle, T):
    """temperature_scale (distribution.cpp:65-97) + inverse CDF on the device,
    against the reference's own temperature_scale and sample_with_uniform."""
    from oracle.oracle_lib import window_uniforms
    from paper_2511_11733_b200.dsdv import VerifyParams
    from tests.parity_util import host_rows
    B, G, V = 8, 4, 5000
    draft, _ = verifier.synth_logits(B, G, V, torch.float32, logits_seed=17)
    p = VerifyParams(gamma=G, seed=5, window=2)
    tok = verifier.draft_sample(draft, p, vocab=V, temperature=T).cpu().numpy()
    from oracle.oracle_lib import Oracle
    from tests.parity_util import EPS_CDF
    rows = host_rows(draft, V)
    U = window_uniforms(5, 2, B, G)
    port = Oracle()
    eps = 0
    for b in range(B):
        for j in range(G):
            _, pr = ref_oracle.softmax(rows[b, j])
            q = ref_oracle.temperature_scale(pr, T)
            ref = ref_oracle.sample_with_uniform(q, U[b, j])[1]
            if ref != tok[b, j]:
                _, margin = port.sample_with_margin(q, U[b, j])
                assert margin < EPS_CDF, (b, j, tok[b, j], ref, margin)
                eps += 1
    assert eps <= 2, eps


@pytest.mark.parametrize("dtype,V", [(torch.bfloat16, 128256), (torch.float32, 151936),
                                     (torch.bfloat16, 1003), (torch.float32, 7)])
def test_host_synth_is_bit_identical_to_device(verifier, oracle, dtype, V):
    """The CPU reference arm builds its window with oracle_synth_logits; it must
    be the device's dsdv_synth_logits window bit for bit (include/dsdv/synth.h)."""
    B, G = 8, 3
    d, t = verifier.synth_logits(B, G, V, dtype, logits_seed=42)
    hd, ht = oracle.synth_logits(B, G, V, dtype == torch.bfloat16, logits_seed=42,
                                 stride=d.shape[-1])
    if dtype == torch.bfloat16:
        gd = d.view(torch.int16).cpu().numpy().view(np.uint16)
        gt = t.view(torch.int16).cpu().numpy().view(np.uint16)
    else:
        gd = d.cpu().numpy().view(np.uint32)
        gt = t.cpu().numpy().view(np.uint32)
        hd, ht = hd.view(np.uint32), ht.view(np.uint32)
    assert np.array_equal(gd, hd), int((gd != hd).sum())
    assert np.array_equal(gt, ht), int((gt != ht).sum())
