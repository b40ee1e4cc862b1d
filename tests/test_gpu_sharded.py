"""Vocabulary-sharded verification against the oracle.

All P ranks of a window run in one process on one device (sharded.shard_slices:
the same device steps as a multi-GPU run, collectives by stacking). Decisions
must equal the unsharded fp64 oracle's except inside the eps bands; the fp32
sums are re-associated across slices, so the bands are where differences may
appear (counted)."""
import pytest
import torch

from oracle.oracle_lib import Oracle
from paper_2511_11733_b200.sharded import shard_slices, slice_bounds
from tests.parity_util import compare_window, run_gpu_window

pytestmark = pytest.mark.gpu


def _run(verifier, oracle, dtype, B, G, V, tau, crit, P, seed=1):
    d64, t64, toks, unsharded, (draft, target, tokens, p) = run_gpu_window(
        verifier, dtype, B, G, V, tau, crit, seed=seed, oracle=oracle)
    out = shard_slices(verifier, draft, target, tokens, p, V, P)
    torch.cuda.synchronize()
    gpu = out.to_host()
    rep = compare_window(oracle, d64, t64, toks, gpu, tau, crit, seed, 0)
    return rep, gpu, unsharded


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_sharded_bf16_matches_oracle(verifier, oracle, P):
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    rep, gpu, uns = _run(verifier, oracle, torch.bfloat16, 16, 4, 32000, 0.2, crit, P)
    assert rep.ok(), rep.mismatches[:5]
    assert rep.eps_events <= 2


@pytest.mark.parametrize("tau", [0.0, 0.5, 1.0])
def test_sharded_f32_tau_sweep(verifier, oracle, tau):
    crit = Oracle.crit(2.0, 0.2, 0.5, 6)
    rep, gpu, uns = _run(verifier, oracle, torch.float32, 8, 4, 5000, tau, crit, 3)
    assert rep.ok(), rep.mismatches[:5]


@pytest.mark.parametrize("dtype,G,P,top_m", [(torch.float32, 16, 12, 12),
                                             (torch.bfloat16, 16, 5, 32),
                                             (torch.bfloat16, 15, 8, 32),
                                             (torch.float32, 31, 3, 4)])
def test_sharded_merge_shapes(verifier, oracle, dtype, G, P, top_m):
    """The decide step's other shapes: gamma + 1 > 16 (one lane per position),
    more than 8 slices (list heads in local memory), top_m up to 32 with lists
    too large to stage in shared memory."""
    crit = Oracle.crit(2.0, 0.2, 0.5, top_m)
    V = 6000
    rep, gpu, uns = _run(verifier, oracle, dtype, 6, G, V, 0.3, crit, P, seed=5)
    assert rep.ok(), rep.mismatches[:5]
    assert rep.eps_events <= 2


@pytest.mark.parametrize("dtype,P", [(torch.bfloat16, 1), (torch.float32, 2)])
def test_sharded_long_slices(verifier, oracle, dtype, P):
    """Long slices (P=1: whole rows in partial mode) and fp32 halves."""
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    rep, gpu, uns = _run(verifier, oracle, dtype, 4, 4, 140000, 0.2, crit, P, seed=9)
    assert rep.ok(), rep.mismatches[:5]
    assert rep.eps_events <= 2


def test_sharded_equals_unsharded_gpu(verifier, oracle):
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    B, G, V = 160, 8, 128256  # 1,440 items: well above one per CTA
    d64, t64, toks, uns, (draft, target, tokens, p) = run_gpu_window(
        verifier, torch.bfloat16, B, G, V, 0.2, crit, seed=1, oracle=oracle)
    gpu = shard_slices(verifier, draft, target, tokens, p, V, 4).to_host()
    from oracle.oracle_lib import window_uniforms
    from tests.parity_util import compare_batch, host_logits
    ref = oracle.verify_batch(host_logits(draft), host_logits(target), toks, [(0.2, crit)],
                              window_uniforms(1, 0, B, G), V, all_positions=True)[0]
    rep_s = compare_batch(ref, gpu)
    rep_u = compare_batch(ref, uns)
    assert rep_s.ok(), rep_s.mismatches[:5]
    assert rep_u.ok(), rep_u.mismatches[:5]
    # sharded and unsharded windows agree on k wherever neither hit an eps event
    differ = int((gpu["accepted_count"] != uns["accepted_count"]).sum())
    assert differ <= rep_s.eps_events + rep_u.eps_events, (differ, rep_s.eps_events,
                                                           rep_u.eps_events)
    assert bool((gpu["norm_match"] == uns["norm_match"]).all())


@pytest.mark.parametrize("P", [2, 4, 8])
def test_peer_exchange_equals_gathered(verifier, oracle, P):
    """The fused exchange (stats kernel storing into every rank's buffer,
    flags, merge from the local buffer) gives the gathered path's window bit
    for bit, and stays parity-green against the oracle."""
    from paper_2511_11733_b200.sharded import shard_slices_peer
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    d64, t64, toks, unsharded, (draft, target, tokens, p) = run_gpu_window(
        verifier, torch.bfloat16, 16, 4, 32000, 0.2, crit, seed=3, oracle=oracle)
    ref = shard_slices(verifier, draft, target, tokens, p, 32000, P).to_host()
    for epoch in (1, 2, 3):  # both buffer sets, advancing flags
        got = shard_slices_peer(verifier, draft, target, tokens, p, 32000, P, epoch=epoch)
        got = got.to_host()
        assert set(got) == set(ref)
        for k in ref:
            a, b = torch.as_tensor(got[k]), torch.as_tensor(ref[k])
            assert torch.equal(a, b) or (a.is_floating_point() and
                                         torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0))), k
    rep = compare_window(oracle, d64, t64, toks, got, 0.2, crit, 3, 0)
    assert rep.ok(), rep.mismatches[:5]


def test_peer_exchange_across_processes():
    """The real thing when the box has two GPUs: torchrun, CUDA IPC mappings,
    NVLink peer stores and flag rounds, compared with the NCCL path on every
    rank over several windows (scripts/peer_check.py)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           str(root / "scripts" / "peer_check.py")]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert "OK (0 differing fields" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("dtype,P,tau", [(torch.float32, 3, 0.5), (torch.bfloat16, 4, 1.0),
                                         (torch.float32, 2, 0.0)])
def test_peer_exchange_dtypes(verifier, oracle, dtype, P, tau):
    """The collective-free window for fp32 slices, odd P and the τ endpoints,
    bit-equal to the gathered window and parity-green against the oracle."""
    from paper_2511_11733_b200.sharded import shard_slices_peer
    crit = Oracle.crit(2.0, 0.2, 0.5, 6)
    V = 5000
    d64, t64, toks, unsharded, (draft, target, tokens, p) = run_gpu_window(
        verifier, dtype, 8, 4, V, tau, crit, seed=11, oracle=oracle)
    ref = shard_slices(verifier, draft, target, tokens, p, V, P).to_host()
    got = shard_slices_peer(verifier, draft, target, tokens, p, V, P, epoch=2).to_host()
    for k in ref:
        a, b = torch.as_tensor(got[k]), torch.as_tensor(ref[k])
        assert torch.equal(a, b) or (a.is_floating_point() and
                                     torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0))), k
    rep = compare_window(oracle, d64, t64, toks, got, tau, crit, 11, 0)
    assert rep.ok(), rep.mismatches[:5]


def test_pipeline_emulation_across_processes():
    """C5 on the box's GPUs (stage s on GPU s mod P): the C++-enqueued hop loop
    (dsdv_pipeline_run, NVLink peer stores + counters) tracks the reference's
    DES (netsim.cpp:110-172) and the closed form (latency.cpp:81-86)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs 2 GPUs")
    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", "29563",
           str(root / "scripts" / "pipeline_emulation.py"), "--rounds", "32", "--t0-us", "20"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 4
    for d in lines:
        assert d["gpus"] == n
        assert abs(d["measured"]["R_comm"] - d["des"]["R_comm"]) < 0.03, d
        assert d["measured"]["sync_rounds_dsd"] < d["measured"]["sync_rounds_standard"]


def test_one_call_window_times_out_into_statuses(verifier):
    """dsdv_shard_verify_peers with a peer that never signals: every flag round
    gives up after timeout_ns and the window's statuses all read DSDV_E_NCCL
    (never a stale window reported as a success)."""
    import ctypes as C

    from paper_2511_11733_b200 import dsdv
    from paper_2511_11733_b200.dsdv import VerifyParams, WindowResult
    from paper_2511_11733_b200.sharded import (PeerExchange, ShardedVerifier,
                                               contiguous_slice, slice_bounds)
    B, G, V, P = 8, 4, 5000, 2
    draft, target = verifier.synth_logits(B, G, V, torch.bfloat16, logits_seed=5)
    p = VerifyParams(gamma=G, tau=0.2, seed=1)
    tokens = verifier.draft_sample(draft, p, vocab=V)
    lo, n = slice_bounds(V, P, 0)
    d, t = contiguous_slice(draft, lo, n), contiguous_slice(target, lo, n)
    sv = ShardedVerifier(verifier)
    _, size = sv.exchange_layout(B, G, p.top_m)
    ex = PeerExchange(verifier, P, 0, size, bases=PeerExchange.allocate_local(verifier, P, size))
    out = WindowResult.allocate(B, G, draft.device, True, records=True)
    cp = sv._cp(p, d, t, tokens, V, lo, n)
    bases = (C.c_void_p * P)(*ex.bases)
    cs = torch.cuda.current_stream()
    st = dsdv.LIB.dsdv_shard_verify_peers(verifier._h, C.byref(cp), d.data_ptr(), t.data_ptr(),
                                          tokens.data_ptr(), P, 0, bases, ex.stride, 1,
                                          int(20e6), C.byref(out._c), cs.cuda_stream)
    assert st == dsdv.OK
    torch.cuda.synchronize()
    assert bool((out.status.cpu() == dsdv.E_NCCL).all())
