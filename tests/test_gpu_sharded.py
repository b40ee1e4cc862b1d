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


def test_sharded_equals_unsharded_gpu(verifier, oracle):
    crit = Oracle.crit(2.0, 0.2, 0.5, 10)
    rep, gpu, uns = _run(verifier, oracle, torch.bfloat16, 32, 8, 128256, 0.2, crit, 4)
    assert rep.ok(), rep.mismatches[:5]
    same = float((gpu["accepted_count"] == uns["accepted_count"]).float().mean())
    assert same >= 0.95
    assert bool((gpu["norm_match"] == uns["norm_match"]).all())
