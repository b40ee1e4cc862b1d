"""Distribution-level check of the whole device round:
the empirical distribution of the first committed token over many
independent sequences (one Philox stream each) against the reference's exact
enumeration of the draft-verify loop (enumerate_output_distribution /
expected_accepted_count, compiled into oracle/_ref). At tau = 0 this is the
losslessness of speculative sampling (acceptance criterion 1); at tau > 0 the
relaxed output distribution the reference defines."""
import math

import numpy as np
import pytest
import torch

from oracle.oracle_lib import Oracle
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams

pytestmark = pytest.mark.gpu

DRAFT = np.array([0.15, 0.2, 0.25, 0.2, 0.1, 0.1])     # support/generators.hpp:77-85
TARGET = np.array([0.45, 0.3, 0.1, 0.08, 0.04, 0.03])


def _rows(p, n_rows, B, stride):
    r = torch.full((B, n_rows, stride), float("-inf"), dtype=torch.float32, device="cuda")
    r[..., :p.size] = torch.tensor(np.log(p), dtype=torch.float32, device="cuda")
    return r


@pytest.mark.parametrize("gamma,tau", [(2, 0.0), (4, 0.0), (2, 0.3), (4, 0.6)])
def test_first_token_distribution_matches_exact_enumeration(verifier, ref_oracle, gamma, tau):
    B, V, stride = 1 << 17, DRAFT.size, 8
    crit = Oracle.crit(2.0, 0.2, 0.5, 6)
    exact, ek = ref_oracle.enumerate_first(DRAFT, TARGET, gamma, tau, crit)
    draft = _rows(DRAFT, gamma, B, stride)
    target = _rows(TARGET, gamma + 1, B, stride)
    p = VerifyParams(gamma=gamma, tau=tau, ratio_limit=2.0, gap_limit=0.2, overlap_floor=0.5,
                     top_m=6, seed=2024, window=7)
    tokens = verifier.draft_sample(draft, p, vocab=V)
    out = verifier.verify(draft, target, tokens, p, vocab=V)
    verifier.sync(p, out, batch=B, vocab=V)
    k = out.accepted_count.long()
    first = torch.where(k > 0, tokens[:, 0].long(), out.extra_token.long())
    emp = torch.bincount(first, minlength=V).double().cpu().numpy() / B
    tv = 0.5 * np.abs(emp - exact).sum()
    # sampling noise: E[TV] ~ sum sqrt(p(1-p)/(2 pi B)) ~ 3e-3 at B = 2^17
    assert tv < 0.012, (tv, emp, exact)
    mk = k.double().mean().item()
    sd = k.double().std().item()
    assert abs(mk - ek) < 5 * sd / math.sqrt(B) + 1e-9, (mk, ek)
    if tau == 0.0:
        assert np.abs(exact - TARGET).max() < 1e-12  # the enumeration itself is lossless
