"""C5 pipeline emulation: the closed forms and the reference's DES semantics
(latency.cpp:63-86, netsim.cpp:110-202) on CPU, replayed against the
reference's known answers (test_latency.cpp, acceptance criterion 3); the
device emulation on GPU."""
import pytest

from paper_2511_11733_b200 import pipeline as pl


def test_closed_forms_known_answers():
    # test_latency.cpp:31-41 with kReference = {N=4, t0=1, t1=5}
    assert pl.standard_decode_time(1.0, 1, 1.0, 5.0) == 1.0
    assert abs(pl.standard_decode_time(4.0, 4, 1.0, 5.0) - 64.0) < 1e-12
    assert pl.standard_decode_time(7.0, 12, 2.0, 0.0) == 14.0
    assert pl.dsd_round_time(1.0, 4, 1.0, 5.0) == pl.standard_decode_time(1.0, 4, 1.0, 5.0)
    assert abs(pl.dsd_round_time(4.0, 4, 1.0, 5.0) - 19.0) < 1e-12
    assert pl.dsd_round_time(5.0, 1, 2.0, 0.0) == 10.0


def test_reduction_ratio_identity_and_monotonicity():
    # acceptance.cpp:126-145: R = 1 - T_dsd / T_std, increasing in k and in t1
    for n in (2, 4, 8):
        for t1 in (0.5, 1.0, 5.0):
            for k in range(1, 9):
                r = pl.comm_reduction_ratio(k, n, 1.0, t1)
                ident = 1 - pl.dsd_round_time(k, n, 1.0, t1) / pl.standard_decode_time(k, n, 1.0, t1)
                assert abs(r - ident) <= 1e-12
                if k < 8:
                    assert pl.comm_reduction_ratio(k + 1, n, 1.0, t1) > r
        assert pl.comm_reduction_ratio(4, n, 1.0, 1.0) < pl.comm_reduction_ratio(4, n, 1.0, 5.0)


def test_des_matches_closed_forms():
    # acceptance.cpp:96-113: the simulator equals the closed forms
    for n in (1, 2, 8):
        t0, t1 = 1.0, 3.0
        assert abs(pl.des_total(pl.standard_units(12, t0), n, t1)
                   - pl.standard_decode_time(12, n, t0, t1)) <= 1e-9
        for k in (1, 3, 7):
            # simulate_dsd charges k t0 of compute per window (netsim.cpp:195-200)
            got = pl.des_total(pl.dsd_units([k] * 4, t0), n, t1)
            assert abs(got - 4 * (k * t0 + (n - 1) * t1)) <= 1e-9


@pytest.mark.gpu
def test_device_emulation_tracks_the_model():
    import torch
    from paper_2511_11733_b200.dsdv import Verifier
    v = Verifier(0)
    emu = pl.PipelineEmulator(v, 8)
    t0, t1 = 20_000, 100_000  # ns
    ks = [3, 0, 8, 2, 5, 1, 4, 2]
    tokens = sum(k + 1 for k in ks)
    t_std = emu.run(pl.standard_units(tokens, t0), t1)
    t_dsd = emu.run(pl.dsd_units(ks, t0), t1)
    des_std = pl.des_total(pl.standard_units(tokens, t0), 8, t1) / 1e6
    des_dsd = pl.des_total(pl.dsd_units(ks, t0), 8, t1) / 1e6
    # device spins track the model within launch overheads (a few us per hop)
    assert abs(t_std - des_std) / des_std < 0.1
    assert abs(t_dsd - des_dsd) / des_dsd < 0.1
    assert abs((1 - t_dsd / t_std) - (1 - des_dsd / des_std)) < 0.03


def test_expected_speedup_known_answers():
    # latency.cpp:88-95 at kReference {N=4, t0=1, t1=5}: rho=1, k=1 -> 1 (no gain);
    # amortisation grows with the accepted span
    assert abs(pl.expected_speedup(1.0, 1.0, 4, 1.0, 5.0) - 1.0) < 1e-12
    assert pl.expected_speedup(0.5, 4.0, 4, 1.0, 5.0) > pl.expected_speedup(0.5, 2.0, 4, 1.0, 5.0)
    assert pl.analytic_speedup(0.0, 2.0, 4, 1.0, 5.0) == 0.0
