"""Trace / summary CSV in the reference schema (test_metrics.cpp:52-170 replayed)."""
import pytest

from paper_2511_11733_b200 import metrics as m


def test_stats_over_a_hand_computed_round_log():
    st = m.compute_stats([2, 4, 3], [0, 0, 0], 8)
    assert abs(st.rho - 1 / 3) <= 1e-12 and abs(st.avg_accepted_len - 4.0) <= 1e-12
    assert st.total_tokens == 12 and st.sync_rounds == 3 and st.tokens_per_ms is None


def test_key_fraction_counts_evaluated_positions_only():
    # 2 accepted (1 key) + 1 rejected non-key: 3 evaluated decisions
    assert abs(m.compute_stats([2], [1], 4).key_token_fraction - 1 / 3) <= 1e-12


def test_tokens_per_ms_only_with_timing():
    assert abs(m.compute_stats([3], [0], 3, total_ms=50.0).tokens_per_ms - 4 / 50) <= 1e-12


def test_six_significant_digits():
    assert m.format_double(0.703125) == "0.703125"
    assert m.format_double(64.0) == "64"
    assert m.format_double(16.0 / 5.75) == "2.78261"
    assert m.format_double(0.2) == "0.2"
    assert m.format_double(1.0 / 3.0) == "0.333333"


def test_trace_csv_exact_schema_and_order():
    assert m.render_trace_csv([]) == m.TRACE_HEADER + "\n"
    row = m.TraceRow("seed1", 0, 8, 0.2, 4, 1.0, 5.0, 4, 1, 4.0, 15.0, 19.0, 1)
    assert m.render_trace_csv([row]) == m.TRACE_HEADER + "\nseed1,0,8,0.2,4,1,5,4,1,4,15,19,1\n"
    a = m.TraceRow(**{**row.__dict__, "run_id": "seed2"})
    b = m.TraceRow(**{**row.__dict__, "round_index": 1})
    multi = m.render_trace_csv([b, a, row])
    assert multi.find("seed1,0") < multi.find("seed2,0") < multi.find("seed1,1")


def test_summary_csv_exact_schema():
    row = m.SummaryRow("seed1", 1 / 3, 4.0, 12, 3, 0.08, 0.25, 2.78260869565, 64 / 19)
    assert m.render_summary_csv([row]) == (
        m.SUMMARY_HEADER + "\nseed1,0.333333,4,12,3,0.08,0.25,2.78261,3.36842\n")


def test_stats_validation():
    with pytest.raises(ValueError):
        m.compute_stats([], [], 8)
    with pytest.raises(ValueError):
        m.compute_stats([1], [0], 0)
