"""C-ABI boundary tests that need no GPU: every symbol include/dsdv/dsdv.h
declares is exported by libdsdv.so, the ctypes layouts match the header, and
host-side validation reproduces the reference's messages (verifier.cpp:55-91)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2511_11733_b200 import dsdv

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dsdv" / "dsdv.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:dsdv_status|double|int|uint64_t|const char \*)\s*(dsdv_\w+)\(",
                                 text, re.M)))


def test_header_declares_the_documented_entry_points():
    names = declared_functions()
    for n in ("dsdv_create", "dsdv_destroy", "dsdv_verify", "dsdv_window_stats",
              "dsdv_sample_extra", "dsdv_draft_sample", "dsdv_sync", "dsdv_validate",
              "dsdv_uniform", "dsdv_last_error", "dsdv_abi_version", "dsdv_synth_logits",
              "dsdv_launch_count"):
        assert n in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(dsdv.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dsdv_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_struct_layouts_match_header_sizes():
    # dsdv_params: 6 int32, 4 double, 2 uint64, uint32, 2 int32, 2 double
    assert C.sizeof(dsdv._Params) == 6 * 4 + 4 * 8 + 2 * 8 + 4 + 2 * 4 + 4 + 2 * 8
    assert C.sizeof(dsdv._Outputs) == 17 * 8
    assert dsdv.LIB.dsdv_abi_version() == 1


@pytest.mark.parametrize("kw,msg", [
    (dict(gamma=0), "gamma must be >= 1, got 0"),
    (dict(tau=1.5), "tau must lie in [0, 1], got 1.500000"),
    (dict(tau=float("nan")), "tau must lie in [0, 1], got nan"),
    (dict(ratio_limit=0.0), "criteria.ratio_limit must be > 0, got 0.000000"),
    (dict(gap_limit=1.5), "criteria.gap_limit must lie in [0, 1], got 1.500000"),
    (dict(overlap_floor=-0.1), "criteria.overlap_floor must lie in [0, 1], got -0.100000"),
    (dict(top_m=0), "criteria.top_m must be >= 1, got 0"),
])
def test_validation_messages_match_reference(kw, msg):
    with pytest.raises(dsdv.DsdvError) as e:
        dsdv.validate(dsdv.VerifyParams(**kw))
    assert e.value.status == dsdv.E_INVARIANT
    assert msg in str(e.value)


def test_infinite_ratio_limit_is_valid():
    dsdv.validate(dsdv.VerifyParams(ratio_limit=float("inf")))


def test_layout_rules():
    with pytest.raises(dsdv.DsdvError) as e:
        dsdv.validate(dsdv.VerifyParams(), vocab=10, row_stride=10, dtype=dsdv.DTYPE_F32)
    assert e.value.status == dsdv.E_UNSUPPORTED
    dsdv.validate(dsdv.VerifyParams(), vocab=10, row_stride=12, dtype=dsdv.DTYPE_F32)
    with pytest.raises(dsdv.DsdvError):
        dsdv.validate(dsdv.VerifyParams(), vocab=1, row_stride=16)
    with pytest.raises(dsdv.DsdvError) as e:
        dsdv.validate(dsdv.VerifyParams(top_m=33), vocab=64, row_stride=64)
    assert e.value.status == dsdv.E_UNSUPPORTED


def test_top_m_clamps_to_vocab():
    # KeyCriteria::top_m is clamped to V at use (verifier.cpp:155)
    dsdv.validate(dsdv.VerifyParams(top_m=100), vocab=8, row_stride=8)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(dsdv.DsdvError):
        dsdv.Verifier(0)
