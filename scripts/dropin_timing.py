"""Per-round time of the C++ drop-in's generate() (libdsd_b200.so over the
device) against the reference's own generate() (oracle/_ref, the reference
sources compiled) on the same categorical rows, at SURVEY §3.1's shapes:
C1 (V=32000, gamma=4) and V=128256, gamma=8 (22.7 / 242.5 ms per round there).
    python scripts/dropin_timing.py > profiles/r2_dropin_timing.json"""
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle.oracle_lib import Oracle, RefOracle  # noqa: E402
from tests.test_cpp_api import EXE, rows_pair, write_rows_case  # noqa: E402

ref = RefOracle()
out = []
for V, gamma, max_new in ((32000, 4, 40), (128256, 8, 40)):
    pd, pt = rows_pair(V, 3)
    crit = (2.0, 0.2, 0.5, 10)
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "rows.bin"
        write_rows_case(f, pd, pt, gamma, 0.2, crit, 5, max_new, 0)
        subprocess.run([str(EXE), "rows", str(f)], capture_output=True, text=True)  # warm-up
        r = subprocess.run([str(EXE), "rows", str(f)], capture_output=True, text=True, check=True)
    lines = r.stdout.split("\n")
    ks = [int(x) for x in lines[2].split()]
    ms_dropin = float(lines[3])
    t0 = time.perf_counter()
    ref_ks = ref.generate_iid(pd, pt, gamma, 0.2, Oracle.crit(*crit), max_new, 5)
    ms_ref = (time.perf_counter() - t0) * 1e3 / len(ref_ks)
    out.append({"vocab": V, "gamma": gamma, "rounds": len(ks), "same_rounds": ks == ref_ks,
                "dropin_ms_per_round": ms_dropin, "reference_ms_per_round": ms_ref,
                "speedup": ms_ref / ms_dropin,
                "note": "drop-in: host draft_window + device window stats (fp64) + host walk + "
                        "device extra draw per round; reference: verify_round on one host core"})
print(json.dumps(out, indent=1))
