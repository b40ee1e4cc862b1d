"""bench.py's JSON line contract, on CPU: the reference arm (`--impl reference`)
times the reference's own verifier (oracle/_ref, the reference sources compiled,
or the oracle port) on the host and prints the driver's line."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    baseline = json.loads((ROOT / "BASELINE.json").read_text())
    assert line["impl"] == "reference"
    assert line["metric"] == baseline["metric"]
    assert line["unit"] == "verified draft tokens/s"
    assert line["n_gpus"] == 1 and line["steps"] == 1 and line["warmup"] == 3
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["higher_is_better"] is True and line["scaling"] == "weak"
    assert line["vs_baseline"] is None
    assert line["config"]["workload"].startswith("C2")
    assert line["config"]["vocab"] == 128256 and line["config"]["gamma"] == 8
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    assert cb["value"] == line["value"] and cb["sample"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
