"""Time dsdv_verify for several builds of the same ABI on one box (development
aid): python scripts/variant_time.py name1 name2 ... -- each name is
libdsdv_<name>.so next to libdsdv.so ("base" = libdsdv.so), run in its own
process through DSDV_LIB, interleaved over `--rounds` rounds."""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
ap = argparse.ArgumentParser()
ap.add_argument("names", nargs="+")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--args", default="")
a = ap.parse_args()
res = {n: [] for n in a.names}
for r in range(a.rounds):
    for n in a.names:
        lib = ROOT / "paper_2511_11733_b200" / ("libdsdv.so" if n == "base" else f"libdsdv_{n}.so")
        env = {**os.environ, "DSDV_LIB": str(lib)}
        out = subprocess.run([sys.executable, str(ROOT / "scripts" / "quick_time.py"),
                              *a.args.split()], capture_output=True, text=True, env=env)
        try:
            j = json.loads(out.stdout.strip().splitlines()[-1])
            res[n].append(j["ms_median"])
        except Exception:
            res[n].append(None)
            print(n, out.stdout[-500:], out.stderr[-1500:], flush=True)
for n, v in res.items():
    ok = [x for x in v if x]
    print(json.dumps({"variant": n, "ms": v, "best": min(ok) if ok else None}), flush=True)
