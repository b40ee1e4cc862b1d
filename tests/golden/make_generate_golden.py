"""Golden per-round accepted counts of the reference's generate() on the
default divergent pair (support/generators.hpp:77-85), produced by the
reference sources compiled here (oracle/_ref/libdsdref.so, oracle/Makefile).

    python tests/golden/make_generate_golden.py   # writes generate_divergent.json

The GPU drop-in API must reproduce them round for round
(tests/test_cpp_api.py). Needs /root/reference (this container only)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle_lib import Oracle, RefOracle  # noqa: E402

DRAFT = [0.15, 0.2, 0.25, 0.2, 0.1, 0.1]
TARGET = [0.45, 0.3, 0.1, 0.08, 0.04, 0.03]
CASES = [  # gamma, tau, seed, max_new, (ratio, gap, overlap, top_m)
    (8, 0.0, 1, 256, (2.0, 0.2, 0.5, 6)),
    (8, 0.2, 2, 256, (2.0, 0.2, 0.5, 6)),
    (8, 0.4, 3, 256, (2.0, 0.2, 0.5, 6)),
    (8, 0.8, 4, 256, (2.0, 0.2, 0.5, 6)),
    (4, 0.3, 7, 128, (1.5, 0.1, 0.7, 3)),
    (2, 1.0, 9, 64, (float("inf"), 1.0, 0.0, 1)),
    (16, 0.5, 11, 256, (3.0, 0.3, 0.4, 6)),
]


def main():
    ref = RefOracle()
    out = []
    for g, tau, seed, max_new, c in CASES:
        ks = ref.generate_iid(DRAFT, TARGET, g, tau, Oracle.crit(*c), max_new, seed)
        out.append({"gamma": g, "tau": tau, "seed": seed, "max_new": max_new,
                    "criteria": [c[0] if c[0] != float("inf") else "inf", *c[1:]], "ks": ks})
    (Path(__file__).parent / "generate_divergent.json").write_text(json.dumps(out))
    print(f"{len(out)} cases")


if __name__ == "__main__":
    main()
