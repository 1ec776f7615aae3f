"""Writes tests/golden/generate.json: for every case of gen_cases.py, the
reference's own generate_events (oracle/_ref: the unmodified reference
headers) — the sha256 of its column-major float64 output, its first and last
events and the observables' final values.  Run here, where /root/reference
exists:  python tests/golden/make_generate_golden.py"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import oracle  # noqa: E402
from gen_cases import CASES  # noqa: E402
from paper_1311_1753_b200 import parfit as pf  # noqa: E402


def main():
    out = {}
    for name, case in sorted(CASES.items()):
        pdf, obs, n, seed, grid = case(pf)
        cols = oracle.ref_generate(pdf, obs, n, seed, grid)
        out[name] = {
            "n": n, "seed": seed, "grid": grid,
            "sha256": hashlib.sha256(cols.tobytes()).hexdigest(),
            "first": [repr(float(v)) for v in cols[:, 0]],
            "last": [repr(float(v)) for v in cols[:, -1]],
        }
        print(name, out[name]["sha256"][:16])
    with open(os.path.join(HERE, "generate.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
