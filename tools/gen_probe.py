"""GPU generate_events timing vs the reference generator (oracle/_ref) on the
same request: C2's mixture at truth, seed 11.  Prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402

from gen_cases import CASES  # noqa: E402
from paper_1311_1753_b200 import parfit as pf  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    n_ref = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    pdf, obs, _, _, grid = CASES["mixture"](pf)
    pf.generate_events(pdf, obs, 1000, 1)  # compile + warm
    t = time.perf_counter()
    ds = pf.generate_events(pdf, obs, n, 11)
    wall = time.perf_counter() - t
    out = {"n": n, "gpu_device_ms": ds.generation_ms, "gpu_wall_s": wall,
           "gpu_events_per_s": n / wall}
    try:
        import oracle
        if oracle.Reference.available():
            t = time.perf_counter()
            ref = oracle.ref_generate(pdf, obs, n_ref, 11, grid)
            rw = time.perf_counter() - t
            out.update(ref_n=n_ref, ref_wall_s=rw, ref_events_per_s=n_ref / rw,
                       prefix_identical=bool(np.array_equal(ds.columns()[:, :n_ref], ref)))
    except Exception as e:  # noqa: BLE001
        out["ref_error"] = str(e)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
