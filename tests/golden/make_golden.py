#!/usr/bin/env python3
"""Regenerates tests/golden/golden.json from the REFERENCE itself.

Each case of cases.py is evaluated by the unmodified reference headers
compiled into oracle/_ref/libparfit_ref.so (BoundModel::eval_metric,
cached norms, log-floor / clamp counters, parfit::fit).  Values are stored
as float.hex strings (bit exact).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import oracle  # noqa: E402
from paper_1311_1753_b200 import parfit as pf  # noqa: E402
from cases import CASES, FIT_CASES  # noqa: E402


def main():
    oracle.build()
    if not oracle.Reference.available():
        raise SystemExit("oracle/_ref not built: /root/reference is required to regenerate")
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj/include/parfit",
           "cases": {}}
    for name, make in CASES.items():
        pdf, ds, grid, points = make(pf)
        binned = isinstance(ds, pf.BinnedDataSet)
        metric = 1 if binned else 0
        ref = oracle.Reference(pdf, ds, grid)
        rec = {"grid": grid, "metric": metric, "param_names": ref.param_names(), "points": []}
        for p in points:
            v = ref.eval(p, metric)
            norms, errs, valid = ref.norms()
            rec["points"].append({
                "params": [float(x).hex() for x in p], "value": float(v).hex(),
                "norms": [float(x).hex() for x in norms], "norm_errs": [float(x).hex() for x in errs],
                "norm_valid": valid, "floor_count": ref.floor_count(),
                "clamp": [ref.clamp_count(i) for i in range(len(norms))]})
            print(f"{name:22s} {p} -> {v!r}")
        if name in FIT_CASES:
            pdf, ds, grid, points = make(pf)  # fresh Variables at their initial values
            r = oracle.Reference(pdf, ds, grid).fit(metric)
            rec["fit"] = {"params": [float(x).hex() for x in r["params"]],
                          "uncertainties": [float(x).hex() for x in r["uncertainties"]],
                          "metric_value": float(r["metric_value"]).hex(), "calls": r["calls"],
                          "status": r["status"], "uncertainties_available": r["uncertainties_available"],
                          "grad_max_norm": float(r["grad_max_norm"]).hex()}
            print(f"{name:22s} fit {list(r['params'])} +- {list(r['uncertainties'])} calls {r['calls']}")
        out["cases"][name] = rec
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
