"""Where do the GPU fit and the reference fit part ways?  Runs the GPU fit of a
workload's bounded sample with PFB200_FIT_TRACE (every evaluated point and its
metric), then evaluates the reference at the same points: how many of the
GPU's metric values are bit-equal to the reference's, the first that is not,
and the reference fit's own call count.  Test infrastructure (uses oracle/).
  python tools/fit_trace.py C1"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1311_1753_b200 import parfit as pf  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402
import oracle  # noqa: E402

W = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
path = os.path.join(tempfile.mkdtemp(), "trace.txt")
os.environ["PFB200_FIT_TRACE"] = path
obs, pdf = W.build(pf)
ds = W.data(pf, obs, W.fit_n)
bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
names = [p.name for p in bm.registry().parameters()]
for p in bm.registry().parameters():
    p.value = W.start[p.name]
ref = oracle.Reference(pdf, ds, W.grid)  # evaluates the traced points
ref_fit = oracle.Reference(pdf, ds, W.grid)  # built at the start point: its fit starts there
r = pf.fit(bm, pf.MetricKind(W.metric))
rows = np.loadtxt(path, ndmin=2)
print("GPU fit: %d calls, status %d, params %s" % (r.n_metric_calls, int(r.status), dict(zip(r.names, r.params))))
equal, first, worst = 0, None, 0.0
for i, row in enumerate(rows):
    v = ref.eval(row[1:], W.metric, 1)
    if v == row[0]:
        equal += 1
    else:
        rel = abs(v - row[0]) / abs(v)
        worst = max(worst, rel)
        if first is None:
            first = (i, row[0], v, rel)
print("traced points %d: bit-equal to the reference %d; max rel diff %.2e" % (len(rows), equal, worst))
if first:
    print("first difference at call %d: gpu %.17g ref %.17g (rel %.2e)" % first)
rr = ref_fit.fit(W.metric, os.cpu_count() or 1)
print("reference fit: %d calls, status %d, params %s" % (rr["calls"], rr["status"], rr["params"]))
print("params order in the trace:", names)
