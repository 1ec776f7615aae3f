"""Small calls for compute-sanitizer (memcheck / racecheck / synccheck):
C2 single (fused kernel), C2 batched K = 8 (setup + event kernels), C4
binned convolution (pre + norm levels + event), C5 TDDP (component grid
tasks), the exchange group of one (peer-memory record path), each checked
against the oracle so a sanitizer-induced change would show.
  compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1311_1753_b200 import parfit as pf  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


W = WORKLOADS["C2"]
obs, pdf = W.build(pf)
ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(200_003, seed=3))
bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
p = W.params(bm)
v = bm.eval_metric(p)
o = oracle.Oracle(pdf, ds, W.grid)
print("C2 fused", v, rel(v, o.eval(list(p))))
pts = np.array([p * (1 + 1e-3 * k) for k in range(8)])
b = bm.eval_metric_batch(pts)
print("C2 batched K=8", list(b[:2]), rel(b[3], o.eval(list(pts[3]))))
W4 = WORKLOADS["C4"]
o4, pdf4 = W4.build(pf)
d4 = W4.data(pf, o4, 2000, seed=3)
bm4 = pf.BoundModel(pdf4, d4, pf.GridSpec(W4.grid))
q = W4.params(bm4)
v4 = bm4.eval_metric(q, pf.MetricKind.ChiSquared)
print("C4", v4, rel(v4, oracle.Oracle(pdf4, d4, W4.grid).eval(list(q), 1)))
W5 = WORKLOADS["C5"]
o5, pdf5 = W5.build(pf)
d5 = pf.UnbinnedDataSet.from_columns(o5, W5.columns(5000, seed=3))
bm5 = pf.BoundModel(pdf5, d5, pf.GridSpec(32))
r5 = [W5.truth[v.name] for v in bm5.registry().parameters()]
v5 = bm5.eval_metric(r5)
print("C5 tddp", v5, rel(v5, oracle.Oracle(pdf5, d5, 32).eval(r5)))
g = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
g.group_join(1, 0, [g.group_handle()])
vg = g.eval_metric(p)
print("group of one", vg, vg == v)
