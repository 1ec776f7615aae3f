"""Timeline of a pf_norm_kernel launch (PFB200_DEFINES="PF_NORM_POINT_TRACE;PF_EVENT_TRACE"):
per block entry, points start/end, arrival; the last block's end.
  python tools/trace_norm.py C4"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1753_b200 import parfit as pf  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402

W = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else W.default_n
obs, pdf = W.build(pf)
data = W.data(pf, obs, n)
bm = pf.BoundModel(pdf, data, pf.GridSpec(W.grid))
p = W.params(bm)
for i in range(3):
    bm.eval_metric(p, pf.MetricKind(W.metric))
buf = (C.c_uint64 * (4096 * 6))()
pf.lib.pf_debug_trace(bm._h, buf, 4096 * 6)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 6).astype(np.float64)[2000:4000]
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
rel = (t[:, :5] - t0) / 1000.0
for name, col in zip(["entry", "points start", "points end", "arrive"], range(4)):
    v = rel[:, col]
    print("%-13s min %7.2f  median %7.2f  max %7.2f us" % (name, v.min(), np.median(v), v.max()))
last = rel[t[:, 4] > 0]
print("last block done: %.2f us; blocks %d" % (last[:, 4].max() if len(last) else -1, len(t)))
