"""Timeline of one fused eval_metric call (pf_fused_kernel) from %globaltimer
stamps (PFB200_DEFINES=PF_EVENT_TRACE build): per CTA entry, setup done, last
warp's loop done, block done; the last CTA's finalize.  Usage:
  PFB200_DEFINES=PF_EVENT_TRACE python tools/trace_fused.py [C2|C1|C3] [events]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1753_b200 import parfit as pf  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402

W = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else W.default_n
obs, pdf = W.build(pf)
bm = pf.BoundModel(pdf, W.data(pf, obs, n), pf.GridSpec(W.grid))
p = W.params(bm)
for i in range(5):
    bm.eval_metric(p)
buf = (C.c_uint64 * (4096 * 6))()
pf.lib.pf_debug_trace(bm._h, buf, 4096 * 6)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 6).astype(np.float64)
blk = t[:4094][t[:4094, 0] > 0]
t0 = blk[:, 0].min()
rel = (blk[:, :4] - t0) / 1000.0
for name, col in zip(["enter", "setup done", "loop done", "block done"], range(4)):
    v = rel[:, col]
    print("%-11s min %7.2f  median %7.2f  max %7.2f us" % (name, v.min(), np.median(v), v.max()))
print("finalize: starts %.2f, ends %.2f us" % ((t[4094, 0] - t0) / 1000, (t[4094, 2] - t0) / 1000))
if t[4095, 1] > 0:
    print("  finalize steps: digits summed %.2f, record built %.2f, published %.2f us"
          % tuple((t[4095, c] - t0) / 1000 for c in (1, 2, 3)))
print("CTAs traced:", len(blk))
wb = (C.c_uint64 * (4096 * 2))()
pf.lib.pf_debug_trace(bm._h, wb, -4096 * 2)
w = np.frombuffer(wb, dtype=np.uint64).reshape(4096, 2).astype(np.float64)
w = w[w[:, 1] > 0]
cnt = w[:, 0]
end = (w[:, 1] - t0) / 1000.0
print("warps %d: chunks per warp min %d median %d max %d; loop end min %.2f median %.2f p90 %.2f max %.2f us"
      % (len(w), cnt.min(), np.median(cnt), cnt.max(), end.min(), np.median(end), np.percentile(end, 90), end.max()))
for c in sorted(set(cnt.astype(int))):
    e = end[cnt == c]
    print("  warps with %d chunks: %4d  end median %.2f max %.2f" % (c, len(e), np.median(e), e.max()))
