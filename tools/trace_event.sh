# timeline of one eval_metric (setup + event kernels) from %globaltimer stamps
# written into a device buffer (PF_EVENT_TRACE build; pf_debug_trace reads it)
PFB200_DEFINES="PF_EVENT_TRACE" python - <<'PY'
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_1311_1753_b200 import parfit as pf
x, pdf = bench.build_model(pf)
xs = bench.make_events(10_000_000)
bm = pf.BoundModel(pdf, pf.UnbinnedDataSet.from_columns([x], xs))
p = [bench.START[v.name] for v in bm.registry().parameters()]
for i in range(5): bm.eval_metric(p)
buf = (C.c_uint64 * (4096 * 6))()
n = pf.lib.pf_debug_trace(bm._h, buf, 4096 * 6)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 6).astype(np.float64)
s0, s1 = t[4095, 0], t[4095, 1]
blk = t[:4094][t[:4094, 0] > 0]
rel = (blk - s0) / 1000.0
print("setup: %.2f us" % ((s1 - s0) / 1000))
print("last block: enters %.2f, published %.2f" % ((t[4094, 0] - s0) / 1000, (t[4094, 2] - s0) / 1000))
for name, col in zip(["in", "prologue", "pdl-wait", "loop", "done"], range(5)):
    v = rel[:, col]
    print("%-9s min %7.2f  median %7.2f  max %7.2f" % (name, v.min(), np.median(v), v.max()))
loop = rel[:, 3] - rel[:, 2]
print("main loop per block: min %.2f median %.2f max %.2f" % (loop.min(), np.median(loop), loop.max()))
nb = int((t[:4095, 0] > 0).sum()); nw = 2 * nb
ch = int(pf.lib.pf_model_chunk(bm._h)); nch = (10_000_000 + ch - 1) // ch
sm = t[:nb, 5].astype(int)
for b in range(nb):
    pass
cnt = np.array([sum(((nch - 1 - g) // nw + 1) if g < nch else 0 for g in (2 * b, 2 * b + 1)) for b in range(nb)])
for c in sorted(set(cnt)):
    v = loop[:nb][cnt == c]
    print("blocks with %d chunks: %4d  loop median %.2f max %.2f" % (c, len(v), np.median(v), v.max()))
per_sm = np.bincount(sm, minlength=148)
print("blocks per SM: min %d max %d" % (per_sm.min(), per_sm.max()))
end = rel[:nb, 3]
sm_end = np.array([end[sm == k].max() if (sm == k).any() else 0 for k in range(148)])
print("SM finish: min %.2f median %.2f max %.2f" % (sm_end.min(), np.median(sm_end), sm_end.max()))
slow = np.argsort(-loop[:nb])[:8]
print("slowest blocks:", [(int(b), int(sm[b]), round(float(loop[b]), 2), round(float(rel[b, 2]), 2)) for b in slow])
PY
