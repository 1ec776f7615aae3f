"""Where the end-to-end time of one C2 call goes (host wall clock, L2 flushed
before each call as bench.py's e2e loop does): the public Python call, the raw
ctypes call of pf_eval_metric with prebuilt arguments, and the device step."""
import ctypes as C
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1311_1753_b200 import _abi, parfit as pf  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402

W = WORKLOADS["C2"]
obs, pdf = W.build(pf)
ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(10_000_000, seed=11))
bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
p = W.params(bm)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
for _ in range(10):
    bm.eval_metric(p)


def timed(fn, n=200, do_flush=True):
    ts = []
    for k in range(n):
        if do_flush:
            flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts) * 1e6, statistics.mean(ts) * 1e6


out, info, st = C.c_double(), _abi.pf_eval_info(), _abi.pf_status()
fn = pf._eval_fast_bound()
args = (bm._h, p.ctypes.data, p.size, 0, C.byref(out), C.byref(info), C.byref(st))
print("python eval_metric   median/mean us: %.1f / %.1f" % timed(lambda: bm.eval_metric(p)))
print("raw ctypes call      median/mean us: %.1f / %.1f" % timed(lambda: fn(*args)))
print("python, no flush     median/mean us: %.1f / %.1f" % timed(lambda: bm.eval_metric(p), do_flush=False))
r = _abi.pf_bench_result()
pf.lib.pf_bench(bm._h, p.ctypes.data_as(C.POINTER(C.c_double)), p.size, 0, 50, 1, C.byref(r), C.byref(st))
print("device step (pf_bench) us: %.1f" % (r.step_ms_mean * 1e3))
