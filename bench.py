#!/usr/bin/env python3
"""bench.py — NLL evaluation throughput of the B200 engine (BASELINE.json metric).

Workload (N=1): BASELINE config 2 — AddPdf(GaussianPdf, ExpPdf) unbinned NLL
on 1e7 synthetic toy events in one observable x in [0, 10], grid 1024.
One step = one full eval_metric call (parameter H2D, normalisation integrals,
fused per-event pass, deterministic reduction, result D2H).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun, one rank per GPU): weak scaling — every rank owns a 1e7-event
shard (a subtree of the global reduction tree) of an N x 1e7-event data set;
the 16-byte double-double partials are all-gathered over NCCL and combined in
a fixed order, so the global NLL is bitwise identical for every N.

--impl reference: the reference's own BoundModel::eval_metric (oracle/_ref,
compiled from /root/reference's unmodified headers) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EVENTS_PER_GPU = 10_000_000
GRID = 1024
TRUTH = dict(m=5.0, s=0.8, a=-0.6, f=0.3)
START = dict(m=4.8, s=1.0, a=-0.5, f=0.4)


def make_events(n: int, seed: int = 11) -> np.ndarray:
    """Toy events of the C2 shape: f * Gauss(5, 0.8) + (1-f) * Exp(-0.6),
    truncated to [0, 10] (exact inverse-CDF sampling, numpy PCG64)."""
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    sig = rng.random(n) < TRUTH["f"]
    a = TRUTH["a"]
    # truncated exponential on [0, 10]
    xe = np.log1p(u * np.expm1(a * 10.0)) / a
    # truncated gaussian by rejection-free clipping of a wide draw
    xg = rng.normal(TRUTH["m"], TRUTH["s"], n)
    bad = (xg < 0) | (xg > 10)
    while bad.any():
        xg[bad] = rng.normal(TRUTH["m"], TRUTH["s"], int(bad.sum()))
        bad = (xg < 0) | (xg > 10)
    return np.where(sig, xg, xe)


def build_model(pf):
    x = pf.new_observable("x", 0.0, 10.0)
    m = pf.new_parameter("m", START["m"], 0.1, 0.0, 10.0)
    s = pf.new_parameter("s", START["s"], 0.1, 0.1, 5.0)
    a = pf.new_parameter("a", START["a"], 0.1, -5.0, 5.0)
    f = pf.new_parameter("f", START["f"], 0.01, 0.0, 1.0)
    pdf = pf.add_pdf("sigbkg", [pf.gaussian_pdf("sig", x, m, s), pf.exp_pdf("bkg", x, a)], [f])
    return x, pdf


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


NCU_SUMMARY = os.path.join(ROOT, "profiles", "r1_event_kernel_ncu.txt")


def ncu_metric(name):
    """one metric of the committed ncu --set full capture of pf_event_kernel
    (profiles/r1_event_kernel_ncu.txt, written by tools/ncu_summary.py), or None"""
    try:
        with open(NCU_SUMMARY) as fh:
            for line in fh:
                parts = line.split()
                if len(parts) == 2 and parts[0] == name:
                    return float(parts[1])
    except (OSError, ValueError):
        pass
    return None


def ncu_traffic():
    """dram read+write bytes per launch (ncu reports Mbyte)"""
    r = ncu_metric("dram__bytes_read.sum")
    w = ncu_metric("dram__bytes_write.sum")
    return None if r is None or w is None else (r + w) * 1e6


def cpu_baseline(pdf, x, xs, steps=4):
    """The reference (oracle/_ref) on a bounded sample, all host threads."""
    import oracle
    from paper_1311_1753_b200 import parfit as pf
    threads = os.cpu_count() or 1
    sample = min(len(xs), 2_000_000)
    ds = pf.UnbinnedDataSet.from_columns([x], xs[:sample])
    if oracle.Reference.available():
        kind, ev = "reference", oracle.Reference(pdf, ds, GRID)
        call = lambda p: ev.eval(p, 0, threads)  # noqa: E731
    else:
        kind, ev = "port", oracle.Oracle(pdf, ds, GRID)
        threads = 1
        call = lambda p: ev.eval(p, 0)  # noqa: E731
    p0 = [START["f"], START["m"], START["s"], START["a"]]
    names = ev.param_names()
    p0 = [dict(f=START["f"], m=START["m"], s=START["s"], a=START["a"])[n] for n in names]
    call(p0)
    t = time.perf_counter()
    for k in range(steps):
        p = list(p0)
        p[0] += 1e-9 * (k + 1)  # jitter: the normalisation recomputes, as in FD probes
        call(p)
    dt = (time.perf_counter() - t) / steps
    return {"value": sample / dt, "unit": "events/s", "cores": threads, "kind": kind,
            "sample": f"{sample} events of the same toy data, {steps} eval_metric calls "
                      f"(C2 model, grid {GRID}), params jittered 1e-9 per call",
            "nll_evals_per_s": 1.0 / dt, "ms_per_eval": dt * 1e3}


def run_reference(args):
    """--impl reference: the reference's BoundModel::eval_metric on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_1311_1753_b200 import parfit as pf
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparfit_ref.so not built"}))
        return
    x, pdf = build_model(pf)
    n = EVENTS_PER_GPU
    xs = make_events(n)
    ds = pf.UnbinnedDataSet.from_columns([x], xs)
    threads = os.cpu_count() or 1
    ref = oracle.Reference(pdf, ds, GRID)
    names = ref.param_names()
    p0 = [START[nm] for nm in names]
    for _ in range(args.warmup):
        ref.eval(p0, 0, threads)
    t = time.perf_counter()
    for k in range(args.steps):
        p = list(p0)
        p[0] += 1e-9 * (k + 1)
        ref.eval(p, 0, threads)
    dt = (time.perf_counter() - t) / args.steps
    val = n / dt
    line = {
        "impl": "reference", "metric": "NLL events/sec", "value": val, "unit": "events/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy PCG64 seed 11 C2 toy)",
        "config": {"workload": f"C2: AddPdf(GaussianPdf, ExpPdf) NLL, {n} events, grid {GRID}",
                   "parallelism": f"{threads} host threads (Backend::with_threads)"},
        "nll_evals_per_s": 1.0 / dt,
        "cpu_baseline": {"value": val, "unit": "events/s", "cores": threads, "kind": "reference",
                         "sample": f"full workload, {args.steps} eval_metric calls"},
        "e2e": {"value": val, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--events", type=int, default=EVENTS_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--diag-no-flush", action="store_true",
                    help="diagnostics only: keep L2 warm between steps (never a reported number)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1311_1753_b200 import parfit as pf
    x, pdf = build_model(pf)
    n_per = args.events
    n_total = n_per * world
    xs = make_events(n_total)
    ds = pf.UnbinnedDataSet.from_columns([x], xs)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(GRID), pf.Backend.gpus(1, local), shard_index=rank,
                       shard_count=world)
    names = [p.name for p in bm.registry().parameters()]
    params = np.array([START[nm] for nm in names])
    import ctypes as C
    from paper_1311_1753_b200 import _abi

    def step_value(p):
        if world == 1:
            return bm.eval_metric(p)
        import torch
        fx, pen = bm.eval_partial(p)
        t = torch.tensor(fx + [1 if pen else 0], dtype=torch.int64, device=f"cuda:{local}")
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)  # 56 bytes per rank over NCCL
        rows = [o.tolist() for o in out]
        if any(r[-1] for r in rows):
            return pf.kPenaltyValue
        return pf.combine_partials([r[:-1] for r in rows])

    for _ in range(args.warmup):
        step_value(params)
    hbm_peak, peak_kind = peaks()

    sampler = ClockSampler(local) if rank == 0 else None
    launches0 = pf.kernel_launches()
    if world == 1:
        res = _abi.pf_bench_result()
        st = _abi.pf_status()
        with sampler:
            rc = pf.lib.pf_bench(bm._h, params.ctypes.data_as(C.POINTER(C.c_double)), params.size, 0,
                                 args.steps, 0 if args.diag_no_flush else 1, C.byref(res), C.byref(st))
        if rc:
            raise RuntimeError(st.message.decode())
        launches = (res.kernels_per_step * args.steps)
        ms_step = res.step_ms_mean
        ev_ms = res.event_kernel_ms_mean
        nll = res.metric
        h2d, d2h = res.h2d_bytes_per_step, res.d2h_bytes_per_step
    else:
        import torch
        with (sampler if sampler else _Null()):
            dist.barrier()
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(args.steps):
                nll = step_value(params)
            torch.cuda.synchronize()
            dist.barrier()
            dt = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        ms_step = dt.item() / args.steps * 1e3
        ev_ms = None
        launches = pf.kernel_launches() - launches0
        h2d, d2h = 8 * params.size, 88

    # e2e: the public API call (pf_eval_metric via BoundModel.eval_metric) with
    # host parameters in and the host scalar out, host wall clock, L2 flushed
    # (by a device memset outside the window) before every step
    e2e_times = []
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    for k in range(min(args.steps, 50)):
        flush.fill_(k & 0xff)
        torch.cuda.synchronize()
        t = time.perf_counter()
        step_value(params)
        e2e_times.append(time.perf_counter() - t)
    e2e_s = statistics.mean(e2e_times)
    if world > 1:
        v = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        e2e_s = v.item()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    events_per_s = n_total / (ms_step * 1e-3)
    line = {
        "metric": "NLL events/sec", "value": events_per_s, "unit": "events/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy PCG64 seed 11 C2 toy: 0.3 Gauss(5,0.8) + 0.7 Exp(-0.6) on [0,10])",
        "config": {"workload": f"C2: AddPdf(GaussianPdf, ExpPdf) unbinned NLL, {n_per} events/GPU, "
                               f"grid {GRID}, params at the fit start",
                   "events_per_gpu": n_per, "global_events": n_total,
                   "l2": "flushed (256 MiB device write) before every timed step",
                   "parallelism": f"dp{world}"},
        "nll_evals_per_s": 1e3 / ms_step,
        "nll": nll,
        "gpu_launches": int(launches),
        "e2e": {"value": n_total / e2e_s, "unit": "events/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3},
        "clocks": sampler.summary() if sampler else None,
    }
    if ev_ms:
        algo_bytes = 8.0 * n_per  # one f64 column per event (EventTable layout)
        achieved = algo_bytes / (ev_ms * 1e-3) / 1e9
        line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                            "frac": achieved / hbm_peak, "traffic": ncu_traffic(),
                            "traffic_source": "profiles/r1_event_kernel_ncu.txt (ncu --set full, 1 launch)",
                            "kernel": "pf_event_kernel", "kernel_ms": ev_ms,
                            "algorithmic_bytes_per_launch": algo_bytes,
                            "kernel_share_of_step": ev_ms / ms_step, "peak_kind": peak_kind}
        # the event pass is issue/FP64-pipe limited, not HBM limited: report
        # the ncu-measured pipe utilisation of the same capture beside it
        fp64 = ncu_metric("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        issue = ncu_metric("smsp__issue_active.avg.pct_of_peak_sustained_active")
        if fp64 is not None:
            line["roofline"]["fp64_pipe_active_frac_ncu"] = fp64 / 100.0
        if issue is not None:
            line["roofline"]["issue_active_frac_ncu"] = issue / 100.0
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(pdf, x, xs)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    main()
