"""`parfit bench` over GPU counts.

Mirrors `cmd_bench` (proj/tools/parfit_cli.cpp:110-182) with GPU counts in
place of thread counts:

  python -m paper_1311_1753_b200 bench --workload C2 --gpus 1 2 --repetitions 3
      [--events N] [--data events.txt] [--out report.txt]

* the same arity rules and error codes: >= 3 repetitions and >= 2 distinct
  counts including 1, else ``bad-arity`` (parfit_cli.cpp:113-122);
* every repetition refits from the workload's start point; a row reports the
  median fit wall time, the metric and the call count of its last fit
  (:135-160);
* determinism gate: every row must land on the bitwise-identical metric, else
  ``determinism-violation`` (:163-166). The exact accumulator makes the sum
  independent of where the events split, so the gate holds across GPU counts;
* report: ``backend gpus time_s speedup metric_calls`` then one
  ``gpus N t s calls`` row per count, speedup = t(1) / t(N), exactly 1 for N = 1
  (:168-179; cli_smoke.sh:48-61).

The model comes from a BASELINE workload (`workloads.py`) instead of the
reference's JSON config loader, which is out of scope (DESIGN "Out of scope").
``--data`` reads the reference's `%.17g` text format (dataset.hpp:184-245).
"""
from __future__ import annotations

import argparse
import sys
from typing import List, Optional, Sequence


def _dataset(pf, W, obs, n: Optional[int], data_path: Optional[str]):
    if data_path:
        return pf.read_text_file(data_path, obs)
    return W.data(pf, obs, n or W.fit_n)


def bench_rows(workload: str, gpu_counts: Sequence[int], repetitions: int,
               n_events: Optional[int] = None, data_path: Optional[str] = None,
               oversubscribe: bool = False) -> List[dict]:
    """One row per GPU count (no arity checks: `cmd_bench` applies them)."""
    from . import parfit as pf
    from .workloads import WORKLOADS
    if workload not in WORKLOADS:
        raise pf.Error("bad-config", f"unknown workload {workload!r} (one of {sorted(WORKLOADS)})")
    W = WORKLOADS[workload]
    obs, pdf = W.build(pf)
    ds = _dataset(pf, W, obs, n_events, data_path)
    rows = []
    for n in gpu_counts:
        times, last, metrics = [], None, set()
        for _ in range(repetitions):
            # one BoundModel per repetition, as the reference builds one per
            # run (parfit_cli.cpp:147-152); identical start every run
            bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid), pf.Backend.gpus(n, oversubscribe=oversubscribe))
            for p in bm.registry().parameters():
                p.value = W.start[p.name]
            r = pf.fit(bm, pf.MetricKind(W.metric))
            times.append(r.wall_time_s)
            metrics.add(r.metric_value)
            last = r
            del bm
        if len(metrics) != 1:
            raise pf.Error("determinism-violation", f"metric value differs across repetitions at {n} GPUs")
        times.sort()
        rows.append({"gpus": n, "median_s": times[len(times) // 2], "metric_value": last.metric_value,
                     "metric_calls": last.n_metric_calls})
    return rows


def format_report(rows: Sequence[dict]) -> str:
    t1 = next((r["median_s"] for r in rows if r["gpus"] == 1), 0.0)
    out = ["backend gpus time_s speedup metric_calls\n"]
    for r in rows:
        speedup = 1.0 if r["gpus"] == 1 else t1 / r["median_s"]
        out.append("gpus %u %.6g %.4g %d\n" % (r["gpus"], r["median_s"], speedup, r["metric_calls"]))
    return "".join(out)


def cmd_bench(workload: str, gpu_counts: Sequence[int], repetitions: int, n_events: Optional[int] = None,
              data_path: Optional[str] = None, out_path: Optional[str] = None, oversubscribe: bool = False) -> int:
    from .parfit import Error
    if repetitions < 3:
        raise Error("bad-arity", "bench needs >= 3 repetitions")
    counts = sorted(set(int(c) for c in gpu_counts))
    if len(counts) < 2 or 1 not in counts:
        raise Error("bad-arity", "bench needs >= 2 GPU counts including 1")
    # the engine shards over powers of two (contiguous subtrees of the
    # reduction tree) and never oversubscribes here: checked before any work
    bad = [c for c in counts if c & (c - 1)]
    if bad:
        raise Error("bad-backend", f"GPU counts must be powers of two (got {bad})")
    from .parfit import device_count
    have = device_count()
    if counts[-1] > have and not oversubscribe:
        raise Error("bad-backend", f"bench asks for {counts[-1]} GPUs, {have} visible")
    rows = bench_rows(workload, counts, repetitions, n_events, data_path, oversubscribe)
    if any(r["metric_value"] != rows[0]["metric_value"] for r in rows):
        raise Error("determinism-violation", "metric value differs across GPU counts: bench aborted")
    report = format_report(rows)
    if out_path:
        with open(out_path, "w") as f:
            f.write(report)
    else:
        sys.stdout.write(report)
    return 0


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1311_1753_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="median fit time over GPU counts, with the bitwise determinism gate")
    b.add_argument("--workload", default="C2")
    b.add_argument("--gpus", type=int, nargs="+", required=True)
    b.add_argument("--repetitions", type=int, default=3)
    b.add_argument("--events", type=int, default=None)
    b.add_argument("--data", default=None)
    b.add_argument("--out", default=None)
    b.add_argument("--oversubscribe", action="store_true",
                   help="place the shards of a count above the visible devices round-robin on them "
                        "(exercises the multi-device path and the determinism gate on fewer GPUs; "
                        "the speedup column then measures nothing)")
    a = ap.parse_args(argv)
    from .parfit import Error
    try:
        return cmd_bench(a.workload, a.gpus, a.repetitions, a.events, a.data, a.out, a.oversubscribe)
    except Error as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
