#!/usr/bin/env python3
"""bench.py — NLL evaluation throughput of the B200 engine (BASELINE.json metric).

Workload (default, N=1): BASELINE config 2 — AddPdf(GaussianPdf, ExpPdf)
unbinned NLL on 1e7 synthetic events per GPU, x in [0, 10], grid 1024.
One step = one full eval_metric call (validity, normalisation integrals,
fused per-event pass, exact reduction, result on the host).
--config C1|C3|C4 selects the other BASELINE configurations
(paper_1311_1753_b200/workloads.py).

  python bench.py [--gpus N --steps K --warmup W] [--config C2] [--impl reference]

N > 1 (torchrun, one rank per GPU): every rank owns its own events (weak
scaling: 1e7 per GPU for C2; strong: the C3 total split N ways); each rank's
exact fixed-point digits (48 bytes) are all-gathered over NCCL and combined
exactly, so the global value does not depend on the combine order.

--impl reference: the reference's own BoundModel::eval_metric (oracle/_ref,
compiled from /root/reference's unmodified headers) on the host cores; for
ArgusPdf (C3), which the reference lacks, the C restatement (oracle port).
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

from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402

# C2 (the default workload), kept importable for tools/
START = WORKLOADS["C2"].start


def make_events(n: int, seed: int = 11) -> np.ndarray:
    return WORKLOADS["C2"].columns(n, seed)


def build_model(pf):
    obs, pdf = WORKLOADS["C2"].build(pf)
    return obs[0], pdf


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


NCU_TAGS = ("r2f", "r2e", "r2d", "r2c", "r2", "r1n", "r1m", "r1l", "r1j", "r1i", "r1h", "r1g", "r1f", "r1e")  # newest first
FP64_BOUND = ("C4", "C5", "C5TI")  # FP64-pipe-bound configs (ncu: FP64 pipe 42-61 %, HBM < 11 %)


def fp64_peak():
    """the builder-measured FP64 peak (profiles/fp64_peak.json: a DFMA
    microkernel, tools/fp64_peak.cu) -- MEASURED_PEAKS.json has none"""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            return float(json.load(fh)["fp64_tflops"]), "builder-measured (profiles/fp64_peak.json, DFMA microkernel)"
    except Exception:
        return 37.0, "nominal (148 SM x 64 DFMA/clk x 2 x 1.965 GHz)"


def fp64_ops(config):
    """algorithmic FP64 flops per unit of the config's dominant kernel, from
    the newest committed SASS op-count capture (tools/fp64_count.sh ->
    profiles/<tag>_fp64_ops.json; DADD, DMUL 1 flop, DFMA 2)"""
    for tag in NCU_TAGS:
        p = os.path.join(ROOT, "profiles", f"{tag}_fp64_ops.json")
        if os.path.exists(p):
            with open(p) as fh:
                d = json.load(fh)
            if config in d:
                return d[config], os.path.relpath(p, ROOT)
    return None, None


def ncu_summary_path(config):
    """the newest committed ncu --set full capture of this config's event
    kernel (tools/ncu_summary.py output under profiles/)"""
    for tag in NCU_TAGS:
        p = os.path.join(ROOT, "profiles", f"{tag}_{config.lower()}_event_ncu.txt")
        if os.path.exists(p):
            return p
    return os.path.join(ROOT, "profiles", f"{NCU_TAGS[0]}_{config.lower()}_event_ncu.txt")


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_metric(config, name):
    """(value, unit) of one metric of the committed capture, or (None, None)"""
    try:
        with open(ncu_summary_path(config)) as fh:
            for line in fh:
                parts = line.split()
                if len(parts) >= 2 and parts[0] == name:
                    return float(parts[1]), (parts[2] if len(parts) > 2 else "")
    except (OSError, ValueError):
        pass
    return None, None


def ncu_traffic(config):
    """DRAM read + write bytes of one event-kernel launch"""
    total = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = ncu_metric(config, m)
        if v is None or u not in _SCALE:
            return None
        total += v * _SCALE[u]
    return total


def workload_config(W, n_local, n_total, world, exchange=None):
    """the `config` dict of BOTH arms (ours and --impl reference): byte-identical
    for the same workload and GPU count"""
    return {"workload": f"{W.name}: {W.description}, {n_local} {W.unit}/GPU, grid {W.grid}, "
                        f"params at the fit start",
            f"{W.unit}_per_gpu": n_local, f"global_{W.unit}": n_total,
            "data": data_description(W),
            "l2": "flushed (256 MiB device write) before every timed step",
            "parallelism": f"dp{world}",
            "exchange": exchange}


def data_description(W):
    if W.name == "C2":
        return ("reference generate_events(AddPdf at truth m=5 s=0.8 a=-0.6 f=0.3, seed 11 + rank) "
                "(generate.hpp:33-86; GPU arm: the bit-identical GPU generator)")
    return f"synthetic ({W.name}, numpy PCG64 seed 11 + rank; {W.description})"


def _at_truth(W, pf):
    obs, pdf = W.build(pf)
    for v in pf.GraphDesc(pdf, obs).vars:
        if v.name in W.truth:
            v.value = W.truth[v.name]
    return obs, pdf


def workload_columns(W, pf, n, seed, device=None):
    """the event columns of a workload.  C2: the reference's own generator
    (generate.hpp:33-86, mt19937_64 seed) at the truth point -- on the GPU for
    our arm (pf.generate_events reproduces the reference stream bit for bit,
    tests/test_gpu_generate.py), oracle/_ref's generate_events for the
    reference arm; the other configs: numpy (workloads.py)."""
    if W.name != "C2":
        return W.columns(n, seed=seed)
    obs, pdf = _at_truth(W, pf)
    if device is None:
        import oracle
        return oracle.ref_generate(pdf, obs, n, seed, W.grid)
    ds = pf.generate_events(pdf, obs, n, seed, pf.GridSpec(W.grid), device=device)
    return np.ascontiguousarray(pf.to_event_table(ds)[0])


def cpu_side(W, pf, obs, pdf, ds_full, metric, gpu_value=None, steps=3):
    """The CPU legs, rank 0 at N = 1 (test infrastructure: oracle/ only as the
    checker and the CPU baseline, never as the measured path):
      cpu_baseline -- the reference (oracle/_ref, all host threads) or, for
                      the PDFs it cannot express (ArgusPdf, DalitzPlotPdf),
                      the C restatement with its event loop on all host
                      threads, timed on a bounded sample of the same data;
      parity       -- ONE evaluation of the same (reference or port) on the
                      FULL benchmarked data at the benchmarked parameters,
                      against the GPU's metric value (north_star bar: 1e-12)."""
    import oracle
    threads = os.cpu_count() or 1
    n_full = ds_full.n_bins() if W.unit == "bins" else ds_full.n_events()
    if W.unit == "bins":
        sample = min(n_full, 100_000)
        ds = W.data(pf, obs, sample) if sample < n_full else ds_full
    else:
        sample = min(n_full, 2_000_000)
        ds = ds_full if sample == n_full else pf.UnbinnedDataSet.from_columns(
            obs, np.ascontiguousarray(pf.to_event_table(ds_full)[:, :sample]))
    use_ref = oracle.Reference.available() and W.has_reference
    make = (lambda d: oracle.Reference(pdf, d, W.grid)) if use_ref else (lambda d: oracle.Oracle(pdf, d, W.grid))
    kind = "reference" if use_ref else "port"
    ev = make(ds)
    call = lambda e, p: e.eval(p, metric, threads)  # noqa: E731
    p0 = [W.start[n] for n in ev.param_names()]
    call(ev, p0)
    t = time.perf_counter()
    for k in range(steps):
        p = list(p0)
        p[0] += 1e-9 * (k + 1)  # jitter: the normalisation recomputes, as in FD probes
        call(ev, p)
    dt = (time.perf_counter() - t) / steps
    out = {"value": sample / dt, "unit": f"{W.unit}/s", "cores": threads, "kind": kind,
           "sample": f"{sample} {W.unit} of the same data, {steps} eval_metric calls "
                     f"({W.name}, grid {W.grid}), params jittered 1e-9 per call, {threads} host threads"
                     + (" (Backend::with_threads)" if use_ref else " (C restatement, event loop threaded)"),
           "evals_per_s": 1.0 / dt, "ms_per_eval": dt * 1e3}
    parity = None
    if gpu_value is not None:
        del ev
        full = make(ds_full) if ds is not ds_full else make(ds)
        t = time.perf_counter()
        ref_value = call(full, p0)
        parity = {"ref_value": ref_value, "gpu_value": gpu_value,
                  "rel": abs(gpu_value - ref_value) / max(abs(ref_value), 1e-300),
                  "units": n_full, "kind": kind, "ref_s": time.perf_counter() - t,
                  "bar": 1e-12}
    return out, parity


def fit_leg(W, pf, obs, pdf, cols, device):
    """GPU fit and reference fit (all host threads) of the same sample"""
    import oracle
    n = W.fit_n
    if cols is None:
        ds = W.data(pf, obs, n)
    else:
        n = min(n, cols.shape[-1])
        ds = pf.UnbinnedDataSet.from_columns(obs, np.ascontiguousarray(cols[..., :n]))
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid), pf.Backend.gpus(1, device))
    for p in bm.registry().parameters():  # start point
        p.value = W.start[p.name]
    r = pf.fit(bm, pf.MetricKind(W.metric))
    out = {"units": n, "gpu_wall_s": r.wall_time_s, "gpu_calls": r.n_metric_calls, "gpu_status": int(r.status),
           "params": dict(zip(r.names, r.params))}
    if oracle.Reference.available() and W.has_reference:
        for p in bm.registry().parameters():  # the fit wrote its result back: same start
            p.value = W.start[p.name]
        threads = os.cpu_count() or 1
        rr = oracle.Reference(pdf, ds, W.grid).fit(W.metric, threads)
        out.update({"ref_wall_s": rr["wall_time_s"], "ref_calls": int(rr["calls"]),
                    "ref_status": int(rr["status"]), "ref_threads": threads,
                    "speedup": rr["wall_time_s"] / r.wall_time_s if r.wall_time_s > 0 else None,
                    "max_rel_param_diff": float(max(abs(a - b) / max(abs(b), 1e-300)
                                                    for a, b in zip(r.params, rr["params"])))})
    return out


def sizes(W, args, world, rank):
    """(events or bins on this rank, total over ranks)"""
    if W.scaling == "weak":
        n_local = args.events or W.default_n
        return n_local, n_local * world
    n_total = args.events or W.default_n
    return n_total // world + (1 if rank < n_total % world else 0), n_total


def exchange_description(args, multi):
    if not multi:
        return None
    if args.exchange == "p2p":
        return ("p2p: exact digit records stored over NVLink into every rank's buffer by the event pass "
                "(CUDA IPC), summed on device")
    return "nccl: device records all-gathered on the model stream"


def run_reference(args):
    """--impl reference: the reference's BoundModel::eval_metric on host cores.

    Only the reference (oracle/_ref/libparfit_ref.so, compiled from the
    unmodified headers) or, for PDFs the reference lacks, the C restatement
    runs here: libpfb200.so is never loaded in this process (the product's
    ctypes binding is lazy and only the pure-Python model description is
    used)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_1311_1753_b200 import parfit as pf
    W = WORKLOADS[args.config]
    if not oracle.Reference.available() and W.has_reference:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparfit_ref.so not built"}))
        return
    obs, pdf = W.build(pf)
    n_local, n_total = sizes(W, args, world, rank)
    n = n_local
    if W.unit == "bins":
        n = min(n, 100_000)  # one reference chi-squared call on 1e6 bins x Q=1024 takes ~5 s on 16 threads
    elif not W.has_reference:
        n = min(n, 2_000_000)
    if W.unit == "bins":
        ds = W.data(pf, obs, n)
    else:
        ds = pf.UnbinnedDataSet.from_columns(obs, workload_columns(W, pf, n, 11))
    threads = os.cpu_count() or 1
    if not W.has_reference:  # ArgusPdf / DalitzPlotPdf: the C restatement stands in
        kind, ev = "port", oracle.Oracle(pdf, ds, W.grid)
        call = lambda p: ev.eval(p, W.metric, threads)  # noqa: E731
    else:
        kind, ev = "reference", oracle.Reference(pdf, ds, W.grid)
        call = lambda p: ev.eval(p, W.metric, threads)  # noqa: E731
    p0 = [W.start[nm] for nm in ev.param_names()]
    metric_value = call(p0)
    for _ in range(args.warmup):
        call(p0)
    t = time.perf_counter()
    for k in range(args.steps):
        p = list(p0)
        p[0] += 1e-9 * (k + 1)  # jitter: the normalisation recomputes, as in FD probes
        call(p)
    dt = (time.perf_counter() - t) / args.steps
    val = n / dt
    metric_name = "NLL events/sec" if W.metric == 0 else "chi2 bins/sec"
    sample = (f"{n} {W.unit} (rank 0's data{'' if n == n_local else ', a bounded prefix'}), "
              f"{args.steps} eval_metric calls, params jittered 1e-9 per call")
    line = {
        "impl": "reference", "metric": metric_name, "value": val, "unit": f"{W.unit}/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": W.scaling, "vs_baseline": None, "dtype": "f64",
        "data": data_description(W),
        "config": workload_config(W, n_local, n_total, world,
                                  exchange_description(args, world > 1 or args.force_exchange)),
        "evals_per_s": 1.0 / dt,
        "metric_value": metric_value, "metric_value_units": n,
        "cpu_baseline": {"value": val, "unit": f"{W.unit}/s", "cores": threads, "kind": kind,
                         "sample": sample,
                         "threads": f"{threads} host threads" + (" (Backend::with_threads)" if kind == "reference"
                                                                  else " (C restatement, event loop threaded)")},
        "e2e": {"value": val, "unit": f"{W.unit}/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--events", type=int, default=0, help="events (bins) per GPU; 0: the config's size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fit", action="store_true")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: p2p = exact records stored into every rank's buffer by the event pass "
                         "over NVLink (CUDA IPC); nccl = device records all-gathered by NCCL on the model stream")
    ap.add_argument("--force-exchange", action="store_true",
                    help="run the multi-rank exchange path even with one rank (tests it on one GPU)")
    ap.add_argument("--diag-no-flush", action="store_true",
                    help="diagnostics only: keep L2 warm between steps (never a reported number)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    W = WORKLOADS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    multi = world > 1 or args.force_exchange
    if multi:
        import torch
        import torch.distributed as dist
        # communicator logging on (NCCL's "comm ... nRanks" lines show every rank joined)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1311_1753_b200 import parfit as pf
    obs, pdf = W.build(pf)
    n_local, n_total = sizes(W, args, world, rank)
    # every rank owns its own events (seed per rank); the exact digits of the
    # ranks' partial sums are combined, so the order of combination is free
    if W.unit == "bins":
        ds = W.data(pf, obs, n_local, seed=11 + rank)
        cols = None
    else:
        cols = workload_columns(W, pf, n_local, 11 + rank, device=local)
        ds = pf.UnbinnedDataSet.from_columns(obs, cols)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid), pf.Backend.gpus(1, local))
    params = W.params(bm)
    metric = pf.MetricKind(W.metric)
    import ctypes as C
    from paper_1311_1753_b200 import _abi

    if multi:
        # the exchange, stream-ordered on the model's own stream: the event
        # pass writes its exact digits to a device record (aliased here as a
        # torch tensor), NCCL all-gathers the 64-byte records, one D2H brings
        # them to the host, where every rank combines them identically
        import torch

        class _DeviceRecord:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                                 "version": 3}

        part_d = torch.as_tensor(_DeviceRecord(bm.partial_device(), 8), device=f"cuda:{local}")
        model_stream = torch.cuda.ExternalStream(bm.stream(), device=f"cuda:{local}")
        recv_d = torch.empty(8 * world, dtype=torch.int64, device=f"cuda:{local}")
        if args.exchange == "p2p":
            # the peer-memory group: handles exchanged once, then every
            # evaluation combines on the device and returns the global value.
            # Where CUDA IPC / peer access is unavailable, every rank falls
            # back to the NCCL record exchange together.
            ok = torch.ones(1, dtype=torch.int32, device=f"cuda:{local}")
            try:
                handles = [None] * world
                dist.all_gather_object(handles, bm.group_handle())
                bm.group_join(world, rank, handles)
                # every rank's receive buffer is reset by its own join: no
                # record may be sent before every rank has joined
                dist.barrier()
                bm.eval_metric(params, metric)  # one grouped call: the peers' records must arrive
            except Exception as e:  # noqa: BLE001 - reported, then the fallback
                print(f"rank {rank}: peer-memory group unavailable ({e}); using NCCL", file=sys.stderr)
                ok.zero_()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 0:
                args.exchange = "nccl"
                bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid), pf.Backend.gpus(1, local))  # ungrouped
                part_d = torch.as_tensor(_DeviceRecord(bm.partial_device(), 8), device=f"cuda:{local}")
                model_stream = torch.cuda.ExternalStream(bm.stream(), device=f"cuda:{local}")
            dist.barrier()

    def step_value(p):
        if not multi or args.exchange == "p2p":
            return bm.eval_metric(p, metric)
        if bm.eval_launch(p, metric):  # invalid parameters: the same on every rank
            return pf.kPenaltyValue
        with torch.cuda.stream(model_stream):
            dist.all_gather_into_tensor(recv_d, part_d)
            rows = recv_d.cpu().view(world, 8).tolist()
        if any(r[6] != 0xFFFFFFFF or r[7] for r in rows):  # zero integral or a non-finite term
            return pf.kPenaltyValue
        return pf.combine_partials([r[:6] for r in rows])

    for _ in range(args.warmup):
        step_value(params)
    hbm_peak, peak_kind = peaks()

    sampler = ClockSampler(local) if rank == 0 else None
    launches0 = pf.kernel_launches()
    if not multi or args.exchange == "p2p":
        # device timing inside the library (CUDA events around each graph
        # launch on the model stream, L2 flushed before each, outside the
        # window); in an exchange group every rank runs it in lockstep, each
        # launch including the peer-memory exchange, and the MAX is taken
        res = _abi.pf_bench_result()
        st = _abi.pf_status()
        if multi:
            dist.barrier()
        with (sampler if sampler else _Null()):
            rc = pf.lib.pf_bench(bm._h, params.ctypes.data_as(C.POINTER(C.c_double)), params.size, W.metric,
                                 args.steps, 0 if args.diag_no_flush else 1, C.byref(res), C.byref(st))
        if rc:
            raise RuntimeError(st.message.decode())
        launches = (res.kernels_per_step * args.steps)
        ms_step = res.step_ms_mean
        ev_ms = res.event_kernel_ms_mean
        value = res.metric
        h2d, d2h = res.h2d_bytes_per_step, res.d2h_bytes_per_step
        if multi:
            import torch
            t = torch.tensor([ms_step, ev_ms], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_step, ev_ms = t.tolist()
    else:
        # NCCL exchange: CUDA events on the model stream around every step
        # (evaluation + collective + D2H), L2 flushed before each, MAX over ranks
        import torch
        flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
        total_ms = 0.0
        with (sampler if sampler else _Null()):
            dist.barrier()
            for k in range(args.steps):
                with torch.cuda.stream(model_stream):
                    flush_buf.fill_(k & 0xff)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(model_stream)
                value = step_value(params)
                with torch.cuda.stream(model_stream):
                    e1.record(model_stream)
                e1.synchronize()
                total_ms += e0.elapsed_time(e1)
            dt = torch.tensor([total_ms / args.steps], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        ms_step = dt.item()
        ev_ms = None
        launches = pf.kernel_launches() - launches0
        h2d, d2h = 8 * params.size, 64 * world

    # e2e: the public API call (pf_eval_metric via BoundModel.eval_metric) with
    # host parameters in and the host scalar out, host wall clock, L2 flushed
    # (by a device memset outside the window) before every step
    e2e_times = []
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    for k in range(50):  # e2e samples (the device-timed value uses exactly --steps)
        flush.fill_(k & 0xff)
        torch.cuda.synchronize()
        t = time.perf_counter()
        step_value(params)
        e2e_times.append(time.perf_counter() - t)
    # the median call: host wall-clock samples carry OS scheduling outliers
    # (the mean is reported beside it)
    e2e_s = statistics.median(e2e_times)
    e2e_mean_s = statistics.mean(e2e_times)
    if multi:
        v = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        e2e_s = v.item()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    metric_name = "NLL events/sec" if W.metric == 0 else "chi2 bins/sec"
    line = {
        "metric": metric_name, "value": n_total / (ms_step * 1e-3), "unit": f"{W.unit}/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": W.scaling, "vs_baseline": None, "dtype": "f64",
        "data": data_description(W),
        "config": workload_config(W, n_local, n_total, world, exchange_description(args, multi)),
        "evals_per_s": 1e3 / ms_step,
        "metric_value": value,
        "gpu_launches": int(launches),
        "e2e": {"value": n_total / e2e_s, "unit": f"{W.unit}/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3, "statistic": "median",
                "calls": len(e2e_times), "ms_per_step_mean": e2e_mean_s * 1e3},
        "clocks": sampler.summary() if sampler else None,
    }
    if ev_ms:
        algo_bytes = W.bytes_per_unit() * n_local  # EventTable columns read per call
        achieved = algo_bytes / (ev_ms * 1e-3) / 1e9
        kernel = res_kernel_name(bm)
        hbm = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
               "frac": achieved / hbm_peak,
               "traffic": ncu_traffic(W.name),
               "traffic_source": os.path.relpath(ncu_summary_path(W.name), ROOT) + " (ncu --set full, 1 launch)",
               "kernel": kernel, "kernel_ms": ev_ms,
               "algorithmic_bytes_per_launch": algo_bytes,
               "kernel_share_of_step": ev_ms / ms_step, "peak_kind": peak_kind}
        ops, ops_src = fp64_ops(W.name)
        fp64 = None
        if ops:
            pk, pk_kind = fp64_peak()
            flops = ops["flops_per_unit"] * n_local
            fa = flops / (ev_ms * 1e-3) / 1e12
            fp64 = {"bound": "fp64", "achieved": fa, "peak": pk, "unit": "TFLOP/s", "frac": fa / pk,
                    "traffic": hbm["traffic"], "kernel": kernel, "kernel_ms": ev_ms,
                    "algorithmic_flops_per_launch": flops, "flops_per_unit": ops["flops_per_unit"],
                    "flops_source": ops_src + " (DADD, DMUL = 1 flop, DFMA = 2; per unit, ncu SASS op counters)",
                    "kernel_share_of_step": ev_ms / ms_step, "peak_kind": pk_kind}
        if W.name in FP64_BOUND and fp64:
            line["roofline"] = fp64
            line["roofline"]["hbm_view"] = {k: hbm[k] for k in ("achieved", "peak", "unit", "frac")}
        else:
            line["roofline"] = hbm
            if fp64:
                line["roofline"]["fp64_view"] = {k: fp64[k] for k in ("achieved", "peak", "unit", "frac",
                                                                      "flops_per_unit")}
        # the event pass is issue/FP64-pipe limited rather than HBM limited:
        # the ncu-measured pipe utilisation of the same capture beside it
        fp64p, _ = ncu_metric(W.name, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        issue, _ = ncu_metric(W.name, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        if fp64p is not None:
            line["roofline"]["fp64_pipe_active_frac_ncu"] = fp64p / 100.0
        if issue is not None:
            line["roofline"]["issue_active_frac_ncu"] = issue / 100.0
    if world == 1 and not args.no_fit and W.has_reference:  # otherwise no reference fit to compare with
        # full fit (fit.hpp:498-581) from the start point, GPU and reference
        # on the same bounded sample (at 1e7 events the reference's absolute
        # gradient tolerance is below the NLL's rounding noise and neither
        # side converges before max_iterations)
        line["fit"] = fit_leg(W, pf, obs, pdf, cols, local)
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"], line["parity"] = cpu_side(W, pf, obs, pdf, ds, W.metric, gpu_value=value)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def res_kernel_name(bm):
    """the kernel the bench's event timing measures: the single fused kernel
    (setup + event pass, K = 1 small-grid models) or the event pass"""
    import ctypes as C
    from paper_1311_1753_b200 import parfit as pf
    try:
        return "pf_fused_kernel" if pf.lib.pf_model_fused(bm._h) else "pf_event_kernel"
    except AttributeError:
        return "pf_event_kernel"


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    main()
