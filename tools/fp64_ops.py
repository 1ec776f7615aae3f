"""profiles/<tag>_fp64_ops.json from the ncu SASS op-count captures of
tools/fp64_count.sh: per config, the dominant kernel's DADD/DMUL/DFMA thread
instructions per unit (event or bin) and the algorithmic FP64 flops per unit
(DADD, DMUL = 1 flop; DFMA = 2), which bench.py's FP64 roofline uses."""
import csv
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
units = {"C2": 10_000_000, "C4": 1_000_000, "C5": 1_000_000, "C5TI": 1_000_000}
out = {}
for cfg, n in units.items():
    path = os.path.join("gpurun_out", f"{tag}_fp64_{cfg}.csv")
    if not os.path.exists(path):
        continue
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    vals = {}
    kernel = None
    for r in rows:
        kernel = r[4]
        name, unit, v = r[-3], r[-2], r[-1]
        vals[name] = (float(v.replace(",", "")), unit)
    get = lambda k: vals.get(k, (0.0, ""))[0]  # noqa: E731
    dadd = get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum")
    dmul = get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum")
    dfma = get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum")
    out[cfg] = {"kernel": kernel, "units": n, "dadd": dadd, "dmul": dmul, "dfma": dfma,
                "flops_per_unit": (dadd + dmul + 2 * dfma) / n,
                "fp64_instr_per_unit": (dadd + dmul + dfma) / n,
                "ncu_time": vals.get("gpu__time_duration.sum"),
                "fp64_pipe_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "source": path + " (ncu --metrics sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum, 1 launch)"}
json.dump(out, open(os.path.join("profiles", f"{tag}_fp64_ops.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
