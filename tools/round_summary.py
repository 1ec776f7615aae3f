"""Markdown table of one measurement round's bench lines (tools/final_round.sh TAG
output copied to profiles/): step, value, e2e, roofline, parity, the reference arm.
  python tools/round_summary.py r2c > /tmp/table.md"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2c"
d = os.path.join(ROOT, "profiles")


def line(path):
    try:
        with open(path) as fh:
            rows = [r for r in fh.read().strip().splitlines() if r.startswith("{")]
        return json.loads(rows[-1]) if rows else None
    except OSError:
        return None


def si(v):
    if v is None:
        return "—"
    e = 0
    while abs(v) >= 10:
        v /= 10
        e += 1
    return "%.2f×10^%d" % (v, e)


print("| Config | step (device) | value | e2e | roofline (kernel) | parity at full size | reference arm |")
print("|---|---|---|---|---|---|---|")
for c in ["c1", "c2", "c3", "c4", "c5", "c5ti"]:
    g = line(os.path.join(d, "%s_%s.json" % (tag, c)))
    r = line(os.path.join(d, "%s_%s_ref.json" % (tag, c)))
    if not g:
        continue
    rf = g.get("roofline", {})
    roof = "%s %.3f (%s %.1f µs)" % (rf.get("bound", "?"), rf.get("frac", float("nan")), rf.get("kernel", "?"),
                                     1e3 * rf.get("kernel_ms", float("nan")))
    par = g.get("parity") or {}
    ref = "%s %s (%s, %s threads)" % (si(r.get("value")), r.get("unit", ""), (r.get("cpu_baseline") or {}).get("kind"),
                                      (r.get("cpu_baseline") or {}).get("cores")) if r else "—"
    if r and r.get("unavailable"):
        ref = "unavailable: " + r["unavailable"]
    print("| %s | %.1f µs | %s %s | %s | %s | %s (%s) | %s |" % (
        c.upper(), 1e3 * g["ms_per_step"], si(g["value"]), g["unit"], si((g.get("e2e") or {}).get("value")),
        roof, "%.1e" % par["rel"] if "rel" in par else "—", par.get("kind", "—"), ref))
