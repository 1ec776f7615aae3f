"""SASS evidence of the generated evaluator (cuobjdump -sass of the nvcc
build-check cubin, __graft_entry__.build): per-kernel instruction counts,
opcode histograms, every TMA bulk copy / mbarrier instruction, and an
excerpt of the C2 quadratic mixture fast path (pf_qfast_terms).
  python tools/sass_summary.py paper_1311_1753_b200/_build/canonical_c2.cubin > profiles/<tag>_c2_sass.txt"""
import collections
import re
import subprocess
import sys

sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout.splitlines()
funcs, cur = collections.OrderedDict(), None
for line in sass:
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
    elif cur and re.match(r"\s+/\*[0-9a-f]+\*/", line):
        funcs[cur].append(line)
print(f"# cuobjdump -sass {sys.argv[1]}")
for name, lines in funcs.items():
    ops = collections.Counter(re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?", "", l).split()[0].split(".")[0]
                              for l in lines if l.strip())
    print(f"\n## {name}: {len(lines)} instructions")
    print("   " + ", ".join(f"{k} {v}" for k, v in ops.most_common(24)))
    for l in lines:
        if re.search(r"UBLKCP|UTMALDG|SYNCS|BLKCP", l):
            print("   " + l.strip().split(";")[0] + ";")
fused = funcs.get("pf_fused_kernel", [])
for i, l in enumerate(fused):
    if "6.75539944105574400000e+15" in l and "|" in l:  # kd = fma(-|d|, 1024/ln2, 1.5 2^52)
        print("\n## pf_fused_kernel: pf_qfast_terms excerpt (one event: d by 2 DFMA, e^-|d| by the 1024-entry table)")
        for x in fused[max(0, i - 12): i + 28]:
            print("   " + x.strip().split(";")[0] + ";")
        break
