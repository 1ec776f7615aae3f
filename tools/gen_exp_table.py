#!/usr/bin/env python3
"""Generates paper_1311_1753_b200/csrc/device/pf_exp_table.cuh: the 128-entry
2^(j/128) table (hi + lo split) and the ln2/128 constants of the device
table-driven exp (pf_device.cuh pf_exp).  60-digit decimal arithmetic."""
import math
import os
import struct
from decimal import Decimal, getcontext

getcontext().prec = 60
LN2 = Decimal(2).ln()
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1311_1753_b200", "csrc",
                   "device", "pf_exp_table.cuh")


def main():
    lines = ["// 2^(j/128) = hi + lo (hi = RN(2^(j/128)), lo = RN(residual)); generated with",
             "// Python decimal at 60 digits (tools/gen_exp_table.py)",
             "__device__ const __align__(16) double pf_exp_tab_g[256] = {"]
    for j in range(128):
        v = (LN2 * j / 128).exp()
        hi = float(v)
        lo = float(v - Decimal(hi))
        lines.append(f"  {hi.hex()}, {lo.hex()},")
    lines.append("};")
    c = LN2 / 128
    m, e = math.frexp(float(c))
    hi = math.ldexp(math.floor(m * 2 ** 36 + 0.5), e - 36)  # k * hi exact for |k| < 2^17
    lo = float(c - Decimal(hi))
    inv = float(Decimal(128) / LN2)
    lines += [f"#define PF_EXP_INVLN2N {inv.hex()}", f"#define PF_EXP_LN2N_HI {hi.hex()}",
              f"#define PF_EXP_LN2N_LO {lo.hex()}"]
    # the mixture fast path (pf_qfast_terms): 2^(j/1024) rounded to nearest,
    # one double per entry (1.1e-16 relative), and ln2/1024 as one double
    # (k * ln2/1024 by a single FMA: |k| < 2^17, error < 4e-20 |k|)
    lines += ["// 2^(j/1024) = RN(2^(j/1024)) (pf_qfast_terms)", "__device__ const __align__(16) double pf_exp2_1024_g[1024] = {"]
    for j in range(1024):
        lines.append(f"  {float((LN2 * j / 1024).exp()).hex()},")
    lines.append("};")
    lines += [f"#define PF_Q_INVLN2N {float(Decimal(1024) / LN2).hex()}",
              f"#define PF_Q_LN2N {float(LN2 / 1024).hex()}"]
    with open(OUT, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    _ = struct


if __name__ == "__main__":
    main()
