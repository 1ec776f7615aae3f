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
             "__device__ const double pf_exp_tab_g[256] = {"]
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
    with open(OUT, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    _ = struct


if __name__ == "__main__":
    main()
