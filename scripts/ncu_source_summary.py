#!/usr/bin/env python
"""Per-opcode summary of an ncu source page (SASS): shared wavefronts and
warp instructions per update, stall-sample shares, and the overall stall
reasons.

    ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
    python scripts/ncu_source_summary.py src.csv UPDATES_PER_LAUNCH
"""
import csv
import sys
from collections import defaultdict


def main(path, updates):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def f(r, k):
        try:
            return float(r[ix[k]] or 0)
        except (KeyError, ValueError):
            return 0.0

    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {c: sum(f(r, c) for r in data) for c in stalls}
    T = sum(tot.values()) or 1.0
    print(f"kernel: {rows[0][1][:100]}")
    print("stall reasons (share of warp samples):")
    for c, v in sorted(tot.items(), key=lambda x: -x[1]):
        if v > 0:
            print(f"  {c:24s} {100 * v / T:5.1f} %")
    byop = defaultdict(lambda: [0.0, 0.0, 0.0])
    for r in data:
        toks = r[ix["Source"]].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        byop[op][0] += f(r, "L1 Wavefronts Shared")
        byop[op][1] += f(r, "Instructions Executed")
        byop[op][2] += f(r, "Warp Stall Sampling (All Samples)")
    S = sum(v[2] for v in byop.values()) or 1.0
    print(f"per update ({updates:.0f} updates): opcode, shared wavefronts, warp instructions, stall samples")
    for op, (w, n, s) in sorted(byop.items(), key=lambda x: -x[1][2])[:24]:
        print(f"  {op:10s} {w / updates:7.3f} {n / updates:7.3f} {100 * s / S:5.1f} %")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
