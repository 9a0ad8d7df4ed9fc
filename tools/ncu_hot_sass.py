#!/usr/bin/env python
"""Hottest SASS instructions (warp stall samples) of an `ncu --page source --csv` export, with the dominant
stall reason of each: tools/ncu_hot_sass.py <source.csv> [top N] [context lines]"""
import csv
import sys

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = list(csv.reader(open(path)))
hdr = rows[1]
body = rows[2:]
i_src, i_samp = hdr.index("Source"), hdr.index("# Samples")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
total = sum(int(r[i_samp] or 0) for r in body)
order = sorted(range(len(body)), key=lambda k: -int(body[k][i_samp] or 0))[:top]
for k in sorted(order):
    r = body[k]
    n = int(r[i_samp] or 0)
    why = sorted(((int(r[c] or 0), hdr[c]) for c in stall_cols), reverse=True)[:2]
    for j in range(max(0, k - ctx), k):
        print(f"        {j:5d}  {body[j][i_src].strip()}")
    print(f"{100 * n / total:6.2f}% {k:5d}  {r[i_src].strip():70s} {why[0][1]}={why[0][0]} {why[1][1]}={why[1][0]}")
