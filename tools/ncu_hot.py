#!/usr/bin/env python3
"""Top stall-sampled SASS instructions from `ncu -i rep --page source --csv --print-source sass`.
  python tools/ncu_hot.py <source.csv> [n]"""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot = sum(f(r[si]) for r in data)
print("total samples", tot, "instructions", len(data))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for r in sorted(data, key=lambda r: -f(r[si]))[:n]:
    print(f"{f(r[si]) / tot * 100:5.1f}%  exec {r[ie]:>8}  {r[0][-5:]}  {r[1].strip()}")
