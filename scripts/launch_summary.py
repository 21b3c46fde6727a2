#!/usr/bin/env python
"""Kernel shares of an ncu launch list (--metrics gpu__time_duration.sum
--clock-control none --csv): launches, total ms and share per kernel.

  python scripts/launch_summary.py LAUNCHES.csv [HEADER TEXT]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
cols = rows[hdr]
ki, mi, vi, ui = (cols.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot, cnt = defaultdict(float), defaultdict(int)
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    cnt[name] += 1
all_ms = sum(tot.values())
if len(sys.argv) > 2:
    print(" ".join(sys.argv[2:]))
print(f"{'kernel':62s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda x: -tot[x]):
    print(f"{k[:62]:62s} {cnt[k]:8d} {tot[k]:10.2f} {100 * tot[k] / all_ms:6.1f}%")
