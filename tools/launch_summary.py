#!/usr/bin/env python
"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum).
usage: python tools/launch_summary.py <csv> [steps]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = None
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:90]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit == "msecond" else v
        tot[name] += v
        cnt[name] += 1
all_us = sum(tot.values())
print(f"total {all_us:.1f} us over {steps:g} steps = {all_us / steps:.1f} us/step")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {v / steps:8.2f} us/step  {cnt[k] / steps:6.2f} launches/step  {100 * v / all_us:5.1f}%  {k}")
