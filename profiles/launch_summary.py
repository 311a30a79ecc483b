"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.

usage: python profiles/launch_summary.py launches.csv [n_step_executions]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki][:80]
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "ns" else v * 1e3 if r[ui] == "ms" else v
    agg[name] = agg.get(name, 0.0) + v
    cnt[name] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    if v / tot < 0.002:
        continue
    print(f"{v / div:10.1f} us  {100 * v / tot:5.1f}%  x{cnt[k] / div:4.1f}  {k}")
print(f"total {tot / div:.1f} us per step-execution (÷{div:g})")
