#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from `ncu -i rep --page source --csv --print-source sass`.
Usage: ncu_sass_hot.py sass.csv [topN]   (prints address, samples, instruction, and a per-opcode total)"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ismp] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for s, a, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {a}  {src}")
ops = collections.Counter()
for s, a, src in data:
    ops[src.split()[0] if src.split() else "?"] += s
print("--- by opcode")
for op, s in ops.most_common(15):
    print(f"{100 * s / tot:5.1f}%  {op}")
