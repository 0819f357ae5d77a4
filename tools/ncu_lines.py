#!/usr/bin/env python
"""Warp-stall samples per CUDA source line from an ncu report (cuda,sass source view; the kernel
must be built with -lineinfo).  Usage: ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, errors="replace").stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, rows = None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
        ismp = hdr.index("Warp Stall Sampling (All Samples)")
    elif fname and r[0].isdigit() and r[2] == "-":  # a CUDA line row (its SASS rows carry addresses)
        try:
            rows.append((int(r[ismp] or 0), fname, int(r[0]), r[1].strip()[:100]))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in rows) or 1
for s, f, l, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{l}  {src}")
