#!/usr/bin/env python
"""Print the headline and sweep of a bench.py JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "gflops", d.get("gflops"), "ms/step", d["ms_per_step"])
print("roofline", d.get("roofline"))
print("e2e", d.get("e2e"))
print("clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
print("cpu", d.get("cpu_baseline"))
for r in d.get("sweep", []):
    rf = r["roofline"]
    print(f'{r["precision"]} N={r["N"]} {r["ms_per_step"]:9.4f} ms  {r["dof_updates_per_s"]:.3g} DOF/s  '
          f'{r["gflops"]:8.0f} GF/s  {rf["bound"]} {rf["frac"]:.3f} of {rf["peak"]}')
if d.get("large"):
    r = d["large"]
    print("large", r.get("workload"), r["ms_per_step"], "ms", f'{r["dof_updates_per_s"]:.3g}', "DOF/s", r["roofline"])
