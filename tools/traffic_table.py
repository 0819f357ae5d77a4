#!/usr/bin/env python
"""profiles/r2_traffic.json: DRAM bytes per stage launch (dram__bytes_read.sum + dram__bytes_write.sum) of the AUTO
stage kernels, keyed precision:variant:N:K like round 1's r1_traffic.json (variant 0 = AUTO), from
  * ncu --set full captures of one stage-1 launch (it reads the residual): <src>/r2_ncu_full_{ws_N4_f64_C2,ws_N4_f64_C4,tc_N4_C2}
  * the C4 order sweep's metrics pass over one whole step (<src>/c4ncu_p*_N*.csv): the mean of stages 1..4.
Usage: python tools/traffic_table.py <src dir>"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from c4_summary import ncu_launches  # noqa: E402


def full_capture(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    r = rows[2]
    u = rows[1]
    def val(k):
        x = float(r[hdr.index(k)].replace(",", ""))
        unit = u[hdr.index(k)]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return {"kernel": r[hdr.index("Kernel Name")][:60], "read": val("dram__bytes_read.sum"),
            "write": val("dram__bytes_write.sum")}


def main(src):
    import bench
    out = {"note": "DRAM bytes per stage launch of the AUTO kernel; stage-1 launches (residual read) from ncu --set full, "
                   "and the mean of stages 1..4 from the C4 sweep metrics pass (tools/gpu_r2_final.sh, tools/traffic_table.py)"}
    for name, key in (("r2_ncu_full_ws_N4_f64_C2", "f64:0:4:K20250"), ("r2_ncu_full_ws_N4_f64_C4", "f64:0:4:K1053696"),
                      ("r2_ncu_full_tc_N4_C2", "f32:0:4:K20250")):
        p = os.path.join(src, name + ".ncu-rep")
        if os.path.exists(p):
            m = full_capture(p)
            out[key] = {"kernel": m["kernel"], "dram_bytes": m["read"] + m["write"], "read": m["read"], "write": m["write"],
                        "source": f"profiles/{name}.txt"}
    for prec in (8, 4):
        for N in range(1, 10):
            L = ncu_launches(os.path.join(src, f"c4ncu_p{prec}_N{N}.csv"))
            st = [L[i] for i in sorted(L) if i % 5 != 0]
            if not st:
                continue
            d = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in st) / len(st)
            key = f"{'f64' if prec == 8 else 'f32'}:0:{N}:K1053696"
            if key not in out:
                K = 1053696
                out[key] = {"kernel": st[0]["kernel"], "dram_bytes": d,
                            "algorithmic": bench.bytes_per_elem_stage(N, prec) * K, "source": "C4 sweep, stages 1..4"}
    with open(os.path.join(ROOT, "profiles", "r2_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1)[:2000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "fin"))
