#!/usr/bin/env python
"""Summarise the HBM-resident order sweep on the C4 mesh (tools/gpu_r2_c4sweep.sh):
bench lines (gpurun_out/c4sweep.jsonl) + per-launch ncu DRAM bytes of one stage launch
(gpurun_out/c4ncu_p{8,4}_N{n}.csv) against the algorithmic B(N) K.
Writes profiles/<tag>_c4_sweep.json and prints a markdown table."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import dg_inputs as di  # noqa: E402


def ncu_metrics(path):
    out = {}
    if not os.path.exists(path):
        return out
    with open(path) as fh:
        rows = [r for r in csv.reader(fh) if len(r) > 14]
    for r in rows:
        if r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "lts__t_sector_hit_rate.pct"):
            try:
                out[r[12]] = float(r[14].replace(",", ""))
            except ValueError:
                pass
        out["kernel"] = r[4]
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    rows = []
    for line in open(os.path.join(src, "c4sweep.jsonl")):
        d = json.loads(line)
        c = d["config"]
        N, prec = c["order"], 8 if c["precision"] == "f64" else 4
        K = c["K_total"]
        m = ncu_metrics(os.path.join(src, f"c4ncu_p{prec}_N{N}.csv"))
        alg = bench.bytes_per_elem_stage(N, prec) * K
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        rows.append({"precision": c["precision"], "N": N, "K": K, "kernel": c["kernel"],
                     "ms_per_step": d["ms_per_step"], "gdof_s": round(d["value"] / 1e9, 3),
                     "roofline": d["roofline"], "ncu_kernel": m.get("kernel"),
                     "ncu_ms_per_launch": round(m.get("gpu__time_duration.sum", 0) / 1e6, 4),
                     "dram_bytes_per_launch": dram, "alg_bytes_per_launch": alg,
                     "dram_over_alg": round(dram / alg, 3) if dram else None,
                     "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct")})
    out = os.path.join(ROOT, "profiles", f"{tag}_c4_sweep.json")
    with open(out, "w") as fh:
        json.dump({"mesh": "C4: Kuhn n=56, K=1053696 (HBM-resident)", "rows": rows}, fh, indent=1)
    print("| prec | N | kernel | ms/step | G DOF/s | bound | frac | DRAM/launch (GB) | alg (GB) | DRAM/alg |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        rf = r["roofline"]
        print(f"| {r['precision']} | {r['N']} | {r['kernel']} | {r['ms_per_step']:.3f} | {r['gdof_s']:.2f} | "
              f"{rf['bound']} | {rf['frac']:.3f} | {r['dram_bytes_per_launch'] / 1e9:.3f} | "
              f"{r['alg_bytes_per_launch'] / 1e9:.3f} | {r['dram_over_alg']} |")


if __name__ == "__main__":
    main()
