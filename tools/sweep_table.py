#!/usr/bin/env python
"""Render the NEXT-4 variant x order table from tools/variant_sweep.py output.
Usage: python tools/sweep_table.py profiles/r1_variant_sweep.jsonl"""
import json
import sys

CASES = ["f64-basic-dfma", "f64-mma-dmma", "f64-ws-dmma", "f64-ffma-tiled",
         "f32-basic-ffma", "f32-ws-3xtf32", "f32-tc-tcgen05", "f32-ffma-tiled"]
HDR = ["FP64 BASIC (DFMA)", "FP64 MMA (DMMA)", "FP64 WS (DMMA)", "FP64 FFMA (tiled DFMA)",
       "FP32 BASIC (FFMA)", "FP32 WS (3×TF32 HMMA)", "FP32 TC (tcgen05)", "FP32 FFMA (tiled FFMA)"]


def main(path):
    d = {}
    for line in open(path):
        if line.strip().startswith("{"):
            r = json.loads(line)
            d[(r["case"], r["N"])] = r
    print("| N | " + " | ".join(HDR) + " |")
    print("|---" * (len(HDR) + 1) + "|")
    for N in range(1, 10):
        cells = []
        for prec in ("f64", "f32"):
            cs = [c for c in CASES if c.startswith(prec)]
            have = [(d[(c, N)]["ms_per_step"], c) for c in cs if (c, N) in d]
            best = min(have)[1] if have else None
            for c in cs:
                if (c, N) not in d:
                    cells.append("—")
                    continue
                r = d[(c, N)]
                t = f"{r['ms_per_step']:.4f} ({r['frac']:.2f})"
                cells.append(f"**{t}**" if c == best else t)
        print(f"| {N} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
