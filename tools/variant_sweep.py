#!/usr/bin/env python
"""NEXT-4: variant x order sweep on the bench config C2 (Kuhn n=15,
K=20250), the B200 analogue of the paper's tuning study (fig:tuning-study,
PAPER.md:1151-1167).  One JSON line per (precision, variant, N): ms per LSERK4 step,
roofline fraction.  Kernels: FP64 BASIC (DFMA), MMA (DMMA, cp.async), MMA_WS (DMMA,
TMA warp-specialized); FP32 BASIC (FFMA), MMA_WS (3xTF32 HMMA), TC (tcgen05 3xTF32),
FFMA (register-tiled FFMA in the WS pipeline).

Usage: python tools/variant_sweep.py [--orders 1,2,...] [--steps 10]
       DG_LIB=paper_1211_0582_b200/tune/libdg_X.so python tools/variant_sweep.py ...  (tile sweep)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

CASES = [(8, 1, "f64-basic-dfma"), (8, 2, "f64-mma-dmma"), (8, 3, "f64-ws-dmma"), (8, 6, "f64-ffma-tiled"),
         (4, 1, "f32-basic-ffma"), (4, 3, "f32-ws-3xtf32"), (4, 4, "f32-tc-tcgen05"),
         (4, 6, "f32-ffma-tiled")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="1,2,3,4,5,6,7,8,9")
    ap.add_argument("--cases", default="")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--mesh-n", type=int, default=15)
    a = ap.parse_args()
    import torch
    stream = torch.cuda.Stream()
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    peaks = bench.load_peaks()
    args = argparse.Namespace(mesh_n=a.mesh_n, steps=a.steps, warmup=3, shuffle_seed=None, reorder=False,
                              variant=0, system=0)
    tag = os.path.basename(os.environ.get("DG_LIB", "libdg.so"))
    for prec, var, name in CASES:
        if a.cases and name not in a.cases.split(","):
            continue
        for N in [int(x) for x in a.orders.split(",")]:
            args.variant = var
            r = bench.run_dg(args, N, prec, 0, 1, 0, None, stream, flush, None, peaks)
            print(json.dumps({"lib": tag, "case": name, "N": N, "ms_per_step": r["ms_per_step"],
                              "gdof_s": round(r["dof_updates_per_s"] / 1e9, 3),
                              "bound": r["roofline"]["bound"], "frac": r["roofline"]["frac"]}), flush=True)


if __name__ == "__main__":
    main()
