#!/usr/bin/env python
"""Quick TC-kernel check on the GPU: RHS and 2-step parity against the oracle on a
shuffled/rotated/jittered K=162 mesh for N = 1..9, then ms per LSERK4 step on C2 for
TC vs the current AUTO kernel.  One JSON line per result."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import dg_inputs as di  # noqa: E402
import oracle  # noqa: E402
from paper_1211_0582_b200.dg import Solver  # noqa: E402


def relerr(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="1,2,3,4,5,6,7,8,9")
    ap.add_argument("--no-time", action="store_true")
    ap.add_argument("--variants", default="4,0")
    a = ap.parse_args()
    orders = [int(x) for x in a.orders.split(",")]
    VX, E = di.kuhn_box(3)
    E, _ = di.shuffle_elements(E, 1)
    E = di.rotate_local_vertices(E, 2)
    VX = di.jitter_interior(VX, 3, 3)
    for N in orders:
        st = oracle.Setup(VX, E, N)
        U = di.random_fields(st.K, N, seed=0)
        s = Solver(N, precision=4, variant=4)
        s.mesh_upload(VX, E)
        s.fields_upload(U)
        r = relerr(s.rhs(), oracle.rhs(st, U))
        dt = di.dt_rule(VX, E, N)
        s.lserk_step(dt, 2)
        r2 = relerr(s.fields_download(), oracle.lserk4(st, U, dt, 2))
        s.close()
        print(json.dumps({"check": "parity", "N": N, "rhs_relerr": r, "step2_relerr": r2,
                          "ok": r < 2e-5 and r2 < 1e-4}), flush=True)
    if a.no_time:
        return
    import torch
    stream = torch.cuda.Stream()
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    peaks = bench.load_peaks()
    args = argparse.Namespace(mesh_n=15, steps=10, warmup=3, shuffle_seed=None, reorder=False, variant=0, system=0)
    for N in orders:
        for v in [int(x) for x in a.variants.split(",")]:
            args.variant = v
            r = bench.run_dg(args, N, 4, 0, 1, 0, None, stream, flush, None, peaks)
            print(json.dumps({"check": "time", "N": N, "variant": v, "kernel": r["kernel"],
                              "ms_per_step": r["ms_per_step"]}), flush=True)


if __name__ == "__main__":
    main()
