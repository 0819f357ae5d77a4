#!/usr/bin/env python
"""External yardstick (bench-only; never linked into libdg): cuBLAS GEMMs of the
two contraction shapes of one stage, as the paper frames them ("fields in
aggregate as a matrix"):  volume (3Np x Np) . (Np x 6K)  and  lift (Np x 4Nfp) . (4Nfp x 6K),
through torch.matmul (cuBLAS), FP64 and FP32 (allow_tf32 off: FP32 accuracy) and TF32
(allow_tf32 on: 1xTF32, NOT accurate enough for the 1e-4 FP32 tolerance; context only).
Prints one JSON line per (precision, N, mesh): ms per stage for the two GEMMs and their
TFLOP/s, next to the whole fused stage (all of a1..a5) from the bench for comparison."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dg_inputs as di  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    orders = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,5,6,7,8,9").split(",")]
    meshes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "15,56").split(",")]
    for n in meshes:
        K = 6 * n ** 3
        for N in orders:
            Np, Nfp = di.np_of(N), di.nfp_of(N)
            for prec, tf32 in (("f64", False), ("f32", False), ("tf32", True)):
                dt = torch.float64 if prec == "f64" else torch.float32
                torch.backends.cuda.matmul.allow_tf32 = tf32
                cols = 6 * K
                if cols * max(Np, 4 * Nfp) * (8 if dt == torch.float64 else 4) > 24e9:
                    continue
                A = torch.randn(3 * Np, Np, device="cuda", dtype=dt)
                L = torch.randn(Np, 4 * Nfp, device="cuda", dtype=dt)
                U = torch.randn(Np, cols, device="cuda", dtype=dt)
                F = torch.randn(4 * Nfp, cols, device="cuda", dtype=dt)
                tv = timeit(lambda: A @ U)
                tl = timeit(lambda: L @ F)
                fv, fl = 2.0 * 3 * Np * Np * cols, 2.0 * Np * 4 * Nfp * cols
                print(json.dumps({"mesh_n": n, "K": K, "N": N, "precision": prec, "volume_ms": round(tv, 4),
                                  "lift_ms": round(tl, 4), "volume_tflops": round(fv / tv / 1e9, 2),
                                  "lift_tflops": round(fl / tl / 1e9, 2),
                                  "gemms_ms_per_stage": round(tv + tl, 4),
                                  "gemms_ms_per_step": round(5 * (tv + tl), 4)}), flush=True)
                del A, L, U, F
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
