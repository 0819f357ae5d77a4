#!/bin/bash
# NEXT-3 acoustics: GPU parity (BASIC, FFMA and FP32 TC kernels) and C2 timing of the kernels, N=1..9, FP64/FP32.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "acoustic" > gpurun_out/pytest_acoustics.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_acoustics.txt
timeout 900 python - > gpurun_out/acoustics_sweep.jsonl 2> gpurun_out/acoustics_sweep.err <<'PY'
import argparse, json, sys
sys.path.insert(0, ".")
import torch, bench
stream = torch.cuda.Stream()
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
peaks = bench.load_peaks()
for var, name in ((6, "ffma"), (4, "tc"), (3, "ws")):
    for prec in ((8, 4) if var == 6 else (4,) if var == 4 else (8,)):
        for N in range(1, 10):
            a = argparse.Namespace(mesh_n=15, steps=10, warmup=3, shuffle_seed=None, reorder=False, variant=var, system=1)
            r = bench.run_dg(a, N, prec, 0, 1, 0, None, stream, flush, None, peaks)
            print(json.dumps({"case": f"acoustics-{'f64' if prec == 8 else 'f32'}-{name}", "N": N,
                              "ms_per_step": r["ms_per_step"], "frac": r["roofline"]["frac"],
                              "bound": r["roofline"]["bound"]}), flush=True)
PY
tail -2 gpurun_out/pytest_acoustics.txt; cat gpurun_out/acoustics_sweep.jsonl; tail -3 gpurun_out/acoustics_sweep.err
