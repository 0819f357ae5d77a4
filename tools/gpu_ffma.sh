#!/bin/bash
# FFMA variant check: GPU parity of the FFMA kernels (FP32 and FP64) and the C2 sweep of
# ${CASES:-f32-ffma-tiled,f64-ffma-tiled} against the tensor-core WS kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "ffma" > gpurun_out/pytest_ffma.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ffma.txt
timeout 900 python tools/variant_sweep.py --cases ${CASES:-f64-ffma-tiled,f64-ws-dmma} > gpurun_out/ffma_sweep.jsonl 2> gpurun_out/ffma_sweep.err
tail -3 gpurun_out/pytest_ffma.txt; cat gpurun_out/ffma_sweep.jsonl; tail -5 gpurun_out/ffma_sweep.err
