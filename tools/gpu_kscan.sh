#!/bin/bash
# Stage time vs mesh size (fixed per-stage cost + per-element cost), AUTO kernels, FP64 and FP32.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for n in 6 10 15 24 32; do
  timeout 300 python tools/variant_sweep.py --mesh-n $n --orders ${ORDERS:-1,2,3,4} --cases f64-ws-dmma,f64-ffma-tiled,f32-ffma-tiled | sed "s/^/{\"mesh_n\": $n, \"r\": /; s/\$/}/" >> gpurun_out/kscan.jsonl
done
cat gpurun_out/kscan.jsonl
