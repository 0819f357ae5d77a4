#!/bin/bash
# Round 2: boundary-first single-launch multi-rank stages.  Stream-memop graph probe, tcgen05
# contention probe, loopback parity (P = 2, 3, 4 all variants; P = 8 at C4 per-rank size), the
# loopback overhead timing, then the whole GPU suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/mg
timeout 120 ./tools/memop_graph_probe > gpurun_out/mg/memop_graph_probe.json 2>&1; echo "rc=$?" >> gpurun_out/mg/memop_graph_probe.json
timeout 120 ./tools/tcgen05_contention_probe > gpurun_out/mg/tcgen05_contention.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "partitioned or acoustics_alpha0" \
  > gpurun_out/mg/pytest_loopback.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/mg/pytest_loopback.txt
for a in "4 8" "2 8" "4 4" "7 4"; do
  timeout 600 python tools/loopback_timing.py $a >> gpurun_out/mg/loopback_timing.jsonl 2>> gpurun_out/mg/loopback_timing.err
done
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/mg/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/mg/pytest_gpu.txt
echo done
