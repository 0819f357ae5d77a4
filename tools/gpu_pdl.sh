#!/bin/bash
# PDL A/B (DG_PDL=0/1) on the variant sweep + a parity subset with PDL on.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "many_tiles or bench_mesh or lserk_steps or partitioned" > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for v in 0 1; do
  DG_PDL=$v timeout 900 python tools/variant_sweep.py --cases f64-mma-dmma,f64-ws-dmma,f32-ws-3xtf32,f32-tc-tcgen05 | sed "s/^{/{\"pdl\": $v, /" >> gpurun_out/pdl_sweep.jsonl 2>> gpurun_out/pdl_sweep.err
done
echo done
