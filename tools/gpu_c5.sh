#!/bin/bash
# configs[4] (C5: N = 7..9 FP32, tensor-core vs FFMA differentiation/lift) on one GPU: the per-rank proxy of the
# 8-GPU run (Kuhn n = 36, K = 279 936 = C5 / 8) for N = 7, 8, 9, and the whole C5 mesh (n = 72, K = 2 239 488) at
# N = 7 (1.6e9 words per state copy: fits one rank; N = 8, 9 exceed the int32 reach and need >= 2 ranks).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/c5
B="python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --precision 4 --steps 3 --warmup 3"
rm -f gpurun_out/c5/c5.jsonl
for N in 7 8 9; do for v in 4 6 3; do
  timeout 900 $B --mesh-n 36 --order $N --variant $v >> gpurun_out/c5/c5.jsonl 2>> gpurun_out/c5/c5.err
done; done
for v in 4 6; do
  timeout 1200 $B --mesh-n 72 --order 7 --variant $v >> gpurun_out/c5/c5.jsonl 2>> gpurun_out/c5/c5.err
done
echo done
