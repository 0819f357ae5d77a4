#!/bin/bash
# DRAM traffic of the stage kernel (ncu --set full): C2 and C4, FP64 and FP32 at N=4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "morton or energy_conserved" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for cfg in "8 15" "4 15" "8 56" "4 56"; do
  set -- $cfg
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 1 -o gpurun_out/full_p$1_n$2 \
     python bench.py --no-sweep --no-large --no-cpu-baseline --steps 2 --warmup 3 --order 4 --precision $1 --mesh-n $2 > gpurun_out/ncu_p$1_n$2.txt 2>&1
done
echo done
