#!/bin/bash
# C4-size (HBM-resident) measurements + FP32 ncu capture + convergence test.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "convergence" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for cfg in "8 1" "8 2" "8 4" "8 6" "4 4" "4 8"; do
  set -- $cfg
  timeout 600 python bench.py --no-sweep --no-cpu-baseline --mesh-n 56 --steps 10 --warmup 3 --precision $1 --order $2 >> gpurun_out/c4.jsonl 2>> gpurun_out/c4.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 1 -o gpurun_out/prof_f32 \
   python bench.py --no-sweep --no-cpu-baseline --steps 2 --warmup 3 --order 4 --precision 4 > gpurun_out/ncu_f32.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 1 -o gpurun_out/prof_c4 \
   python bench.py --no-sweep --no-cpu-baseline --steps 2 --warmup 3 --order 4 --precision 8 --mesh-n 56 > gpurun_out/ncu_c4.txt 2>&1
echo done
