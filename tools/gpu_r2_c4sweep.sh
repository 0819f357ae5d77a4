#!/bin/bash
# Round 2: tcgen05 kind::tf32 peak; HBM-resident order sweep on the C4 mesh (Kuhn n=56,
# K = 1 053 696) for N = 1..9 x {FP64, FP32} with the AUTO kernels, and ncu DRAM bytes per
# stage launch for each (precision, order).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
./tools/tcgen05_peak > gpurun_out/tcgen05_peak.json 2>&1
for p in 8 4; do
  for n in 1 2 3 4 5 6 7 8 9; do
    timeout 600 python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --mesh-n 56 --steps 5 --warmup 3 \
      --precision $p --order $n >> gpurun_out/c4sweep.jsonl 2>> gpurun_out/c4sweep.err
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:dg_stage -s 16 -c 1 --csv \
      python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --mesh-n 56 --steps 1 --warmup 3 \
      --precision $p --order $n > gpurun_out/c4ncu_p${p}_N${n}.csv 2>&1
  done
done
echo done
