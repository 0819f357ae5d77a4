#!/bin/bash
# Round-2 measurement set: HBM-resident order sweep on C4 (AUTO kernels) with ncu DRAM bytes per
# stage launch, element-order study, ncu --set full of the tcgen05 stage kernel, NEXT-4 variant
# sweep, cuBLAS yardstick.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/c4sweep.jsonl gpurun_out/order.jsonl gpurun_out/variant_sweep.jsonl
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
for n in 15 56; do for p in 8 4; do
  for opt in "" "--shuffle-seed 1" "--shuffle-seed 1 --reorder"; do
    timeout 600 python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --mesh-n $n --precision $p --steps 10 --warmup 3 $opt >> gpurun_out/order.jsonl 2>> gpurun_out/order.err
  done
done; done
for n in 4 6 9; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dg_stage_tc -s 16 -c 1 \
    -o gpurun_out/r2_ncu_tc_N$n -f python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --steps 1 --warmup 3 \
    --precision 4 --order $n > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dg_stage_tc -s 16 -c 1 \
  -o gpurun_out/r2_ncu_tc_N4_C4 -f python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --steps 1 --warmup 3 \
  --precision 4 --order 4 --mesh-n 56 > /dev/null 2>&1
timeout 1200 python tools/variant_sweep.py > gpurun_out/variant_sweep.jsonl 2> gpurun_out/variant_sweep.err
timeout 600 python tools/cublas_yardstick.py > gpurun_out/cublas_yardstick.jsonl 2> gpurun_out/cublas_yardstick.err
echo done
