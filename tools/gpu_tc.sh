#!/bin/bash
# TC kernel: parity + timing check, tcgen05 peak shapes, ncu --set full of the TC stage kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
./tools/tcgen05_peak > gpurun_out/tcgen05_peak2.json 2>&1
timeout 600 python tools/tc_check.py ${TC_ORDERS:+--orders $TC_ORDERS} > gpurun_out/tc_check.jsonl 2> gpurun_out/tc_check.err
for n in ${NCU_ORDERS:-4 8}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dg_stage_tc -s 16 -c 1 \
    -o gpurun_out/tc_N$n -f python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e --steps 1 --warmup 3 \
    --precision 4 --order $n --variant 4 > gpurun_out/tc_ncu_N$n.txt 2>&1
done
echo done
