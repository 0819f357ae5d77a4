#!/bin/bash
# FFMA (DG_VARIANT_FFMA): default library over N=1..9, tuning builds
# (paper_1211_0582_b200/tune/libdg_n<N>_*.so) on their order, and (NCU=1) one
# ncu --set full capture of the N=${NCU_N:-4} FFMA stage kernel on C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/variant_sweep.py --cases f32-ffma-tiled --orders ${ORDERS:-1,2,3,4,5,6,7,8,9} | sed "s/^/default /" >> gpurun_out/ffma_tune.jsonl 2>> gpurun_out/ffma_tune.err
for lib in paper_1211_0582_b200/tune/libdg_n*.so; do
  [ -e "$lib" ] || continue
  n=$(basename $lib | sed -E 's/libdg_n([0-9]+)_.*/\1/')
  DG_LIB=$lib timeout 300 python tools/variant_sweep.py --orders $n --cases f32-ffma-tiled | sed "s/^/$(basename $lib) /" >> gpurun_out/ffma_tune.jsonl 2>> gpurun_out/ffma_tune.err
done
if [ "${NCU:-0}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dg_stage_ffma -s 25 -c 1 -o gpurun_out/ffma_n${NCU_N:-4} \
   python bench.py --no-sweep --no-cpu-baseline --no-large --steps 2 --warmup 3 --precision 4 --variant 6 --order ${NCU_N:-4} > gpurun_out/ncu_ffma.txt 2>&1
fi
cat gpurun_out/ffma_tune.jsonl
echo done
