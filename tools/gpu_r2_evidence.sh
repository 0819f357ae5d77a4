#!/bin/bash
# Round-2 evidence set (one gpurun call):
#  1. HBM-resident order sweep on the C4 mesh (Kuhn n=56, K = 1 053 696), AUTO kernels, N = 1..9 x {FP64, FP32}:
#     bench line + one ncu metrics pass over ONE WHOLE LSERK4 step (5 stage launches: stage 0 does not read
#     the residual, stages 1..4 do) with DRAM bytes, pipe utilisation and executed-instruction counters
#     (SURVEY §8d ncu protocol: executed flops vs the F(N) model, padding and 3xTF32 multiplicity)
#  2. ncu --set full of the tcgen05 stage kernel at N = 4, 6, 9 (C2) and N = 4 (C4), FP64 WS N = 4 (C2)
#  3. element-order study (natural / shuffled / shuffled + Morton) on C2 and C4, N = 4 and N = 1
#  4. NEXT-4 variant x order sweep (C2), cuBLAS yardstick
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/ev
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
M=$M,dram__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tc.sum
M=$M,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum
M=$M,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum
B="python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e"
rm -f gpurun_out/ev/c4sweep.jsonl
for p in 8 4; do
  for n in 1 2 3 4 5 6 7 8 9; do
    timeout 600 $B --mesh-n 56 --steps 5 --warmup 3 --precision $p --order $n >> gpurun_out/ev/c4sweep.jsonl 2>> gpurun_out/ev/c4sweep.err
    timeout 900 ncu --metrics $M --clock-control none -k regex:dg_stage -s 15 -c 5 --csv \
      $B --mesh-n 56 --steps 1 --warmup 3 --precision $p --order $n > gpurun_out/ev/c4ncu_p${p}_N${n}.csv 2>&1
  done
done
for n in 4 6 9; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dg_stage_tc -s 16 -c 1 \
    -o gpurun_out/ev/r2_ncu_full_tc_N${n}_C2 -f $B --steps 1 --warmup 3 --precision 4 --order $n > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage_tc -s 16 -c 1 \
  -o gpurun_out/ev/r2_ncu_full_tc_N4_C4 -f $B --steps 1 --warmup 3 --precision 4 --order 4 --mesh-n 56 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dg_stage_ws -s 16 -c 1 \
  -o gpurun_out/ev/r2_ncu_full_ws_N4_f64_C2 -f $B --steps 1 --warmup 3 --precision 8 --order 4 > /dev/null 2>&1
rm -f gpurun_out/ev/order.jsonl
for n in 15 56; do for p in 8 4; do for N in 4 1; do
  for opt in "" "--shuffle-seed 1" "--shuffle-seed 1 --reorder"; do
    timeout 600 $B --mesh-n $n --precision $p --order $N --steps 10 --warmup 3 $opt >> gpurun_out/ev/order.jsonl 2>> gpurun_out/ev/order.err
  done
done; done; done
timeout 1500 python tools/variant_sweep.py > gpurun_out/ev/variant_sweep.jsonl 2> gpurun_out/ev/variant_sweep.err
timeout 600 python tools/cublas_yardstick.py > gpurun_out/ev/cublas_yardstick.jsonl 2> gpurun_out/ev/cublas_yardstick.err
echo done
