#!/bin/bash
# Round-2 final evidence (one gpurun call): smoke, GPU parity suite, bench line (+ reference arm),
# NEXT-4 variant sweep, ncu launch list of the bench command, ncu --set full of the headline stage
# kernel (C2 and C4, N = 4 FP64) and of the tcgen05 kernel (C2, N = 4), and the HBM-resident C4 order
# sweep with per-step ncu metrics (tools/c4_summary.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/fin
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1500 python tools/variant_sweep.py > $O/variant_sweep.jsonl 2> $O/variant_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --no-sweep --no-cpu-baseline --no-large --steps 4 --warmup 3 > $O/ncu_launch_run.txt 2>&1
B="python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 16 -c 1 -o $O/r2_ncu_full_ws_N4_f64_C2 -f \
   $B --steps 1 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 16 -c 1 -o $O/r2_ncu_full_ws_N4_f64_C4 -f \
   $B --steps 1 --warmup 3 --mesh-n 56 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 16 -c 1 -o $O/r2_ncu_full_tc_N4_C2 -f \
   $B --steps 1 --warmup 3 --precision 4 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
M=$M,dram__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tc.sum
M=$M,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum
M=$M,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum
rm -f $O/c4sweep.jsonl
for p in 8 4; do
  for n in 1 2 3 4 5 6 7 8 9; do
    timeout 600 $B --mesh-n 56 --steps 5 --warmup 3 --precision $p --order $n >> $O/c4sweep.jsonl 2>> $O/c4sweep.err
    timeout 900 ncu --metrics $M --clock-control none -k regex:dg_stage -s 15 -c 5 --csv \
      $B --mesh-n 56 --steps 1 --warmup 3 --precision $p --order $n > $O/c4ncu_p${p}_N${n}.csv 2>&1
  done
done
echo done
