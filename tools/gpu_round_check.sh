#!/bin/bash
# One gpurun call for the round's evidence: smoke, GPU parity suite, bench (full JSON line),
# variant sweep, ncu launch list of the bench command, ncu --set full of the stage kernel at
# C2 and C4 (N=4 FP64).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1200 python tools/variant_sweep.py > gpurun_out/variant_sweep.jsonl 2> gpurun_out/variant_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --no-sweep --no-cpu-baseline --no-large --steps 4 --warmup 3 > gpurun_out/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 1 -o gpurun_out/full_c2 \
   python bench.py --no-sweep --no-cpu-baseline --no-large --steps 2 --warmup 3 > gpurun_out/ncu_full_c2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 1 -o gpurun_out/full_c4 \
   python bench.py --no-sweep --no-cpu-baseline --no-large --steps 2 --warmup 3 --mesh-n 56 > gpurun_out/ncu_full_c4.txt 2>&1
echo done
