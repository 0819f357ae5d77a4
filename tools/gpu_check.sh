#!/bin/bash
# One gpurun call: smoke, GPU parity tests, ALU peaks, bench, ncu launch list + full capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
[ -x tools/alu_peaks ] && timeout 120 ./tools/alu_peaks > gpurun_out/alu_peaks.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
if [ -z "${SKIP_BENCH}" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --no-sweep --no-cpu-baseline --steps 4 --warmup 3 > gpurun_out/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 2 -o gpurun_out/prof_stage \
   python bench.py --no-sweep --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_full_run.txt 2>&1
fi
echo done
