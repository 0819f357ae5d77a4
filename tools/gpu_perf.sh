#!/bin/bash
# Perf iteration: quick parity subset, bench sweep, ncu capture of the N=${NCU_N:-4} stage kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-many_tiles and f64-mma}" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -z "${SKIP_NCU}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dg_stage -s 25 -c 1 -o gpurun_out/prof_stage \
   python bench.py --no-sweep --no-cpu-baseline --steps 2 --warmup 3 --order ${NCU_N:-4} --precision ${NCU_P:-8} > gpurun_out/ncu_full_run.txt 2>&1
fi
echo done
