cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "ffma" > gpurun_out/pytest_ffma.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ffma.txt
timeout 600 python tools/variant_sweep.py --cases f32-ffma-tiled,f32-ws-3xtf32 > gpurun_out/ffma_sweep.jsonl 2> gpurun_out/ffma_sweep.err
tail -3 gpurun_out/pytest_ffma.txt; cat gpurun_out/ffma_sweep.jsonl; tail -5 gpurun_out/ffma_sweep.err
