cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
rm -f gpurun_out/ffma_tune.jsonl
ORDERS=4,5 bash tools/gpu_ffma_tune.sh
timeout 300 python tools/variant_sweep.py --orders 4,5 --cases f32-ws-3xtf32 >> gpurun_out/ffma_tune.jsonl
cat gpurun_out/ffma_tune.jsonl
