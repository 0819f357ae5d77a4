#!/bin/bash
# Refresh after the last tuning commits: bench line, NEXT-4 variant sweep, C4 order sweep (both precisions,
# bench lines only; the ncu metrics of tools/gpu_r2_final.sh stand for the unchanged kernels).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/fin2
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 1500 python tools/variant_sweep.py > $O/variant_sweep.jsonl 2> $O/variant_sweep.err
B="python bench.py --no-sweep --no-large --no-cpu-baseline --no-e2e"
rm -f $O/c4sweep.jsonl
for p in 8 4; do for n in 1 2 3 4 5 6 7 8 9; do
  timeout 600 $B --mesh-n 56 --steps 5 --warmup 3 --precision $p --order $n >> $O/c4sweep.jsonl 2>> $O/c4sweep.err
done; done
echo done
