#!/bin/bash
# element-order study: natural vs shuffled vs shuffled+Morton, C2 and C4, N=4 FP64 and FP32
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "morton or energy_conserved" 2>&1 | tail -3 > gpurun_out/order_tests.txt
python bench.py > gpurun_out/order_default.json 2> gpurun_out/order_default.err
for n in 15 56; do for p in 8 4; do
  for opt in "" "--shuffle-seed 1" "--shuffle-seed 1 --reorder" "--reorder"; do
    tag=$(echo "n$n p$p $opt" | tr ' ' '_' | tr -s '_')
    python bench.py --no-sweep --no-large --no-cpu-baseline --mesh-n $n --precision $p --steps 10 --warmup 3 $opt > gpurun_out/order_$tag.json 2>&1
  done
done; done
