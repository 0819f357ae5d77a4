#!/bin/bash
# NEXT-4: variant x order sweep (default library) + FP64 WS tile-size sweep (tune builds), C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python tools/variant_sweep.py > gpurun_out/variant_sweep.jsonl 2> gpurun_out/variant_sweep.err
for lib in paper_1211_0582_b200/tune/libdg_n*_e*s*.so; do
  n=$(basename $lib | sed -E 's/libdg_n([0-9]+)_.*/\1/')
  DG_LIB=$lib timeout 300 python tools/variant_sweep.py --orders $n --cases f64-ws-dmma >> gpurun_out/tile_sweep.jsonl 2>> gpurun_out/tile_sweep.err
done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
