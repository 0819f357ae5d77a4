#!/bin/bash
# FP64 WS tuning builds (paper_1211_0582_b200/tune/libdg_n<N>_*.so) against the default library, same box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for lib in paper_1211_0582_b200/libdg.so paper_1211_0582_b200/tune/libdg_n*.so; do
  n=$(basename $lib | sed -E 's/libdg_n([0-9]+)_.*/\1/')
  [ "$n" = "libdg.so" ] && n=${ORDERS:-1,2,3,4,5,6,7,8,9}
  DG_LIB=$lib timeout 600 python tools/variant_sweep.py --orders $n --cases ${CASES:-f64-ws-dmma,f64-mma-dmma} >> gpurun_out/tile_sweep.jsonl 2>> gpurun_out/tile_sweep.err
done
echo done
