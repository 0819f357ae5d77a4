#!/bin/bash
# TC kernel role knock-outs (DG_TC_X builds, paper_1211_0582_b200/tune/libdg_tc*.so; results are
# wrong by design, timing only): which role bounds the stage at N = 1, 4, 9 (C2).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/tcx
O=gpurun_out/tcx/tc_knockout.jsonl
timeout 300 python tools/variant_sweep.py --steps 10 --orders 1,4,6,9 --cases f32-tc-tcgen05 | sed "s/^/{\"lib\": \"default\", \"row\": /; s/$/}/" >> $O 2>> gpurun_out/tcx/err.txt
for lib in paper_1211_0582_b200/tune/libdg_tc*.so; do
  name=$(basename $lib .so)
  DG_LIB=$lib timeout 300 python tools/variant_sweep.py --steps 10 --orders 1,4,6,9 --cases f32-tc-tcgen05 | sed "s/^/{\"lib\": \"$name\", \"row\": /; s/$/}/" >> $O 2>> gpurun_out/tcx/err.txt
done
echo done
