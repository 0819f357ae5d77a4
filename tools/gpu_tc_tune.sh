#!/bin/bash
# TC kernel ring / batch tuning builds (paper_1211_0582_b200/tune/libdg_*.so) against the default, C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/tct
O=gpurun_out/tct/tc_tune.jsonl
rm -f $O
for r in 1 2; do
timeout 300 python tools/variant_sweep.py --steps 20 --orders ${ORDERS:-3,4,5,6,7,9} --cases f32-tc-tcgen05 | sed "s/^/{\"lib\": \"default\", \"row\": /; s/$/}/" >> $O 2>> gpurun_out/tct/err.txt
for lib in paper_1211_0582_b200/tune/libdg_*.so; do
  name=$(basename $lib .so)
  DG_LIB=$lib timeout 300 python tools/variant_sweep.py --steps 20 --orders ${ORDERS:-3,4,5,6,7,9} --cases f32-tc-tcgen05 | sed "s/^/{\"lib\": \"$name\", \"row\": /; s/$/}/" >> $O 2>> gpurun_out/tct/err.txt
done
done
echo done
