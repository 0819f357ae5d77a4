#!/bin/bash
# Low-order FFMA kernel (HBM-bound regime): ring depth / trace look-ahead / tile size tuning builds
# (paper_1211_0582_b200/tune/libdg_n<N>_*.so) against the default library on the HBM-resident C4 mesh
# and on C2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/lown
O=gpurun_out/lown/ffma_lown.jsonl
for mesh in 56 15; do
  timeout 600 python tools/variant_sweep.py --mesh-n $mesh --steps 5 --orders 1,2 --cases f32-ffma-tiled,f64-ffma-tiled | sed "s/^/{\"lib\": \"default\", \"mesh\": $mesh, \"row\": /; s/$/}/" >> $O 2>> gpurun_out/lown/err.txt
  for lib in paper_1211_0582_b200/tune/libdg_n*.so; do
    name=$(basename $lib .so)
    n=$(echo $name | sed -E 's/libdg_n([0-9]+)_.*/\1/')
    case $name in *f64*) c=f64-ffma-tiled;; *) c=f32-ffma-tiled;; esac
    DG_LIB=$lib timeout 600 python tools/variant_sweep.py --mesh-n $mesh --steps 5 --orders $n --cases $c | sed "s/^/{\"lib\": \"$name\", \"mesh\": $mesh, \"row\": /; s/$/}/" >> $O 2>> gpurun_out/lown/err.txt
  done
done
echo done
