#!/bin/bash
# Low-order ring-depth tuning builds (paper_1211_0582_b200/tune/libdg_{d,w}<N>*.so: d = FP64 FFMA, w = FP64 WS,
# f = FP32 FFMA) against the default library, on C2 and the HBM-resident C4 mesh, twice.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/lt
O=gpurun_out/lt/lown.txt
rm -f $O
for mesh in 15 56; do for r in 1 2; do
  timeout 300 python tools/variant_sweep.py --mesh-n $mesh --steps 10 --orders 1,2,3 --cases f64-ffma-tiled,f64-ws-dmma | sed "s/^/default /" >> $O 2>&1
  for l in paper_1211_0582_b200/tune/libdg_*.so; do
    n=$(basename $l .so); o=$(echo $n | sed -E "s/libdg_[a-z]([0-9]).*/\1/")
    case $n in libdg_d*) c=f64-ffma-tiled;; libdg_w*) c=f64-ws-dmma;; *) c=f32-ffma-tiled;; esac
    DG_LIB=$l timeout 300 python tools/variant_sweep.py --mesh-n $mesh --steps 10 --orders $o --cases $c | sed "s/^/$n /" >> $O 2>&1
  done
done; done
echo done
