#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the small C1 workload, every variant, acoustics
# through the tensor-core kernels and 2 loopback partitions (tools/sanitize_run.py).  The TC kernel is
# also racechecked with DG_TC_SPIN (its mbarrier waits as plain try_wait loops, no suspend-time hint):
# the same synchronisation protocol, to tell racecheck's view of the hinted waits from a real race.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/san
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/san/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san/sanitize_$tool.txt
done
if [ -e paper_1211_0582_b200/tune/libdg_tcspin.so ]; then
  DG_LIB=paper_1211_0582_b200/tune/libdg_tcspin.so timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 \
    python tools/sanitize_run.py 4:4:3,4:4:8 > gpurun_out/san/sanitize_racecheck_tc_spin.txt 2>&1
  echo "rc=$?" >> gpurun_out/san/sanitize_racecheck_tc_spin.txt
fi
echo done
