#!/bin/bash
# Benchmark every paper_1211_0582_b200/tune/libdg_*.so build on the FP64 bench config for orders ${ORDERS:-3 4 5}.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for lib in paper_1211_0582_b200/tune/libdg_*.so; do
  name=$(basename $lib .so)
  for N in ${ORDERS:-3 4 5}; do
    DG_LIB=$lib timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 20 --warmup 5 --order $N > /tmp/t.json 2>/tmp/t.err
    python -c "import json,sys; d=json.loads(open('/tmp/t.json').read().strip().splitlines()[-1]); print('$name', 'N=$N', d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null || (echo "$name N=$N FAILED"; tail -3 /tmp/t.err)
  done
done
