#!/usr/bin/env python
"""Cycle breakdown of the WS stage kernel (needs the profiling build:
make -C paper_1211_0582_b200/csrc prof; DG_LIB=paper_1211_0582_b200/libdg_prof.so)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DG_LIB", os.path.join(ROOT, "paper_1211_0582_b200", "libdg_prof.so"))
import dg_inputs as di  # noqa: E402
from paper_1211_0582_b200 import dg  # noqa: E402

f = dg.lib.dg_debug_ws_profile
f.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
NAMES = ["prod_wait_empty", "prod_wait_load", "prod_wait_traces", "prod_flux", "prod_trace_issue",
         "cons_wait_full", "cons_task", "tiles", "tasks", "prod_total", "cons_total"]
n = int(os.environ.get("MESH_N", "15"))
for N in [int(a) for a in sys.argv[1:]] or range(1, 10):
    VX, E = di.kuhn_box(n)
    s = dg.Solver(N, precision=8)
    s.mesh_upload(VX, E)
    s.fields_upload(di.random_fields(s.K_local, N, 0))
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 2)
    s.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    f(N, buf, 1)
    steps = 4
    s.lserk_step(dt, steps)
    s.synchronize()
    f(N, buf, 0)
    v = list(buf)
    tiles, tasks = max(v[7], 1), max(v[8], 1)
    # producer counters are per producer warp (lane 0 of each): 4 warps; consumer per MMA warp: 8
    line = {k: v[i] for i, k in enumerate(NAMES)}
    print(f"N={N} tiles={tiles} tasks={tasks}")
    print("  per tile (cycles, per producer warp): " + ", ".join(
        f"{k}={line[k] / tiles / 4:.0f}" for k in NAMES[:5]) + f", total={line['prod_total'] / tiles / 4:.0f}")
    print("  per task (cycles, per MMA warp):      " + f"wait_full={line['cons_wait_full'] / tasks:.0f}, "
          f"task={line['cons_task'] / tasks:.0f}; cons_total/tile/warp={line['cons_total'] / tiles / 8:.0f}")
    s.close()
