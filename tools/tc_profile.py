#!/usr/bin/env python
"""Cycle breakdown of the tcgen05 TC stage kernel (profiling build, see tools/ws_profile.py)."""
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
NAMES = ["load_wait_empty", "flux_wait_load", "flux_trace_issue", "flux_wait_traces", "flux_compute", "flux_lo_split",
         "mma_wait_full", "mma_wait_acc_empty", "mma_issue", "epi_wait_acc_full", "epi_pass1", "epi_pass2",
         "epi_store_release"]
WARPS = [1, 4, 4, 4, 4, 4, 1, 1, 1, 4, 4, 4, 4]  # lane-0 counters per role
n = int(os.environ.get("MESH_N", "15"))
for N in [int(a) for a in sys.argv[1:]] or [4]:
    VX, E = di.kuhn_box(n)
    s = dg.Solver(N, precision=4, variant=4)
    s.mesh_upload(VX, E)
    s.fields_upload(di.random_fields(s.K_local, N, 0))
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 2)
    s.synchronize()
    buf = (ctypes.c_ulonglong * 32)()
    f(N, buf, 1)
    s.lserk_step(dt, 4)
    s.synchronize()
    f(N, buf, 0)
    v = list(buf)[16:]
    tiles = max(v[13], 1)
    print(f"N={N} tiles={tiles}  cycles per tile per warp of the role:")
    for i, k in enumerate(NAMES):
        print(f"  {k:20s} {v[i] / tiles / WARPS[i]:10.0f}")
    s.close()
