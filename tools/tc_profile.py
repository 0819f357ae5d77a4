#!/usr/bin/env python
"""Cycle breakdown of the tcgen05 TC stage kernel (profiling build libdg_prof.so, `make prof`):
per-role clock64 counters of stage_tc.cuh, cycles per tile per warp of the role."""
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
NAMES = ["epi_wait_acc_full", "epi_work", "wr_wait_input", "wr_wait_tmem_slot", "wr_work", "flux_wait_slot",
         "flux_total", "mma_wait_operand", "unused", "mma_wait_op", "mma_issue", "ldr_wait_slab_free"]
WARPS = [4, 4, 4, 4, 4, 6, 6, 1, 1, 1, 1, 1]
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
    tiles = max(v[12], 1)
    ctas = 148
    print(f"N={N} tiles={tiles}  CTA cycles per tile {v[13] / tiles:.0f}; cycles per tile per warp of the role:")
    for i, k in enumerate(NAMES):
        print(f"  {k:20s} {v[i] / tiles / WARPS[i]:10.0f}")
    s.close()
