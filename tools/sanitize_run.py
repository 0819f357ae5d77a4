#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): the C1 cavity
mesh (48 tets), one RHS and one LSERK4 step per kernel variant and precision, N = 3 (and
N = 8 for the tcgen05 kernel, whose operator ring streams there); acoustics through the tensor-core
kernels; and 2 loopback partitions (boundary-first stages: the store warps' boundary signal, the
stream-memop wait, the pack kernel) for the WS, TC and FFMA kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import dg_inputs as di  # noqa: E402
from paper_1211_0582_b200.dg import DG_SYSTEM_ACOUSTICS, Solver, group_lserk_step  # noqa: E402

CASES = [(8, 1, 3, 0), (8, 2, 3, 0), (8, 3, 3, 0), (8, 6, 3, 0), (4, 1, 3, 0), (4, 3, 3, 0), (4, 4, 3, 0), (4, 4, 8, 0),
         (4, 6, 3, 0), (8, 3, 3, 1), (4, 4, 3, 1), (4, 4, 8, 1)]
only = sys.argv[1] if len(sys.argv) > 1 else ""
VX, E = di.kuhn_box(2)
for prec, var, N, sys_ in CASES:
    if only and f"{prec}:{var}:{N}" not in only.split(","):
        continue
    s = Solver(N, precision=prec, variant=var, system=sys_)
    s.mesh_upload(VX, E)
    U = di.random_fields(E.shape[0], N, seed=0, nfields=6 if sys_ == 0 else 4)
    s.fields_upload(U)
    R = s.rhs()
    s.lserk_step(di.dt_rule(VX, E, N), 1)
    Un = s.fields_download()
    print(f"prec={prec} variant={var} N={N} system={sys_} finite={bool(np.isfinite(R).all() and np.isfinite(Un).all())}",
          flush=True)
    s.close()
for prec, var, N in ((8, 3, 3), (4, 4, 3), (4, 6, 3)):  # 2 loopback partitions: boundary signal + memop wait + pack
    VX2, E2 = di.kuhn_box(3)
    K2 = E2.shape[0]
    U = di.random_fields(K2, N, seed=1)
    sv = []
    for r in range(2):
        p = Solver(N, precision=prec, variant=var, rank=r, nranks=2)
        p.mesh_upload(VX2, E2)
        p.fields_upload(U[:, p.local_elements()])
        sv.append(p)
    group_lserk_step(sv, di.dt_rule(VX2, E2, N), 2)
    ok = all(bool(np.isfinite(p.fields_download()).all()) for p in sv)
    print(f"loopback prec={prec} variant={var} N={N} finite={ok}", flush=True)
    for p in sv:
        p.close()
