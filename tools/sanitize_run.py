#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): the C1 cavity
mesh (48 tets), one RHS and one LSERK4 step per kernel variant and precision, N = 3 (and
N = 8 for the tcgen05 kernel, whose operator ring streams there)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import dg_inputs as di  # noqa: E402
from paper_1211_0582_b200.dg import Solver  # noqa: E402

CASES = [(8, 1, 3), (8, 2, 3), (8, 3, 3), (8, 6, 3), (4, 1, 3), (4, 3, 3), (4, 4, 3), (4, 4, 8), (4, 6, 3)]
only = sys.argv[1] if len(sys.argv) > 1 else ""
VX, E = di.kuhn_box(2)
for prec, var, N in CASES:
    if only and f"{prec}:{var}:{N}" not in only.split(","):
        continue
    s = Solver(N, precision=prec, variant=var)
    s.mesh_upload(VX, E)
    U = di.random_fields(E.shape[0], N, seed=0)
    s.fields_upload(U)
    R = s.rhs()
    s.lserk_step(di.dt_rule(VX, E, N), 1)
    Un = s.fields_download()
    print(f"prec={prec} variant={var} N={N} finite={bool(np.isfinite(R).all() and np.isfinite(Un).all())}", flush=True)
    s.close()
