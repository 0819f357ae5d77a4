#!/usr/bin/env python
"""Cost of the multi-rank data path (a6 / §8(e)) measured on ONE GPU with the loopback transport:
P z-slab partitions of the C2 mesh stepped in lockstep by dg_group_lserk_step (pack kernel, ghost
records, interior/boundary split launches, device-to-device copies in place of ncclSend/Recv),
against one partition.  On one GPU the partitions' persistent kernels share the SMs, so the P > 1
time is the single-GPU work plus the halo machinery's overhead; it is not a scaling number.
Usage: python tools/loopback_timing.py [N] [prec]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dg_inputs as di  # noqa: E402
from paper_1211_0582_b200.dg import Solver, group_lserk_step  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n, steps = 15, 20
VX, E = di.kuhn_box(n)
K = E.shape[0]
U0 = di.random_fields(K, N, seed=0)
dt = di.dt_rule(VX, E, N)
for P in (1, 2, 3, 5):
    solvers = []
    for r in range(P):
        sv = Solver(N, precision=prec, rank=r, nranks=P) if P > 1 else Solver(N, precision=prec)
        sv.mesh_upload(VX, E)
        sv.fields_upload(U0[:, sv.local_elements()])
        solvers.append(sv)
    step = (lambda: group_lserk_step(solvers, dt, 1)) if P > 1 else (lambda: solvers[0].lserk_step(dt, 1))
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    for sv in solvers:
        sv.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    for sv in solvers:
        sv.synchronize()
    ms = (time.perf_counter() - t0) / steps * 1e3
    print(json.dumps({"N": N, "precision": prec, "K": K, "P": P, "ms_per_step": round(ms, 4),
                      "launches_per_step_per_rank": solvers[0].launches_per_step()}), flush=True)
    for sv in solvers:
        sv.close()
