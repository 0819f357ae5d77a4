#!/usr/bin/env python
"""Cost of the multi-rank data path (a6 / §8(e)) measured on ONE GPU with the loopback transport:
P z-slab partitions stepped in lockstep by dg_group_lserk_step (boundary-first single-launch stages,
boundary-tile signal, pack kernel and ghost records, device-to-device copies in place of
ncclSend/Recv beside the interior tiles), against one partition.  On one GPU the partitions' persistent
kernels share the SMs, so the P > 1 time is P ranks' work plus the halo machinery's overhead; it is not
a scaling number.  Two meshes: "split" = the C2 mesh cut into P slabs (total work fixed), "weak" = a
Kuhn 15 x 15 x 15P box, i.e. C2-sized partitions (the per-rank size of the weak-scaling bench), where
overhead = t_P / (P t_1) - 1.
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
t1 = None
for mode in ("split", "weak"):
    for P in ((1, 2, 3, 5) if mode == "split" else (1, 2, 4)):
        VX, E = di.kuhn_box(n) if mode == "split" else di.kuhn_box(n, nz=n * P)
        K = E.shape[0]
        U0 = di.random_fields(K, N, seed=0)
        dt = di.dt_rule(VX, E, N)
        solvers = []
        for r in range(P):
            sv = Solver(N, precision=prec, rank=r, nranks=P) if P > 1 else Solver(N, precision=prec)
            sv.mesh_upload(VX, E)
            sv.fields_upload(U0[:, sv.local_elements()])
            solvers.append(sv)
        step = (lambda: group_lserk_step(solvers, dt, 1)) if P > 1 else (lambda: solvers[0].lserk_step(dt, 1))
        for _ in range(3):
            step()
        for sv in solvers:
            sv.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        for sv in solvers:
            sv.synchronize()
        ms = (time.perf_counter() - t0) / steps * 1e3
        if P == 1:
            t1 = ms
        print(json.dumps({"mode": mode, "N": N, "precision": prec, "K": K, "P": P, "ms_per_step": round(ms, 4),
                          "overhead_vs_P_x_one_partition": round(ms / (P * t1) - 1, 4) if mode == "weak" else None,
                          "overhead_vs_one_solver": round(ms / t1 - 1, 4) if mode == "split" else None,
                          "launches_per_step_per_rank": solvers[0].launches_per_step()}), flush=True)
        for sv in solvers:
            sv.close()
