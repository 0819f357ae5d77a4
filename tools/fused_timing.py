#!/usr/bin/env python
"""Stage-fused vs per-stage launch timing: ms per LSERK4 step for k steps per dg_lserk_step
call, with and without an L2 flush before each call, for DG_VARIANT_FUSED (5) and MMA_WS (3)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import dg_inputs as di  # noqa: E402
from paper_1211_0582_b200.dg import Solver  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
stream = torch.cuda.Stream()
for N, var in [(int(a), v) for a in (sys.argv[1:] or [4, 9]) for v in (5, 3)]:
    VX, E = di.kuhn_box(15)
    s = Solver(N, variant=var, stream=stream.cuda_stream)
    s.mesh_upload(VX, E)
    s.fields_upload(di.random_fields(s.K_local, N, 0))
    dt = di.dt_rule(VX, E, N)
    for k in (1, 4):
        for fl in (False, True):
            with torch.cuda.stream(stream):
                s.lserk_step(dt, k)
                torch.cuda.synchronize()
                tot, reps = 0.0, 8
                for _ in range(reps):
                    if fl:
                        flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    s.lserk_step(dt, k)
                    b.record(stream)
                    torch.cuda.synchronize()
                    tot += a.elapsed_time(b)
            print(f"variant={var} N={N} steps/call={k} flush={fl}: "
                  f"{tot / reps / k:.4f} ms/step", flush=True)
    s.close()
