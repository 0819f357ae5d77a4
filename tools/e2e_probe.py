"""e2e pipeline probe: per-cycle time of upload_async / lserk_step / download_async variants (C2, N=4, FP64)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import dg_inputs as di
from paper_1211_0582_b200 import Solver

N, n, steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4, 15, 20
VX, E = di.kuhn_box(n)
K = E.shape[0]
stream = torch.cuda.Stream()
s = Solver(N, precision=8, stream=stream.cuda_stream)
work = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
s.mesh_upload(VX, E)
U0 = di.random_fields(K, N, seed=0)
hin = [torch.from_numpy(np.ascontiguousarray(U0)).pin_memory().numpy() for _ in range(2)]
hout = [torch.empty(U0.shape, dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
s.fields_upload(U0)
dt = di.dt_rule(VX, E, N)

def timed(fn):
    fn(0); s.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        fn(k)
    s.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3

def full(k):
    s.fields_upload_async(hin[k % 2]); s.lserk_step(dt, 1); s.fields_download_async(hout[k % 2])
def io_only(k):
    s.fields_upload_async(hin[k % 2]); s.fields_download_async(hout[k % 2])
def up_only(k):
    s.fields_upload_async(hin[k % 2]); s.lserk_step(dt, 1)
def down_only(k):
    s.lserk_step(dt, 1); s.fields_download_async(hout[k % 2])
def step_only(k):
    s.lserk_step(dt, 1)
def full_busy(k):  # the step replaced by ~0.44 ms of torch elementwise work on the solver's stream
    s.fields_upload_async(hin[k % 2])
    with torch.cuda.stream(stream):
        for _ in range(9):
            work.mul_(1.0000001)
    s.fields_download_async(hout[k % 2])
for name, fn in (("full", full), ("full_busy", full_busy), ("io_only", io_only), ("up+step", up_only),
                 ("step+down", down_only), ("step", step_only)):
    print(f"{name:10s} {timed(fn):.4f} ms/cycle", flush=True)
