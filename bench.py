#!/usr/bin/env python
"""Benchmark: DOF-updates/s and GFLOP/s per LSERK4 step (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): Kuhn box mesh n=15 (K = 20 250 tets per
GPU), random U(-1,1) fields (seed 0, synthetic), PEC walls, upwind flux.  The
headline line is order N=4 in FP64; the N=1..9 x {FP64, FP32} sweep of the same
config is attached under "sweep".  A step = one LSERK4 step = 5 stages of the
full hot path (volume + flux + lift + update), graph-launched.

Multi-GPU (torchrun, one rank per GPU): weak scaling — every rank owns a 15x15x15
z-slab of a 15x15x(15P) box; partition-face traces are exchanged with NCCL each
stage (the path's one real exchange step).

Timing: W untimed warm-up steps; then K steps, each preceded by an L2 flush
(256 MiB write; the C2 state is smaller than the 126 MB L2) that is NOT timed;
each step bracketed by CUDA events on the solver's stream; barrier + synchronize
around the timed region; max over ranks.

`--impl reference` times the CPU oracle (oracle/, numpy FP64) on the same config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import dg_inputs as di  # noqa: E402

L2_FLUSH_BYTES = 256 << 20


def flops_per_elem_stage(N):
    """F(N): algorithmic flops per element per RHS + stage update."""
    Np, Nfp = di.np_of(N), di.nfp_of(N)
    return 36 * Np * Np + 48 * Np * Nfp + 102 * Np + 256 * Nfp


def flops_per_elem_stage_acoustics(N):
    """Acoustics (NEXT-3) analogue of F(N): volume 3 x 4 fields x 2Np^2, lift 4 fields x
    2 Np 4Nfp, chain rule + div/grad 32Np, update 16Np, flux 20 per face node."""
    Np, Nfp = di.np_of(N), di.nfp_of(N)
    return 24 * Np * Np + 32 * Np * Nfp + 48 * Np + 80 * Nfp


def bytes_per_elem_stage(N, w, nfields=6):
    """B(N): fused-stage algorithmic HBM bytes per element:
    u in, res in, res out, u out (24 Np words) + 25 geometry words + 20 B connectivity."""
    return w * (4 * nfields * di.np_of(N) + 25) + 20


def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            mp = json.load(fh)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json)"
    a = os.path.join(ROOT, "profiles", "alu_peaks.json")
    if os.path.exists(a):
        with open(a) as fh:
            ap = json.load(fh)
        peaks["fp64_tflops"] = float(ap["fp64_dfma_tflops"])
        peaks["fp32_tflops"] = float(ap["fp32_ffma_tflops"])
        peaks["dmma_tflops"] = float(ap["fp64_dmma_tflops"])
        # FP32 on tensor cores is 3xTF32 (3 MMA passes per algorithmic FMA): the denominator is the
        # measured tcgen05 kind::tf32 peak / 3, for the tcgen05 (TC) and the mma.sync (WS) kernels alike
        peaks["tf32x3_tflops"] = float(ap.get("tf32_tcgen05_tflops", 1113.7)) / 3.0
        peaks["tf32_mma_sync_tflops"] = float(ap.get("tf32_mma_sync_tflops", 301.3))
        peaks["alu_src"] = ("measured (profiles/alu_peaks.json: tools/alu_peaks.cu DFMA/FFMA/DMMA, "
                            "tools/tcgen05_peak.cu tcgen05 kind::tf32)")
    else:
        # unit counts x max clock: 148 SMs x 64 DFMA (128 FFMA) lanes x 2 flop x 1.965 GHz
        peaks["fp64_tflops"] = 148 * 64 * 2 * 1.965e9 / 1e12
        peaks["fp32_tflops"] = 148 * 128 * 2 * 1.965e9 / 1e12
        peaks["dmma_tflops"] = peaks["fp64_tflops"]
        peaks["tf32x3_tflops"] = peaks["fp32_tflops"]
        peaks["alu_src"] = "derived from unit counts and clocks (not measured)"
    return peaks


def ws_kind(N, prec, variant):
    """Kernel family of a RESOLVED dg_variant (Solver.kernel_variant(): the library resolves AUTO)."""
    return {1: "basic", 2: "mma" if prec == 8 else "basic", 3: "ws", 4: "tc", 5: "ws", 6: "ffma"}.get(variant, "ws")


def load_traffic(N, prec, variant, K):
    """Per-launch DRAM bytes of the stage kernel from committed ncu captures of the same (precision,
    variant, order, mesh size), if any: profiles/r2_traffic.json (a stage that reads the residual;
    tools/traffic_table.py), else round 1's profiles/r1_traffic.json."""
    key = f"{'f64' if prec == 8 else 'f32'}:{variant}:{N}:K{K}"
    for name in ("r2_traffic.json", "r1_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                v = json.load(fh).get(key, {}).get("dram_bytes")
            if v:
                return v
        except Exception:
            pass
    return None


def roofline(N, prec, K_total, kernel_ms, peaks, variant=0, traffic=None, fpe=None, bpe=None):
    """Roofline of the fused stage kernel.  FP64 MMA/WS variants: contractions on the
    FP64 tensor pipe (DMMA) -> bound "tensor" against the measured DMMA peak.  FP32
    WS variant: 3xTF32 on HMMA -> "tensor" against the measured TF32 mma.sync peak / 3
    (algorithmic flops counted once).  BASIC and FFMA (register-tiled SIMT): "alu" against
    the measured DFMA / FFMA peak."""
    w = 8 if prec == 8 else 4
    F = (fpe or flops_per_elem_stage(N)) * K_total
    B = (bpe or bytes_per_elem_stage(N, w)) * K_total
    kind = ws_kind(N, prec, variant)
    tensor = kind in ("ws", "mma", "tc")
    if prec == 8:
        pipe = peaks["dmma_tflops"] if tensor else peaks["fp64_tflops"]
    else:
        pipe = peaks["tf32x3_tflops"] if tensor else peaks["fp32_tflops"]
    ridge = pipe * 1e12 / (peaks["hbm_gbs"] * 1e9)
    ai = F / B
    if ai < ridge:
        ach = B / (kernel_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": traffic, "ai_flop_per_byte": round(ai, 2)}
    ach = F / (kernel_ms * 1e-3) / 1e12
    out = {"bound": "tensor" if tensor else "alu", "achieved": round(ach, 3), "peak": round(pipe, 2), "unit": "TFLOP/s",
           "frac": round(ach / pipe, 4), "traffic": traffic, "ai_flop_per_byte": round(ai, 2)}
    if prec != 8:  # FP32: also against the FFMA pipe (the SIMT side of the TF32-or-FFMA choice)
        out["frac_ffma"] = round(ach / peaks["fp32_tflops"], 4)
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while active."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws == 1:
        return 0, 1, 0, None
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, ws, local, dist


def nccl_unique_id(rank, dist):
    # ncclGetUniqueId on rank 0 through the library's own NCCL (dlopen), broadcast via torch.distributed
    import ctypes
    obj = [None]
    if rank == 0:
        lib = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)
        buf = ctypes.create_string_buffer(128)
        assert lib.ncclGetUniqueId(buf) == 0
        obj[0] = bytes(buf.raw)
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def run_dg(args, N, prec, rank, world, local, dist, stream, flush, nccl_id, peaks, e2e=False):
    import torch
    from paper_1211_0582_b200.dg import Solver

    if world > 1:
        # a fresh ncclUniqueId per solver: an id's bootstrap root serves one communicator only
        nccl_id = nccl_unique_id(rank, dist)

    n = args.mesh_n
    VX, E = di.kuhn_box(n, nz=n * world)
    if args.shuffle_seed is not None:
        E, _ = di.shuffle_elements(E, args.shuffle_seed)
    K_total = E.shape[0]
    system = getattr(args, "system", 0)
    nf = 4 if system == 1 else 6
    s = Solver(N, precision=prec, device=local, stream=stream.cuda_stream, rank=rank, nranks=world,
               nccl_id=nccl_id, variant=args.variant, reorder=args.reorder, system=system)
    s.mesh_upload(VX, E)
    Kl = s.K_local
    # this rank's elements only (per-rank host memory O(K_local)); identical to the global draw
    U0 = di.random_fields_local(s.local_elements(), K_total, N, seed=0, nfields=nf)
    s.fields_upload(U0)
    dt = di.dt_rule(VX, E, N)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            s.lserk_step(dt, 1)
        s.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for a, b in evs:
            flush.zero_()                       # L2 flush, outside the timed events
            a.record(stream)
            s.lserk_step(dt, 1)
            b.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms_total = sum(ms_steps)
    if dist:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    Np = di.np_of(N)
    dofs = nf * Np * K_total
    fpe = flops_per_elem_stage_acoustics(N) if system == 1 else flops_per_elem_stage(N)
    res = {"N": N, "precision": "f64" if prec == 8 else "f32", "K_total": K_total, "K_local": Kl,
           "ms_per_step": round(ms_step, 5), "dof_updates_per_s": dofs / (ms_step * 1e-3),
           "gflops": 5 * K_total * fpe / (ms_step * 1e-3) / 1e9,
           "launches_per_step": s.launches_per_step(),
           # SURVEY §8(d) row fields: per-step spread (this rank), node updates, L2 residency
           "ms_step_median": round(float(np.median(ms_steps)), 5), "ms_step_min": round(min(ms_steps), 5),
           "ms_step_max": round(max(ms_steps), 5), "node_updates_per_s": Np * K_total / (ms_step * 1e-3),
           "l2_resident": bool(3 * nf * Np * Kl * (8 if prec == 8 else 4) < 126e6)}
    kv = s.kernel_variant()  # the stage kernel actually in use (AUTO resolved by the library)
    res["kernel"] = ws_kind(N, prec, kv)
    # dominant kernel: the fused stage kernel (5 launches per step, the step's only kernel at 1 GPU)
    kernel_ms = ms_step / 5 if world == 1 else s.time_stage_kernel(10)
    res["stage_kernel_ms"] = round(kernel_ms, 5)
    if system == 1:
        # acoustics: the FFMA / BASIC kernels (FMA contractions: alu) or the tcgen05 TC kernel
        # (3xTF32: tensor), each against its own pipe, or hbm by its own F/B
        res["system"] = "acoustics"
        res["roofline"] = roofline(N, prec, Kl, kernel_ms, peaks, kv, None, fpe,
                                   bytes_per_elem_stage(N, 8 if prec == 8 else 4, 4))
    else:
        res["roofline"] = roofline(N, prec, Kl, kernel_ms, peaks, kv,
                                   traffic=load_traffic(N, prec, args.variant, Kl) if world == 1 else None)
    if e2e:
        # end to end through the C ABI with HOST buffers, every step: H2D of the step's
        # input fields from pinned memory, the LSERK4 step, D2H of the resulting fields.
        # Headline: the pipelined API (dg_fields_upload_async / dg_fields_download_async:
        # copy streams + double-buffered staging, so step k's copies overlap steps k-1 and
        # k+1); "sync" is the blocking dg_fields_upload / dg_fields_download sequence.
        host_in = [torch.from_numpy(np.ascontiguousarray(U0)).pin_memory().numpy() for _ in range(2)]
        host_out = [torch.empty((nf, Kl, Np), dtype=torch.float64).pin_memory().numpy() for _ in range(2)]

        def timed(fn):
            fn(0)
            s.synchronize()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            for k in range(args.steps):
                fn(k)
            s.synchronize()
            el = time.perf_counter() - t0
            if dist:
                t = torch.tensor([el], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t.item())
            return el

        def cycle_async(k):
            s.fields_upload_async(host_in[k % 2])
            s.lserk_step(dt, 1)
            s.fields_download_async(host_out[k % 2])

        def cycle_sync(k):
            s.fields_upload(host_in[k % 2])
            s.lserk_step(dt, 1)
            s.fields_download(host_out[k % 2])

        # three repeats of the K-step loop, median reported (host-side jitter moves a single
        # wall-clock repeat by up to ~20 %); all repeats are listed
        reps = [timed(cycle_async) for _ in range(3)]
        el = float(np.median(reps))
        el_sync = timed(cycle_sync)
        res["e2e"] = {"value": dofs * args.steps / el, "unit": "DOF-updates/s",
                      "h2d_bytes_per_step": int(host_in[0].nbytes), "d2h_bytes_per_step": int(host_out[0].nbytes),
                      "ms_per_step": round(el / args.steps * 1e3, 4),
                      "repeats_ms_per_step": [round(r / args.steps * 1e3, 4) for r in reps],
                      "api": "pipelined async upload/step/download",
                      "sync": {"value": dofs * args.steps / el_sync, "ms_per_step": round(el_sync / args.steps * 1e3, 4),
                               "api": "blocking dg_fields_upload / dg_lserk_step / dg_fields_download"}}
    s.close()
    return res


def oracle_rhs_rate(N, n, budget_s=2.0):
    """Bounded oracle sample for the order sweep: whole RHS evaluations (numpy FP64, C2
    mesh) for about budget_s; one LSERK4 step = 5 RHS + the stage updates, so
    DOF-updates/s is quoted as 6 Np K / (5 t_rhs) (an upper bound: the updates are ignored)."""
    import oracle
    VX, E = di.kuhn_box(n)
    st = oracle.Setup(VX, E, N)
    U = di.random_fields(st.K, N, seed=0)
    oracle.rhs(st, U)
    reps = 0
    t0 = time.perf_counter()
    while True:
        oracle.rhs(st, U)
        reps += 1
        el = time.perf_counter() - t0
        if el > budget_s:
            break
    t_rhs = el / reps
    return {"N": N, "value": 6 * di.np_of(N) * st.K / (5 * t_rhs), "unit": "DOF-updates/s",
            "rhs_s": round(t_rhs, 4), "rhs_evals": reps}


def oracle_baseline(N, n, budget_s=20.0, max_steps=None):
    """The CPU oracle as it stands, timed on this host on the C2 mesh (FP64)."""
    import oracle
    VX, E = di.kuhn_box(n)
    st = oracle.Setup(VX, E, N)
    U = di.random_fields(st.K, N, seed=0)
    dt = di.dt_rule(VX, E, N)
    oracle.rhs(st, U)                      # warm-up (BLAS threads, caches)
    steps = 0
    t0 = time.perf_counter()
    while True:
        U = oracle.lserk4(st, U, dt, 1)
        steps += 1
        el = time.perf_counter() - t0
        if el > budget_s or (max_steps and steps >= max_steps):
            break
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = len(os.sched_getaffinity(0))
    dofs = 6 * di.np_of(N) * st.K
    return {"value": dofs * steps / el, "unit": "DOF-updates/s", "cores": int(threads), "kind": "oracle",
            "sample": f"C2 mesh (Kuhn n={n}, K={st.K}), N={N}, FP64 numpy, {steps} LSERK4 step(s) "
                      f"in {el:.1f} s (mesh setup excluded)", "steps": steps, "seconds": el}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dg", choices=["dg", "reference"])
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--precision", type=int, default=8, choices=[4, 8])
    ap.add_argument("--mesh-n", type=int, default=15)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the HBM-resident C4 line (K = 1.05M)")
    ap.add_argument("--shuffle-seed", type=int, default=None, help="random element numbering (unstructured-like)")
    ap.add_argument("--reorder", action="store_true", help="library Morton renumbering of the elements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end measurement")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")

    rank, world, local, dist = dist_setup()
    N, prec = args.order, args.precision
    Np = di.np_of(N)
    cname = {15: "C2", 56: "C4"}.get(args.mesh_n, "custom")
    workload = (f"{cname}: Kuhn box n={args.mesh_n} per GPU (K={6 * args.mesh_n ** 3}/GPU), N={N}, LSERK4, "
                f"PEC walls, upwind flux, U(-1,1) fields (seed 0)")

    def config_of(K_total, precision, engine):
        # identical keys for both arms, so the driver can match the workloads
        return {"workload": workload, "K_total": K_total, "order": N, "precision": precision,
                "parallelism": f"mesh z-slabs x{world}, NCCL halo", "engine": engine}
    base = {"metric": "DOF-updates/s per LSERK4 step (and GFLOP/s)", "unit": "DOF-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "data": "synthetic (seeded U(-1,1) fields on a generated Kuhn tet box)"}

    if args.impl == "reference":
        if rank != 0:
            return
        K = 6 * args.mesh_n ** 3
        t0 = time.perf_counter()
        cb = oracle_baseline(N, args.mesh_n, budget_s=1e9, max_steps=args.steps)
        out = dict(base)
        out.update({"impl": "reference", "value": cb["value"], "ms_per_step": cb["seconds"] / cb["steps"] * 1e3,
                    "dtype": "f64", "n_gpus": 1,
                    "config": config_of(K, "f64", "CPU oracle (numpy FP64, host cores)"),
                    "cpu_baseline": {"value": cb["value"], "unit": cb["unit"], "cores": cb["cores"],
                                     "kind": "oracle", "sample": cb["sample"]},
                    "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0},
                    "wall_s": round(time.perf_counter() - t0, 2)})
        print(json.dumps(out), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    nccl_id = None  # run_dg bootstraps a fresh NCCL id per solver
    peaks = load_peaks()

    with ClockSampler(local) as clk:
        head = run_dg(args, N, prec, rank, world, local, dist, stream, flush, nccl_id, peaks, e2e=not args.no_e2e)
        sweep = []
        if not args.no_sweep:
            for p in (8, 4):
                for n_ in range(1, 10):
                    r = run_dg(args, n_, p, rank, world, local, dist, stream, flush, nccl_id, peaks)
                    sweep.append({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
        acoustics = []
        if not args.no_sweep:
            # NEXT-3: the second linear system on the same C2 mesh (AUTO: FFMA / TC kernel, 4 fields)
            import copy
            a3 = copy.copy(args)
            a3.system, a3.variant = 1, 0
            for p in (8, 4):
                r = run_dg(a3, 4, p, rank, world, local, dist, stream, flush, nccl_id, peaks)
                acoustics.append({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
        large = None
        if not args.no_large and world == 1:
            # configs[3] at one GPU: Kuhn n=56, K = 1 053 696 (state 1.8 GB >> 126 MB L2), N=4 FP64
            import copy
            a2 = copy.copy(args)
            a2.mesh_n, a2.steps, a2.warmup = 56, max(3, min(args.steps, 10)), 3
            r = run_dg(a2, 4, 8, rank, world, local, dist, stream, flush, nccl_id, peaks)
            large = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}
            large["workload"] = "C4 (configs[3]) at 1 GPU: Kuhn n=56, K=1053696, N=4, FP64; HBM-resident"
    clocks = clk.summary()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(N, args.mesh_n, budget_s=args.cpu_budget)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if not args.no_sweep:
            # the oracle across the order sweep: bounded RHS samples (~2 s per order)
            cpu["sweep"] = [oracle_rhs_rate(n_, args.mesh_n, 2.0) for n_ in range(1, 10)]

    if rank == 0:
        out = dict(base)
        out.update({"value": head["dof_updates_per_s"], "ms_per_step": head["ms_per_step"],
                    "gflops": round(head["gflops"], 2), "dtype": "f64" if prec == 8 else "f32",
                    "config": {**config_of(head["K_total"], head["precision"], "libdg (sm_100a)"),
                               "l2": "flushed before every timed step (256 MiB write, not timed)",
                               "variant": args.variant, "kernel": head["kernel"],
                               "element_order": ("shuffled(seed %d)" % args.shuffle_seed
                                                 if args.shuffle_seed is not None else "natural")
                                                + (" + Morton reorder" if args.reorder else "")},
                    "roofline": head["roofline"], "e2e": head.get("e2e"),
                    "gpu_launches": head["launches_per_step"] * args.steps,
                    "stage_kernel_ms": head["stage_kernel_ms"],
                    "clocks": clocks, "cpu_baseline": cpu,
                    "peaks": {k: v for k, v in peaks.items()},
                    "sweep": sweep, "acoustics": acoustics, "large": large})
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
