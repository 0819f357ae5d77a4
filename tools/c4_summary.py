#!/usr/bin/env python
"""Summarise the HBM-resident order sweep on the C4 mesh (tools/gpu_r2_evidence.sh):
bench lines (<src>/c4sweep.jsonl) + the ncu metrics of ONE WHOLE LSERK4 step (5 stage launches;
<src>/c4ncu_p{8,4}_N{n}.csv).  Per (precision, N): DRAM bytes per launch for stage 0 (no residual
read) and for stages 1..4 against the algorithmic bytes (B(N) K for stages 1..4, B(N) K minus the
residual read for stage 0), pipe utilisation, and the executed floating-point work
(SASS thread-instruction counters; tensor: DMMA / HMMA warp instructions, tcgen05 kind::tf32 ops)
against the F(N) K model, which shows padding and the 3xTF32 multiplicity.
Writes profiles/<tag>_c4_sweep.json and prints a markdown table.
Usage: python tools/c4_summary.py <tag> <src dir>"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import dg_inputs as di  # noqa: E402


def ncu_launches(path):
    """{launch id: {metric: value, 'kernel': name}}"""
    out = defaultdict(dict)
    if not os.path.exists(path):
        return {}
    with open(path) as fh:
        rows = [r for r in csv.reader(fh) if len(r) == 15 and r[0] != "ID"]
    for r in rows:
        try:
            v = float(r[14].replace(",", ""))
        except ValueError:
            continue
        out[int(r[0])][r[12]] = v
        out[int(r[0])]["kernel"] = r[4].split("(")[0]
    return dict(out)


def executed_flops(m):
    """Executed FP work of one launch, counting an FMA as 2 flops (SASS thread-instruction counters)."""
    g = lambda k: m.get(k, 0.0)  # noqa: E731
    simt = (2 * g("sm__sass_thread_inst_executed_op_dfma_pred_on.sum") + g("sm__sass_thread_inst_executed_op_dadd_pred_on.sum")
            + g("sm__sass_thread_inst_executed_op_dmul_pred_on.sum") + 2 * g("sm__sass_thread_inst_executed_op_ffma_pred_on.sum")
            + g("sm__sass_thread_inst_executed_op_fadd_pred_on.sum") + g("sm__sass_thread_inst_executed_op_fmul_pred_on.sum")
            + 4 * g("sm__sass_thread_inst_executed_op_ffma2_pred_on.sum") + 2 * g("sm__sass_thread_inst_executed_op_fadd2_pred_on.sum")
            + 2 * g("sm__sass_thread_inst_executed_op_fmul2_pred_on.sum"))
    # DMMA.8x8x4 warp instruction = 256 FMA; legacy HMMA m16n8k8 tf32 = 1024 FMA; the tcgen05 ops-path
    # counter counts flops (checked: at N = 8 it gives 3.27 x F(N) K, the 3xTF32 multiplicity times the
    # NP16 / Np and K-chunk padding, 3 x 176/165 x 688/675)
    tensor = (2 * 256 * g("sm__inst_executed_pipe_tensor_subpipe_dmma.sum")
              + 2 * 1024 * g("sm__inst_executed_pipe_tensor_subpipe_hmma.sum")
              + g("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum"))
    return simt, tensor


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "ev")
    rows = []
    for line in open(os.path.join(src, "c4sweep.jsonl")):
        d = json.loads(line)
        c = d["config"]
        N, prec = c["order"], 8 if c["precision"] == "f64" else 4
        K = c["K_total"]
        Np = di.np_of(N)
        L = ncu_launches(os.path.join(src, f"c4ncu_p{prec}_N{N}.csv"))
        alg = bench.bytes_per_elem_stage(N, prec) * K
        alg0 = alg - 6 * Np * prec * K  # stage 0 does not read the residual
        ids = sorted(L)
        st0 = [L[i] for i in ids if i % 5 == 0]
        st14 = [L[i] for i in ids if i % 5 != 0]
        dram = lambda m: m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)  # noqa: E731
        avg = lambda ms, k: sum(m.get(k, 0) for m in ms) / max(len(ms), 1)  # noqa: E731
        d14 = sum(dram(m) for m in st14) / max(len(st14), 1)
        d0 = sum(dram(m) for m in st0) / max(len(st0), 1)
        fpe = bench.flops_per_elem_stage(N)
        simt, tensor = (0.0, 0.0)
        for m in st14:
            a, b = executed_flops(m)
            simt += a / len(st14)
            tensor += b / len(st14)
        row = {"precision": c["precision"], "N": N, "K": K, "kernel": c["kernel"],
               "ms_per_step": d["ms_per_step"], "gdof_s": round(d["value"] / 1e9, 3), "roofline": d["roofline"],
               "ncu_kernel": st14[0]["kernel"] if st14 else None, "ncu_launches": len(ids),
               "ncu_ms_per_launch_stage1_4": round(avg(st14, "gpu__time_duration.sum") / 1e6, 4),
               "dram_bytes_per_launch_stage1_4": d14, "alg_bytes_per_launch_stage1_4": alg,
               "dram_over_alg_stage1_4": round(d14 / alg, 3) if d14 else None,
               "dram_bytes_stage0": d0, "alg_bytes_stage0": alg0,
               "dram_over_alg_stage0": round(d0 / alg0, 3) if d0 else None,
               "dram_pct_of_peak": round(avg(st14, "dram__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
               "l2_hit_pct": round(avg(st14, "lts__t_sector_hit_rate.pct"), 1),
               "tensor_pipe_pct": round(avg(st14, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"), 1),
               "tc_pipe_pct": round(avg(st14, "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"), 1),
               "fp64_pipe_pct": round(avg(st14, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
               "fma_pipe_pct": round(avg(st14, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 1),
               "model_flops_per_launch": fpe * K, "exec_simt_flops": simt, "exec_tensor_flops": tensor,
               "exec_over_model": round((simt + tensor) / (fpe * K), 3) if simt + tensor else None}
        rows.append(row)
    out = os.path.join(ROOT, "profiles", f"{tag}_c4_sweep.json")
    with open(out, "w") as fh:
        json.dump({"mesh": "C4: Kuhn n=56, K=1053696 (HBM-resident)", "source": "tools/gpu_r2_final.sh (tools/gpu_r2_evidence.sh layout)",
                   "rows": rows}, fh, indent=1)
    print("| prec | N | kernel | ms/step | G DOF/s | bound | frac | DRAM % peak | DRAM/alg (st 1-4) | DRAM/alg (st 0) "
          "| tensor % | FP64 % | FMA % | exec/model flops |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        rf = r["roofline"]
        print(f"| {r['precision']} | {r['N']} | {r['kernel']} | {r['ms_per_step']:.3f} | {r['gdof_s']:.2f} | "
              f"{rf['bound']} | {rf['frac']:.3f} | {r['dram_pct_of_peak']} | {r['dram_over_alg_stage1_4']} | "
              f"{r['dram_over_alg_stage0']} | {r['tensor_pipe_pct']} | {r['fp64_pipe_pct']} | {r['fma_pipe_pct']} | "
              f"{r['exec_over_model']} |")


if __name__ == "__main__":
    main()
