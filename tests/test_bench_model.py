"""bench.py's measurement model against SURVEY.md §8(d)'s table (F(N) flops and B(N) fused-floor
bytes per element and stage, both precisions) and the roofline bookkeeping.  CPU only."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

# N -> (F(N), B FP64, B FP32)
TABLE = {1: (2328, 988, 504), 2: (9036, 2140, 1080), 3: (28600, 4060, 2040), 4: (76710, 6940, 3480),
         5: (180432, 10972, 5496), 6: (382648, 16348, 8184), 7: (747216, 23260, 11640),
         8: (1364850, 31900, 15960), 9: (2359720, 42460, 21240)}


@pytest.mark.parametrize("N", range(1, 10))
def test_flop_and_byte_model_match_survey_table(N):
    F, B64, B32 = TABLE[N]
    assert bench.flops_per_elem_stage(N) == F
    assert bench.bytes_per_elem_stage(N, 8) == B64
    assert bench.bytes_per_elem_stage(N, 4) == B32


def test_roofline_bound_follows_kernel_and_ridge():
    peaks = {"hbm_gbs": 6545.6, "dmma_tflops": 37.11, "fp64_tflops": 34.17, "tf32x3_tflops": 100.43,
             "fp32_tflops": 72.39}
    K = 20250
    # FP64 N=1 on DMMA: AI 2.36 < ridge 5.7 -> HBM-bound; N=4: AI 11.05 -> tensor
    r1 = bench.roofline(1, 8, K, 0.0119, peaks, 3)
    assert r1["bound"] == "hbm" and r1["unit"] == "GB/s"
    assert abs(r1["achieved"] - bench.bytes_per_elem_stage(1, 8) * K / 0.0119e-3 / 1e9) < 0.2
    r4 = bench.roofline(4, 8, K, 0.0741, peaks, 3)
    assert r4["bound"] == "tensor" and r4["peak"] == 37.11
    assert abs(r4["frac"] - bench.flops_per_elem_stage(4) * K / 0.0741e-3 / 1e12 / 37.11) < 1e-3
    # the FFMA kernel (variant 6) is SIMT: "alu" against the FFMA / DFMA peak
    assert bench.roofline(9, 4, K, 1.6, peaks, 6)["bound"] == "alu"
    assert bench.roofline(9, 4, K, 1.6, peaks, 6)["peak"] == 72.39
    assert bench.roofline(9, 8, K, 1.7, peaks, 6)["peak"] == 34.17
    # kernel families of resolved variants
    assert [bench.ws_kind(4, 8, v) for v in (1, 2, 3, 4, 5, 6)] == ["basic", "mma", "ws", "tc", "ws", "ffma"]


def test_random_fields_local_equals_global_draw():
    # bench.py draws each rank's fields by global element id without the global array
    # (per-rank host memory O(K_local)); the values must be exactly the global draw's
    import numpy as np

    import dg_inputs as di
    K, N = 777, 4
    full = di.random_fields(K, N, seed=3, nfields=6)
    for ids in (np.arange(K), np.arange(200, 389), np.random.default_rng(5).permutation(K)[:301], np.array([], int)):
        assert np.array_equal(di.random_fields_local(ids, K, N, seed=3, nfields=6), full[:, ids])
