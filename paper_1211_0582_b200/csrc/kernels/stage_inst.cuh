// Stage-kernel instantiations for one order N = DG_N (stage_N<N>.cu defines DG_N and
// includes this file; nine translation units so nvcc builds the orders in parallel).
// Variants (include/dg.h): 1 BASIC, 2 MMA (FP64 DMMA, element-major), 3/0 MMA_WS
// (FP64 DMMA / FP32 3xTF32 mma.sync WS kernels), 4 TC (FP32 tcgen05 3xTF32), 6 FFMA.
#include "stage_tc.cuh"
#include "stage_ws32.cuh"

#include "stage_ffma.cuh"

#ifndef DG_N
#error "define DG_N before including stage_inst.cuh"
#endif
#define DG_CAT2(a, b) a##b
#define DG_CAT(a, b) DG_CAT2(a, b)
#define DG_FN(name) DG_CAT(name, DG_CAT(_N, DG_N))

namespace dg {

void DG_FN(launch_stage_f64)(const StageParams<double>& p, int mode, int variant, void* st) {
  if (variant == 1)       // DG_VARIANT_BASIC
    launch_stage_basic<double, DG_N>(p, mode, static_cast<cudaStream_t>(st));
  else if (variant == 6)  // DG_VARIANT_FFMA: register-tiled DFMA WS kernel
    launch_stage_ffma<double, DG_N>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else if (variant == 2)  // DG_VARIANT_MMA: DMMA, cp.async-pipelined, element-major layout
    launch_stage_mma<DG_N>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else                    // AUTO / DG_VARIANT_MMA_WS: DMMA, warp-specialized TMA pipeline, tiled layout
    launch_stage_ws<DG_N>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

void DG_FN(launch_stage_f32)(const StageParams<float>& p, int mode, int variant, void* st) {
  if (variant == 1 || variant == 2)  // BASIC (MMA has no FP32 kernel of its own)
    launch_stage_basic<float, DG_N>(p, mode, static_cast<cudaStream_t>(st));
  else if (variant == 6)             // FFMA: register-tiled FFMA WS kernel
    launch_stage_ffma<float, DG_N>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else if (variant == 4)             // TC: tcgen05 kind::tf32 (3xTF32), TMEM accumulators
    launch_stage_tc<DG_N>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else                               // MMA_WS: 3xTF32 mma.sync WS kernel
    launch_stage_ws32<DG_N>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

TileLayout DG_FN(ffma_layout)() { return ffma_layout<float, DG_N>(); }
size_t DG_FN(ffma_ops_count)() { return FfCfg<float, DG_N>::A_FLOATS; }
void DG_FN(ffma_ops)(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  ffma_ops<float, DG_N>(Dr, Ds, Dt, L, out);
}
TileLayout DG_FN(ffma64_layout)() { return ffma_layout<double, DG_N>(); }
size_t DG_FN(ffma64_ops_count)() { return FfCfg<double, DG_N>::A_FLOATS; }
void DG_FN(ffma64_ops)(const double* Dr, const double* Ds, const double* Dt, const double* L, double* out) {
  ffma_ops<double, DG_N>(Dr, Ds, Dt, L, out);
}
TileLayout DG_FN(ws32_layout)() { return ws32_layout<DG_N>(); }
TileLayout DG_FN(tc_layout)(int nc) { return tc_layout<DG_N>(nc); }
size_t DG_FN(tc_ops_count)() { return TcCfg<DG_N>::OPS_FLOATS; }
void DG_FN(tc_ops)(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  tc_ops<DG_N>(Dr, Ds, Dt, L, out);
}
size_t DG_FN(ws32_ops_count)() { return 2 * Ws32Cfg<DG_N>::OPS_ONE; }
void DG_FN(ws32_ops)(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  ws32_ops<DG_N>(Dr, Ds, Dt, L, out);
}

TileLayout DG_FN(ws_layout)() { return ws_layout<DG_N>(); }

#ifdef DG_WS_PROFILE
void DG_FN(tc_dbg)(float* p) { tc_dbg_set(p); }
void DG_FN(ws_prof)(unsigned long long* out, int reset) {
  if (reset) {
    ws_prof_reset();
    tc_prof_reset();
  } else {
    ws_prof_read(out);
    tc_prof_read(out + 16);  // TC-kernel counters follow the WS ones
  }
}
#endif

}  // namespace dg
