// Stage-kernel instantiations for order N=4 (stage_basic.cuh, stage_mma.cuh, stage_ws.cuh).
#include "stage_tc.cuh"

#include "stage_ffma.cuh"

namespace dg {

void launch_stage_f64_N4(const StageParams<double>& p, int mode, int variant, void* st) {
  if (variant == 1)       // DG_VARIANT_BASIC
    launch_stage_basic<double, 4>(p, mode, static_cast<cudaStream_t>(st));
  else if (variant == 6)  // DG_VARIANT_FFMA: register-tiled DFMA WS kernel
    launch_stage_ffma<double, 4>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else if (variant == 2)  // DG_VARIANT_MMA: DMMA, cp.async-pipelined, element-major layout
    launch_stage_mma<4>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else                    // AUTO / DG_VARIANT_MMA_WS: DMMA, warp-specialized TMA pipeline, tiled layout
    launch_stage_ws<4>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

void launch_stage_f32_N4(const StageParams<float>& p, int mode, int variant, void* st) {
  if (variant == 1 || variant == 2)  // BASIC (MMA has no FP32 kernel of its own)
    launch_stage_basic<float, 4>(p, mode, static_cast<cudaStream_t>(st));
  else if (variant == 6)             // FFMA: register-tiled FFMA WS kernel
    launch_stage_ffma<float, 4>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else if (variant == 4)             // TC: tcgen05 kind::tf32 (3xTF32), TMEM accumulators
    launch_stage_tc<4>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else                               // MMA_WS: 3xTF32 mma.sync WS kernel
    launch_stage_ws32<4>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

TileLayout ffma_layout_N4() { return ffma_layout<float, 4>(); }
size_t ffma_ops_count_N4() { return FfCfg<float, 4>::A_FLOATS; }
void ffma_ops_N4(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  ffma_ops<float, 4>(Dr, Ds, Dt, L, out);
}
TileLayout ffma64_layout_N4() { return ffma_layout<double, 4>(); }
size_t ffma64_ops_count_N4() { return FfCfg<double, 4>::A_FLOATS; }
void ffma64_ops_N4(const double* Dr, const double* Ds, const double* Dt, const double* L, double* out) {
  ffma_ops<double, 4>(Dr, Ds, Dt, L, out);
}
TileLayout ws32_layout_N4() { return ws32_layout<4>(); }
TileLayout tc_layout_N4() { return tc_layout<4>(); }
size_t tc_ops_count_N4() { return TcCfg<4>::OPS_FLOATS; }
void tc_ops_N4(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  tc_ops<4>(Dr, Ds, Dt, L, out);
}
size_t ws32_ops_count_N4() { return 2 * Ws32Cfg<4>::OPS_ONE; }
void ws32_ops_N4(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  ws32_ops<4>(Dr, Ds, Dt, L, out);
}

TileLayout ws_layout_N4() { return ws_layout<4>(); }
bool launch_fused_f64_N4(const StageParams<double>& p, const FusedParams<double>& fp, void* st) {
  return launch_stage_ws_fused<4>(p, p.ops_pad, fp, static_cast<cudaStream_t>(st));
}

#ifdef DG_WS_PROFILE
void ws_prof_N4(unsigned long long* out, int reset) {
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
