// Stage-kernel instantiations for order N=6 (stage_basic.cuh, stage_mma.cuh, stage_ws.cuh).
#include "stage_ws32.cuh"

#include "stage_ffma.cuh"

namespace dg {

void launch_stage_f64_N6(const StageParams<double>& p, int mode, int variant, void* st) {
  if (variant == 1)       // DG_VARIANT_BASIC
    launch_stage_basic<double, 6>(p, mode, static_cast<cudaStream_t>(st));
  else if (variant == 6)  // DG_VARIANT_FFMA: register-tiled DFMA WS kernel
    launch_stage_ffma<double, 6>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else if (variant == 2)  // DG_VARIANT_MMA: DMMA, cp.async-pipelined, element-major layout
    launch_stage_mma<6>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else                    // AUTO / DG_VARIANT_MMA_WS: DMMA, warp-specialized TMA pipeline, tiled layout
    launch_stage_ws<6>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

void launch_stage_f32_N6(const StageParams<float>& p, int mode, int variant, void* st) {
  if (variant == 1 || variant == 2)  // BASIC (MMA has no FP32 kernel of its own)
    launch_stage_basic<float, 6>(p, mode, static_cast<cudaStream_t>(st));
  else if (variant == 6)             // FFMA: register-tiled FFMA WS kernel
    launch_stage_ffma<float, 6>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
  else                               // AUTO / MMA_WS: 3xTF32 tensor-core WS kernel
    launch_stage_ws32<6>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

TileLayout ffma_layout_N6() { return ffma_layout<float, 6>(); }
size_t ffma_ops_count_N6() { return FfCfg<float, 6>::A_FLOATS; }
void ffma_ops_N6(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  ffma_ops<float, 6>(Dr, Ds, Dt, L, out);
}
TileLayout ffma64_layout_N6() { return ffma_layout<double, 6>(); }
size_t ffma64_ops_count_N6() { return FfCfg<double, 6>::A_FLOATS; }
void ffma64_ops_N6(const double* Dr, const double* Ds, const double* Dt, const double* L, double* out) {
  ffma_ops<double, 6>(Dr, Ds, Dt, L, out);
}
TileLayout ws32_layout_N6() { return ws32_layout<6>(); }
TileLayout tc_layout_N6() { return TileLayout{}; }  // TC covers N <= 4
size_t tc_ops_count_N6() { return 0; }
void tc_ops_N6(const double*, const double*, const double*, const double*, float*) {}
size_t ws32_ops_count_N6() { return 2 * Ws32Cfg<6>::OPS_ONE; }
void ws32_ops_N6(const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  ws32_ops<6>(Dr, Ds, Dt, L, out);
}

TileLayout ws_layout_N6() { return ws_layout<6>(); }
bool launch_fused_f64_N6(const StageParams<double>& p, const FusedParams<double>& fp, void* st) {
  return launch_stage_ws_fused<6>(p, p.ops_pad, fp, static_cast<cudaStream_t>(st));
}

#ifdef DG_WS_PROFILE
void ws_prof_N6(unsigned long long* out, int reset) {
  if (reset)
    ws_prof_reset();
  else
    ws_prof_read(out);
}
#endif

}  // namespace dg
