// Stage-kernel instantiations for order N=2 (stage_basic.cuh, stage_mma.cuh).
#include "stage_mma.cuh"

namespace dg {

void launch_stage_f64_N2(const StageParams<double>& p, int mode, int variant, void* st) {
  if (variant == 1)  // DG_VARIANT_BASIC
    launch_stage_basic<double, 2>(p, mode, static_cast<cudaStream_t>(st));
  else               // AUTO / MMA: FP64 tensor-core (DMMA) contractions
    launch_stage_mma<2>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

void launch_stage_f32_N2(const StageParams<float>& p, int mode, int variant, void* st) {
  (void)variant;
  launch_stage_basic<float, 2>(p, mode, static_cast<cudaStream_t>(st));
}

size_t ops_pad_doubles_N2() { return MmaCfg<2>::OPS_DOUBLES; }

}  // namespace dg
