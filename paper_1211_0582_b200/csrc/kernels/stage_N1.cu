// Stage-kernel instantiations for order N=1 (stage_basic.cuh, stage_mma.cuh).
#include "stage_mma.cuh"

namespace dg {

void launch_stage_f64_N1(const StageParams<double>& p, int mode, int variant, void* st) {
  if (variant == 1)  // DG_VARIANT_BASIC
    launch_stage_basic<double, 1>(p, mode, static_cast<cudaStream_t>(st));
  else               // AUTO / MMA: FP64 tensor-core (DMMA) contractions
    launch_stage_mma<1>(p, p.ops_pad, mode, static_cast<cudaStream_t>(st));
}

void launch_stage_f32_N1(const StageParams<float>& p, int mode, int variant, void* st) {
  (void)variant;
  launch_stage_basic<float, 1>(p, mode, static_cast<cudaStream_t>(st));
}

size_t ops_pad_doubles_N1() { return MmaCfg<1>::OPS_DOUBLES; }

}  // namespace dg
