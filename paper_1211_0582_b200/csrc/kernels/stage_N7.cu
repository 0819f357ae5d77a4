// Stage-kernel instantiations for order N=7 (see stage_basic.cuh).
#include "stage_basic.cuh"

namespace dg {

void launch_stage_f64_N7(const StageParams<double>& p, int mode, int variant, void* st) {
  (void)variant;
  launch_stage_basic<double, 7>(p, mode, static_cast<cudaStream_t>(st));
}

void launch_stage_f32_N7(const StageParams<float>& p, int mode, int variant, void* st) {
  (void)variant;
  launch_stage_basic<float, 7>(p, mode, static_cast<cudaStream_t>(st));
}

}  // namespace dg
