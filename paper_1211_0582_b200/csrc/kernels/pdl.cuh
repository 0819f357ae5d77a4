// Programmatic dependent launch (PDL) for the persistent stage kernels.
//
// Consecutive LSERK stages are a chain of launches on one stream; stage s+1 reads
// what stage s wrote (u_out, res, and every neighbour's trace), so it cannot start
// its tile loop early.  Its prologue — mbarrier init, TMEM allocation, the operator
// copy into shared memory — touches only constant data, so with PDL the CTAs of
// stage s+1 run it on each SM as soon as stage s's CTA there exits, and then block
// in griddepcontrol.wait until stage s has completed and its writes are visible.
// This hides the launch latency and prologue of every stage after the first.
//
// Kernels call pdl_trigger() at entry (all their CTAs are resident: grid <= #SMs)
// and pdl_wait() after the prologue, before the first global read of field data.
// Without the launch attribute both instructions are no-ops.  DG_PDL=0 in the
// environment disables the attribute (A/B measurements, profiles/r1_pdl_sweep.jsonl:
// +1.5..6 % on the WS / WS32 / TC kernels; the MMA kernel loses 4..8 % at N <= 2, where
// it keeps the plain launch).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

namespace dg {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const int v = [] {
    const char* e = std::getenv("DG_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(bool use, void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (use && pdl_enabled()) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// One-time launcher setup per device: cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is
// per device context, so a second solver on another device must run it again.
struct PerDevice {
  int sms[64] = {0};
};
template <typename F>
inline int sms_for_device(PerDevice& pd, F&& setup) {
  int dev = 0;
  cudaGetDevice(&dev);
  int& s = pd.sms[dev & 63];
  if (!s) {
    setup();
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  }
  return s;
}

}  // namespace dg
