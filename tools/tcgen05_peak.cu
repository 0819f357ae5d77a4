// tcgen05.mma kind::tf32 throughput on B200: the denominator of the FP32 tensor
// roofline (3xTF32 effective = this / 3).  One persistent CTA per SM; one thread
// issues back-to-back tcgen05.mma.cta_group::1.kind::tf32 (K = 8 per instruction)
// on shared-memory operands (K-major SWIZZLE_NONE, the layout the TC stage kernel
// uses) into a TMEM accumulator, commits to an mbarrier at the end.  Shapes: M = 128
// at the N the stage kernel uses per order (NP16 = 16, 32, 48, 64, 96, 128, 176, 224)
// plus N = 256, and M = 64.  Prints one JSON object.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcgen05_peak tcgen05_peak.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc(const void* smem, unsigned lbo, unsigned sbo) {
  uint64_t d = uint64_t((su32(smem) >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

template <int M, int N, int NACC>
__global__ void __launch_bounds__(128, 1) peak(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = reinterpret_cast<float*>(sm);    // [M rows x 8 k] per chunk, 4 chunks
  float* sB = sA + 4 * 128 * 8;               // [N rows x 8 k] per chunk, 4 chunks
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 4 * (128 + 256) * 8; i += blockDim.x) sA[i] = 1e-3f * (i & 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    constexpr uint32_t id = idesc_tf32(M, N);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t da = desc(sA + q * 128 * 8, 128, 256), db = desc(sB + q * 256 * 8, 128, 256);
        const uint32_t acc = (it > 0 || q >= NACC) ? 1u : 0u;
        const uint32_t dcol = uint32_t((q % NACC) * N);  // NACC independent accumulators, round robin
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + dcol),
            "l"(da), "l"(db), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W;\n}\n" ::"r"(su32(&bar)));
    if (blockIdx.x == 0) *cyc = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int M, int N, int NACC = 1>
void run(int sms, unsigned long long* dcyc, bool last) {
  const int smem = 4 * (128 + 256) * 8 * 4;
  cudaFuncSetAttribute(peak<M, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  peak<M, N, NACC><<<sms, 128, smem>>>(100, dcyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  peak<M, N, NACC><<<sms, 128, smem>>>(iters, dcyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  const double mmas = double(iters) * 4;
  const double flop = double(sms) * mmas * M * N * 8 * 2;
  printf("{\"M\": %d, \"N\": %d, \"accumulators\": %d, \"tflops\": %.1f, \"cycles_per_mma\": %.2f, \"err\": \"%s\"}%s\n", M, N, NACC,
         flop / (ms * 1e-3) / 1e12, double(cyc) / mmas, cudaGetErrorString(cudaGetLastError()), last ? "" : ",");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 8);
  printf("{\"kind\": \"tf32\", \"sms\": %d, \"shapes\": [\n", sms);
  run<128, 16>(sms, dcyc, false);
  run<128, 32>(sms, dcyc, false);
  run<128, 48>(sms, dcyc, false);
  run<128, 64>(sms, dcyc, false);
  run<128, 96>(sms, dcyc, false);
  run<128, 128>(sms, dcyc, false);
  run<128, 176>(sms, dcyc, false);
  run<128, 224>(sms, dcyc, false);
  run<128, 256>(sms, dcyc, false);
  run<64, 256>(sms, dcyc, false);
  // independent accumulators (round robin over NACC TMEM column ranges): the small-N floor
  run<128, 16, 2>(sms, dcyc, false);
  run<128, 16, 4>(sms, dcyc, false);
  run<128, 48, 2>(sms, dcyc, false);
  run<128, 48, 4>(sms, dcyc, false);
  run<128, 64, 2>(sms, dcyc, false);
  run<128, 96, 2>(sms, dcyc, true);
  printf("]}\n");
  return 0;
}
