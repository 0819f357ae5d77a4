// tcgen05 contention probe (TC stage kernel diagnosis, DESIGN.md §8 "TC kernel"): cycles per
// kind::tf32 TS-mode MMA (M = 128, N = 48 as at N = 4, A in tensor memory, B in shared memory)
// issued back to back by one thread, while other warps of the same CTA concurrently
//   st: 4 warps tcgen05.st 32x32b.x16 into other TMEM columns (the operand writers' traffic)
//   ld: 4 warps tcgen05.ld 32x32b.x16 from other TMEM columns (the epilogue's traffic)
//   cm: the issuing thread also commits to an mbarrier every 6 MMAs (the kernel's pattern:
//       3 MMAs per 8-k chunk, one commit per two chunks)
// One CTA per SM on every SM.  Prints one JSON line per configuration.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tcgen05_contention_probe tools/tcgen05_contention_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(const void* smem) {
  uint64_t d = uint64_t((su32(smem) >> 4) & 0x3FFF);
  d |= uint64_t(128 >> 4) << 16;
  d |= uint64_t(256 >> 4) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(288, 1) probe(int iters, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sB = reinterpret_cast<float*>(sm);  // [4 chunks][N x 8] (values irrelevant: timing only)
  __shared__ uint64_t bar, cbar, fbar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int w = tid; w < 4 * N * 8; w += blockDim.x) sB[w] = 0.5f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&fbar)));  // phase 0 pending: parity 1 passes
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const bool st_on = mode & 1, ld_on = mode & 2, cm_on = mode & 4;
  if (warp == 0) {
    if (lane == 0) {
      const long long t0 = clock64();
      constexpr uint32_t id = idesc_tf32(128, N);
      for (int it = 0; it < iters; ++it) {
        for (int q = 0; q < 6; ++q) {
          if ((mode & 8) && q % 3 == 0) {  // the stage kernel's per-chunk pattern: wait (already complete) + fence
            asm volatile(
                "{\n.reg .pred P1;\nWF_%=:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1;\n"
                "@!P1 bra WF_%=;\n}\n" ::"r"(su32(&fbar)));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          if ((mode & 16) && q % 3 == 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
              "r"(tmem + 256 + 8 * (q & 3)), "l"(desc(sB + (q & 3) * N * 8)), "r"(id), "r"((it | q) ? 1u : 0u));
        }
        if (cm_on)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&cbar))
                       : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
      asm volatile(
          "{\n.reg .pred P1;\nW:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
          "@!P1 bra W;\n}\n" ::"r"(su32(&bar)));
      if (blockIdx.x == 0) *cyc = clock64() - t0;
      done = 1;
    }
  } else if (warp >= 1 && warp <= 4) {
    if (st_on) {  // operand-writer traffic: lane quarter (warp % 4), 16 columns per store, columns 320..447
      const uint32_t row = uint32_t(32 * (warp & 3)) << 16;
      uint32_t v[16];
      for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(float(lane + i));
      int c = 0;
      while (!done) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                tmem + row + 320 + 16 * (c & 7)),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
            "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
        if ((++c % 3) == 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  } else {
    if (ld_on) {  // epilogue traffic: columns 64..127
      const uint32_t row = uint32_t(32 * (warp & 3)) << 16;
      uint32_t acc = 0;
      int c = 0;
      while (!done) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + row + 64 + 16 * (c & 3)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) acc += v[i];
        ++c;
      }
      if (acc == 0x12345678u) *cyc = 0;  // keep the loads
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  constexpr int N = 48;
  const int smem = 4 * 256 * 8 * 4;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[32] = {"alone", "st", "ld", "st+ld", "commit", "st+commit", "ld+commit", "st+ld+commit"};
  names[8] = "wait+fence per 3 MMAs";
  names[12] = "commit+wait+fence";
  names[16] = "fence per 3 MMAs";
  names[23] = "st+ld+commit+fence";
  const int iters = 4000;
  const int modes[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 23};
  for (int mode : modes) {
    probe<N><<<sms, 288, smem>>>(iters, mode, dc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\": \"tcgen05_contention\", \"N\": %d, \"config\": \"%s\", \"err\": \"%s\", \"cycles_per_mma\": %.2f}\n",
           N, names[mode], cudaGetErrorString(e), double(cyc) / (6.0 * iters));
  }
  return 0;
}
