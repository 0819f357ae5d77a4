// tcgen05 "TS" probe: D[128 x N] = A[128 x K] . B[K x N], kind::tf32, with A in TENSOR
// memory (written by the 4 warps of the CTA with tcgen05.st.32x32b: lane = row,
// column = k, one 32-bit column per tf32 element) and B in shared memory (K-major
// SWIZZLE_NONE canonical 8-k chunks, LBO 128 B, SBO 256 B).  Checks the numerics against
// a host reference with truncated-TF32 operands, then times back-to-back TS MMAs
// against the same shape in SS mode.  Prints JSON lines.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcgen05_ts_probe tcgen05_ts_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

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
__host__ __device__ constexpr int cm(int r, int kk) { return ((r >> 3) * 2 + (kk >> 2)) * 32 + (r & 7) * 4 + (kk & 3); }

constexpr int K = 32;  // 4 chunks of 8
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(const float* A, const float* B, float* D, int iters,
                                                 unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = reinterpret_cast<float*>(sm);   // SS mode: [4 chunks][128 x 8]
  float* sB = sA + 4 * 128 * 8;               // [4 chunks][N x 8]
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int w = tid; w < 128 * K; w += 128) {
    const int r = w / K, k = w % K;
    sA[(k / 8) * 1024 + cm(r, k % 8)] = A[w];
  }
  for (int w = tid; w < N * K; w += 128) {
    const int n = w / K, k = w % K;
    sB[(k / 8) * (N * 8) + cm(n, k % 8)] = B[w];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t acol = 256;  // A at columns 256.. (k = column offset)
  {
    // warp w writes lanes 32w..32w+31: row = lane, 32 columns = k
    const int r = 32 * warp + lane;
    uint32_t v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(A[r * K + k]);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + (uint32_t(32 * warp) << 16) + acol),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const long long t0 = clock64();
    constexpr uint32_t id = idesc_tf32(128, N);
    for (int it = 0; it < iters; ++it)
      for (int q = 0; q < 4; ++q) {
        const uint32_t acc = (it | q) ? 1u : 0u;
        if (TS) {
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
              "r"(tmem + acol + 8 * q), "l"(desc(sB + q * N * 8)), "r"(id), "r"(acc));
        } else {
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(desc(sA + q * 1024)), "l"(desc(sB + q * N * 8)), "r"(id), "r"(acc));
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
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (blockIdx.x == 0 && iters == 1) {
    const int r = 32 * warp + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + (uint32_t(32 * warp) << 16) + uint32_t(c0)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 8; ++i) D[r * N + c0 + i] = __uint_as_float(v[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

static float trunc_tf32(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

template <int N, bool TS>
void run() {
  std::vector<float> A(128 * K), B(N * K), D(128 * N);
  unsigned s = 4242;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float((s >> 8) & 0xffff) / 65536.0f) * 2.0f - 1.0f; };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dD;
  unsigned long long* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (4 * 128 * 8 + 4 * 256 * 8) * 4;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, TS><<<1, 128, smem>>>(dA, dB, dD, 1, dc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += double(trunc_tf32(A[m * K + k])) * trunc_tf32(B[n * K + k]);
      err = std::fmax(err, std::fabs(r - D[m * N + n]));
      mx = std::fmax(mx, std::fabs(r));
    }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<N, TS><<<sms, 128, smem>>>(dA, dB, dD, iters, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  const double mmas = double(iters) * 4;
  printf("{\"mode\": \"%s\", \"N\": %d, \"err\": \"%s\", \"maxabs\": %.3g, \"err_vs_trunc_tf32\": %.3g, \"tflops\": %.1f, "
         "\"cycles_per_mma\": %.2f}\n",
         TS ? "TS (A in TMEM)" : "SS", N, cudaGetErrorString(e), mx, err,
         double(sms) * mmas * 128 * N * 8 * 2 / (ms * 1e-3) / 1e12, double(cyc) / mmas);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}


// Canary: does an MMA with D at columns [0, N) write TMEM columns >= N?  Columns N..N+63
// are filled with 12345.0 by tcgen05.st before the MMA and read back after it.
template <int N>
__global__ void __launch_bounds__(128, 1) canary(const float* A, const float* B, int* changed) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sB = reinterpret_cast<float*>(sm);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int w = tid; w < N * 8; w += 128) sB[cm(w / 8, w % 8)] = B[w];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t lrow = uint32_t(32 * warp) << 16;
  {
    uint32_t v[8];
    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(A[(32 * warp + lane) * 8 + k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + 448),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    const uint32_t c = __float_as_uint(12345.0f);
    for (int c0 = N; c0 < N + 64 && c0 < 448; c0 += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + c0),
                   "r"(c), "r"(c), "r"(c), "r"(c), "r"(c), "r"(c), "r"(c), "r"(c));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
        "r"(tmem + 448), "l"(desc(sB)), "r"(idesc_tf32(128, N)), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW2:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@!P1 bra W2;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  int bad = 0;
  for (int c0 = N; c0 < N + 64 && c0 < 448; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + lrow + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i)
      if (__uint_as_float(v[i]) != 12345.0f) bad = max(bad, c0 + i - N + 1);
  }
  atomicMax(changed, bad);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int N>
void run_canary() {
  std::vector<float> A(128 * 8, 0.5f), B(N * 8, 0.25f);
  float *dA, *dB;
  int* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dc, 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dc, 0, 4);
  cudaFuncSetAttribute(canary<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  canary<N><<<1, 128, 64 * 1024>>>(dA, dB, dc);
  cudaError_t e = cudaDeviceSynchronize();
  int c = 0;
  cudaMemcpy(&c, dc, 4, cudaMemcpyDeviceToHost);
  printf("{\"canary_N\": %d, \"err\": \"%s\", \"columns_written_beyond_N\": %d}\n", N, cudaGetErrorString(e), c);
  cudaFree(dA); cudaFree(dB); cudaFree(dc);
}

// Issue-path cost: per "chunk" 3 TS MMAs (K=8) then, optionally, tcgen05.fence::after_thread_sync
// and a tcgen05.commit to an mbarrier (as the stage kernel's MMA warp does).
template <int N, bool FENCE, bool COMMIT>
__global__ void __launch_bounds__(128, 1) issue_cost(int chunks, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sB = reinterpret_cast<float*>(sm);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int w = tid; w < 2 * N * 8; w += 128) sB[w] = 1e-3f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const long long t0 = clock64();
    constexpr uint32_t id = idesc_tf32(128, N);
    for (int c = 0; c < chunks; ++c) {
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ta = tmem + 256 + 16 * (c & 7);
      const uint64_t db = desc(sB), dbl = desc(sB + N * 8);
      const uint32_t acc = c ? 1u : 0u;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                   ::"r"(tmem), "r"(ta), "l"(db), "r"(id), "r"(acc));
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                   ::"r"(tmem), "r"(ta + 8), "l"(db), "r"(id), "r"(1u));
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                   ::"r"(tmem), "r"(ta), "l"(dbl), "r"(id), "r"(1u));
      if (COMMIT)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1]))
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0]))
                 : "memory");
    asm volatile("{\n.reg .pred P1;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W3;\n}\n" ::"r"(su32(&bar[0])));
    if (blockIdx.x == 0) *cyc = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int N, bool FENCE, bool COMMIT>
void run_issue() {
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  cudaFuncSetAttribute(issue_cost<N, FENCE, COMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int chunks = 4000;
  issue_cost<N, FENCE, COMMIT><<<148, 128, 64 * 1024>>>(chunks, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("{\"issue_N\": %d, \"fence\": %d, \"commit\": %d, \"err\": \"%s\", \"cycles_per_chunk_of_3_mma\": %.1f}\n", N, FENCE,
         COMMIT, cudaGetErrorString(e), double(c) / chunks);
  cudaFree(dc);
}

int main() {
  run_issue<48, false, false>();
  run_issue<48, true, false>();
  run_issue<48, false, true>();
  run_issue<48, true, true>();
  run_issue<224, false, false>();
  run_issue<224, true, true>();
  return 0;
  run_canary<48>();
  run_canary<80>();
  run_canary<96>();
  run_canary<112>();
  run_canary<128>();
  run_canary<144>();
  run_canary<176>();
  run_canary<224>();
  return 0;
  run<48, true>();
  run<48, false>();
  run<16, true>();
  run<16, false>();
  run<128, true>();
  run<224, true>();
  run<224, false>();
  return 0;
}
