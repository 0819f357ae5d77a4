// tcgen05 (5th-gen tensor core) probe on B200: D[128 x N] = A[128 x K] . B[K x N]
// with kind::tf32, operands in shared memory in the K-major SWIZZLE_NONE canonical
// layout (8-row x 16-byte core matrices), accumulator in TMEM, one thread issuing
// tcgen05.mma, tcgen05.commit -> mbarrier, tcgen05.ld.32x32b epilogue.
// Checks 1xTF32 (hardware conversion: truncation or rounding?) and 3xTF32
// (A_hi.B + A_hi.B_lo + A_lo.B) against an FP64 host reference.  Prints JSON.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

constexpr int M = 128;  // rows of the A buffers (the M=64 probe uses the first 64)

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// element (r, k) of a rows x K K-major operand in the SWIZZLE_NONE canonical layout:
// core matrix (r/8, k/4) of 8 rows x 4 floats (128 B) at ((r/8)*(K/4) + k/4)*32 floats.
__host__ __device__ inline int cm_off(int r, int k, int K) { return ((r >> 3) * (K >> 2) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }

__device__ __forceinline__ uint64_t umma_desc(const void* smem, unsigned lbo_bytes, unsigned sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((su32(smem) >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)                  // c_format F32
         | (2u << 7)                // a_format TF32
         | (2u << 10)               // b_format TF32
         | (0u << 15) | (0u << 16)  // a, b K-major
         | (uint32_t(n >> 3) << 17) // N / 8
         | (uint32_t(m >> 4) << 24);// M / 16
}

template <int N, int K, int PASSES, int MM = 128>
__global__ void probe(const float* A, const float* Alo, const float* B, const float* Blo, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = reinterpret_cast<float*>(sm);
  float* sAl = sA + M * K;
  float* sB = sAl + M * K;
  float* sBl = sB + N * K;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int w = tid; w < M * K; w += blockDim.x) {
    const int r = w / K, k = w % K;
    sA[cm_off(r, k, K)] = A[w];
    sAl[cm_off(r, k, K)] = Alo[w];
  }
  for (int w = tid; w < N * K; w += blockDim.x) {  // B given as [N][K]
    const int r = w / K, k = w % K;
    sB[cm_off(r, k, K)] = B[w];
    sBl[cm_off(r, k, K)] = Blo[w];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(MM, N);
    for (int pass = 0; pass < PASSES; ++pass) {
      const float* a = pass == 1 ? sAl : sA;  // pass 0: A.B, 1: Alo.B, 2: A.Blo
      const float* b = pass == 2 ? sBl : sB;
      for (int kk = 0; kk < K; kk += 8) {
        const uint64_t da = umma_desc(a + (kk >> 2) * 32, 128, (K / 4) * 128);
        const uint64_t db = umma_desc(b + (kk >> 2) * 32, 128, (K / 4) * 128);
        const uint32_t acc = (pass > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n.reg .pred P1;\nWAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@!P1 bra WAIT;\n}\n" ::"r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (row = lane), 8 columns at a time
  const int row = 32 * warp + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + (uint32_t(32 * warp) << 16) + uint32_t(c0);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) D[row * N + c0 + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

static float trunc_tf32(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
static float rna_tf32(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

template <int N, int K>
void run() {
  std::vector<float> A(M * K), B(N * K), Al(M * K), Bl(N * K), D(M * N);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float((s >> 8) & 0xffff) / 65536.0f) * 2.0f - 1.0f; };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  // 3xTF32 split: hi = the raw value (hardware takes its TF32 part), lo = x - trunc(x)
  for (int i = 0; i < M * K; ++i) Al[i] = A[i] - trunc_tf32(A[i]);
  for (int i = 0; i < N * K; ++i) Bl[i] = B[i] - trunc_tf32(B[i]);
  float *dA, *dB, *dAl, *dBl, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dAl, Al.size() * 4);
  cudaMalloc(&dBl, Bl.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dAl, Al.data(), Al.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dBl, Bl.data(), Bl.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (2 * M * K + 2 * N * K) * 4;
  for (int passes : {1, 3}) {
    if (passes == 1) {
      cudaFuncSetAttribute(probe<N, K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      probe<N, K, 1><<<1, 128, smem>>>(dA, dAl, dB, dBl, dD);
    } else {
      cudaFuncSetAttribute(probe<N, K, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      probe<N, K, 3><<<1, 128, smem>>>(dA, dAl, dB, dBl, dD);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double ex = 0, et = 0, er = 0, mx = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double full = 0, tr = 0, rn = 0;
        for (int k = 0; k < K; ++k) {
          full += double(A[m * K + k]) * B[n * K + k];
          tr += double(trunc_tf32(A[m * K + k])) * trunc_tf32(B[n * K + k]);
          rn += double(rna_tf32(A[m * K + k])) * rna_tf32(B[n * K + k]);
        }
        const double d = D[m * N + n];
        ex = std::fmax(ex, std::fabs(d - full));
        et = std::fmax(et, std::fabs(d - tr));
        er = std::fmax(er, std::fabs(d - rn));
        mx = std::fmax(mx, std::fabs(full));
      }
    printf("{\"N\": %d, \"K\": %d, \"passes\": %d, \"err\": \"%s\", \"maxabs\": %.3g, \"err_vs_fp64\": %.3g, "
           "\"err_vs_trunc_tf32\": %.3g, \"err_vs_rna_tf32\": %.3g}\n",
           N, K, passes, cudaGetErrorString(e), mx, ex, et, er);
  }
  cudaFree(dA); cudaFree(dB); cudaFree(dAl); cudaFree(dBl); cudaFree(dD);
}

// M=64: which TMEM lanes hold which rows?  Reads all 128 lanes and matches them to rows.
void run_m64() {
  constexpr int N = 48, K = 40;
  std::vector<float> A(M * K), B(N * K), Z(M * K, 0.0f), D(M * N);
  unsigned s = 777;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float((s >> 8) & 0xffff) / 65536.0f) * 2.0f - 1.0f; };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dZ, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dZ, Z.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), Z.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  const int smem = (2 * M * K + 2 * N * K) * 4;
  cudaFuncSetAttribute(probe<N, K, 1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, K, 1, 64><<<1, 128, smem>>>(dA, dZ, dB, dZ, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  printf("{\"M\": 64, \"err\": \"%s\", \"lane_to_row\": [", cudaGetErrorString(e));
  for (int lane = 0; lane < 128; ++lane) {
    int match = -1;
    for (int m = 0; m < 64 && match < 0; ++m) {
      double md = 0;
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += double(trunc_tf32(A[m * K + k])) * trunc_tf32(B[n * K + k]);
        md = std::fmax(md, std::fabs(r - D[lane * N + n]));
      }
      if (md < 1e-4) match = m;
    }
    printf("%s%d", lane ? "," : "", match);
  }
  printf("]}\n");
}

int main() {
  run_m64();
  run<96, 40>();
  run<144, 40>();
  run<256, 64>();
  return 0;
}
