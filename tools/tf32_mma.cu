// Legacy warp-level TF32 MMA (mma.sync.m16n8k8, SASS HMMA) throughput on B200,
// alone and concurrently with FFMA warps.  Prints JSON lines.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k(float* out, long long* cyc, int iters, int mma_warps, int fma_on) {
  const int warp = threadIdx.x >> 5;
  float s = 0;
  long long t0 = clock64();
  if (warp < mma_warps) {
    unsigned a0 = __float_as_uint(1.0f + threadIdx.x * 1e-3f), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    unsigned b0 = __float_as_uint(0.5f), b1 = b0 + 7;
    float c[4][4] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  } else if (fma_on) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], 0.999999f, 1e-7f);
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  long long t1 = clock64();
  if (s == -1.2345f) out[0] = s;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}

int main() {
  float* d;
  long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 148 * 32 * sizeof(long long));
  long long h[32];
  const int iters = 4096;
  int cfgs[][3] = {{4, 4, 0}, {8, 8, 0}, {16, 16, 0}, {8, 12, 1}};  // mma warps, total warps, fma on
  for (auto& cf : cfgs) {
    const int mw = cf[0], tw = cf[1], fo = cf[2];
    k<<<148, 32 * tw>>>(d, c, iters, mw, fo);
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double mc = 0, fc = 0;
    for (int w = 0; w < mw; ++w) mc += h[w] / double(mw);
    for (int w = mw; w < tw; ++w) fc += h[w] / double(tw - mw);
    // per SM: mw warps x iters x 4 mma x (16*8*8=1024 FMA)
    printf("{\"mma_warps\": %d, \"fma_warps\": %d, \"tf32_fma_per_clk_sm\": %.1f, \"ffma_per_clk_sm\": %.1f}\n", mw,
           tw - mw, mw * double(iters) * 4 * 1024 / mc, fo ? (tw - mw) * double(iters) * 8 * 32 / fc : 0.0);
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
