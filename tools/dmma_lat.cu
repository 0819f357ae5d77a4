// DMMA.8x8x4 latency / issue characteristics on B200: cycles per DMMA for
// (warps per SM) x (independent accumulator chains per warp).  Prints JSON lines.
#include <cuda_runtime.h>
#include <cstdio>

template <int CH>
__global__ void chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps, double* d, long long* dc) {
  const int iters = 4096;
  chain<CH><<<1, 32 * warps>>>(d, dc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per = double(c) / (double(iters) * CH);  // cycles per DMMA per warp
  printf("{\"warps\": %d, \"chains\": %d, \"cyc_per_dmma_per_warp\": %.2f, \"sm_fma_per_clk\": %.1f}\n", warps, CH,
         per, 256.0 * warps / per);
}

int main() {
  double* d;
  long long* dc;
  cudaMalloc(&d, 64);
  cudaMalloc(&dc, 64 * sizeof(long long));
  for (int w : {1, 2, 4, 8, 16}) {
    run<1>(w, d, dc);
    run<2>(w, d, dc);
    run<3>(w, d, dc);
    run<4>(w, d, dc);
    run<6>(w, d, dc);
    run<9>(w, d, dc);
  }
  return 0;
}
