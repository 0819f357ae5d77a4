// Measures the B200's FP64 DFMA, FP32 FFMA and FP64 DMMA (mma.sync m8n8k4)
// throughput with long dependent-chain-free loops, so the roofline denominators
// for the ALU-bound stage kernels are measured rather than taken from a
// datasheet.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peaks alu_peaks.cu
// Prints one JSON object.
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ILP = 8;

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = T(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == T(-1.2345)) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

template <typename K>
float time_kernel(K launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 64);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  const double nthr = double(blocks) * threads;
  float ms64 = time_kernel([&] { fma_loop<double><<<blocks, threads>>>(d, iters, 0.999999, 1e-7); });
  float ms32 = time_kernel([&] { fma_loop<float><<<blocks, threads>>>((float*)d, iters, 0.999999f, 1e-7f); });
  float msmm = time_kernel([&] { dmma_loop<<<blocks, threads>>>(d, iters / 4); });
  const double f64 = nthr * iters * ILP * 2 / (ms64 * 1e-3) / 1e12;
  const double f32 = nthr * iters * ILP * 2 / (ms32 * 1e-3) / 1e12;
  // one m8n8k4 per warp = 8*8*4 = 256 FMA = 512 flop
  const double fmm = (nthr / 32) * (iters / 4) * ILP * 512.0 / (msmm * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"fp64_dfma_tflops\": %.3f, \"fp32_ffma_tflops\": %.3f, "
         "\"fp64_dmma_tflops\": %.3f, \"err\": \"%s\"}\n",
         sms, clk / 1000, f64, f32, fmm, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
