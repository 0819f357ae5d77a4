// Probe: does the multi-rank stage structure of dg_api.cu work inside a
// captured CUDA graph?  Compute stream: record fork -> persistent "stage" kernel that, after
// its first tiles, adds their count to a counter (release) and then keeps working.  Comm
// stream: wait fork -> cuStreamWaitValue32(counter >= n) -> cuStreamWriteValue32(counter, 0)
// -> "pack" kernel that copies the boundary outputs -> record join; compute waits join.
// The graph is replayed R times; every replay must see the pack read complete boundary data
// and the counter must be 0 again at the end.  It also times the replay with and without the
// comm branch.  Nothing in this probe spins on a flag inside a kernel.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/memop_graph_probe tools/memop_graph_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("{\"err\": \"%s: %s\"}\n", #x, cudaGetErrorString(e));                   \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

__global__ void stage(float* out, unsigned* sig, int nbt, int ntiles, int iter, int work) {
  // tile t = blockIdx.x + j * gridDim.x; boundary tiles first
  const int nb = nbt > int(blockIdx.x) ? (nbt - int(blockIdx.x) + gridDim.x - 1) / gridDim.x : 0;
  for (int j = 0;; ++j) {
    const int t = blockIdx.x + j * gridDim.x;
    if (t >= ntiles) break;
    float v = float(iter) + t;
    for (int w = 0; w < work; ++w) v = v * 1.0000001f + 1e-7f;
    out[t * blockDim.x + threadIdx.x] = float(iter) + t + (v - v);
    if (sig && j == nb - 1) {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(sig, unsigned(nb));
      }
    }
  }
}

__global__ void pack(const float* out, float* sent, int nbt, int iter, int* bad) {
  for (int t = blockIdx.x; t < nbt; t += gridDim.x) {
    const float v = out[t * blockDim.x + threadIdx.x];
    sent[t * blockDim.x + threadIdx.x] = v;
    if (v != float(iter) + t) atomicAdd(bad, 1);
  }
}

int main() {
  using W = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  void* f1 = nullptr;
  void* f2 = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f1, 12000, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f2, 12000, cudaEnableDefault, &q));
  W wait32 = reinterpret_cast<W>(f1), write32 = reinterpret_cast<W>(f2);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int ntiles = 40 * sms, nbt = 300, T = 256, R = 50;
  float *out, *sent;
  unsigned* sig;
  int* bad;
  CK(cudaMalloc(&out, size_t(ntiles) * T * 4));
  CK(cudaMalloc(&sent, size_t(nbt) * T * 4));
  CK(cudaMalloc(&sig, 4));
  CK(cudaMalloc(&bad, 4));
  CK(cudaMemset(sig, 0, 4));
  CK(cudaMemset(bad, 0, 4));
  cudaStream_t st, comm;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&comm, cudaStreamNonBlocking));
  cudaEvent_t fork, join, t0, t1;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  // stage k of replay r writes iteration value 5 r + k (baked into the graph of replay r)
  double ms[2] = {0, 0};
  for (int with_comm = 0; with_comm < 2; ++with_comm) {
    cudaGraphExec_t ge[R];
    for (int r = 0; r < R; ++r) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < 5; ++k) {
        const int iter = 5 * r + k;
        if (with_comm) CK(cudaEventRecord(fork, st));
        stage<<<sms - 4, T, 0, st>>>(out, with_comm ? sig : nullptr, nbt, ntiles, iter, 2000);
        if (with_comm) {
          CK(cudaStreamWaitEvent(comm, fork, 0));
          if (wait32(CUstream(comm), CUdeviceptr(reinterpret_cast<uintptr_t>(sig)), cuuint32_t(nbt),
                     CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS ||
              write32(CUstream(comm), CUdeviceptr(reinterpret_cast<uintptr_t>(sig)), 0u,
                      CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
            printf("{\"err\": \"stream memop capture failed\"}\n");
            return 1;
          }
          pack<<<4, T, 0, comm>>>(out, sent, nbt, iter, bad);
          CK(cudaEventRecord(join, comm));
          CK(cudaStreamWaitEvent(st, join, 0));
        }
      }
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&ge[r], g, 0));
      CK(cudaGraphDestroy(g));
    }
    CK(cudaGraphLaunch(ge[0], st));  // warm-up
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(t0, st));
    for (int r = 0; r < R; ++r) CK(cudaGraphLaunch(ge[r], st));
    CK(cudaEventRecord(t1, st));
    CK(cudaStreamSynchronize(st));
    float el = 0;
    CK(cudaEventElapsedTime(&el, t0, t1));
    ms[with_comm] = el / R / 5;
    for (int r = 0; r < R; ++r) CK(cudaGraphExecDestroy(ge[r]));
  }
  int hbad = -1;
  unsigned hsig = 99;
  CK(cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&hsig, sig, 4, cudaMemcpyDeviceToHost));
  printf("{\"probe\": \"memop_graph\", \"sms\": %d, \"ntiles\": %d, \"boundary_tiles\": %d, \"stages\": %d, "
         "\"bad_values\": %d, \"counter_after\": %u, \"ms_per_stage_no_comm\": %.4f, \"ms_per_stage_comm\": %.4f}\n",
         sms, ntiles, nbt, 5 * R, hbad, hsig, ms[0], ms[1]);
  return hbad == 0 && hsig == 0 ? 0 : 2;
}
