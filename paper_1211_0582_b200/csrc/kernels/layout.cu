// Layout conversion between the C-ABI field layout [nc][K][Np] (nc = L.nc) (component-major,
// HW's Np x K per component) and the device element-tile layout [K][ES]
// (element-major, see stage_params.h).  Not on the timed device path; they run
// inside dg_fields_upload/download and dg_rhs.
#include <cuda_runtime.h>

#include <cstdint>

#include "stage_params.h"

namespace dg {

// [6][K][Np] (component-major) -> device layout L (padding and absent elements zeroed)
template <typename S, typename T>
__global__ void k_cm_to_tiles(const S* __restrict__ src, T* __restrict__ dst, int64_t K, int Np, TileLayout L) {
  const int64_t total = L.ntiles(K) * L.TS;
  const int cols = L.nc * L.E;
  for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < total; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = w / L.TS;
    const int64_t r = w - t * L.TS;
    int col, n;
    if (L.perm == 2) {  // inverse of the core-matrix placement
      const int chunk = int(r >> 5), q = int(r & 31), kc = L.LD >> 2;
      col = (chunk / kc) * 8 + (q >> 2);
      n = (chunk % kc) * 4 + (q & 3);
    } else if (L.perm == 3) {  // (c*LD + n)*E + e
      const int64_t q = r / L.E;
      const int e3 = int(r - q * L.E), c3 = int(q / L.LD);
      n = int(q - int64_t(c3) * L.LD);
      col = c3 * L.E + e3;
    } else if (L.perm == 4) {  // n*(nc*E) + col
      n = int(r / cols);
      col = int(r - int64_t(n) * cols);
    } else {
      col = int(r / L.LD);
      n = int(r - int64_t(col) * L.LD);
    }
    T v = T(0);
    if (col < cols && n < Np) {
      int e, c;
      if (L.perm == 1) {
        const int gw = 4 * L.nc, g = col / gw, q = col - gw * g, nt = q >> 3, rr = q & 7;  // 4-element groups
        e = 4 * g + (rr >> 1);
        c = 2 * nt + (rr & 1);
      } else if (L.perm == 3) {
        e = col % L.E;
        c = col / L.E;
      } else {
        e = col / L.nc;
        c = col - L.nc * e;
      }
      const int64_t k = t * L.E + e;
      if (k < K) v = T(src[(int64_t(c) * K + k) * Np + n]);
    }
    dst[w] = v;
  }
}

// Padding hygiene: is word r of a tile a real DOF (element k < K, component,
// node n < Np) of layout L?  Mirrors the placement of k_cm_to_tiles.
__device__ inline bool tile_word_valid(int64_t t, int64_t r, int64_t K, int Np, const TileLayout& L) {
  const int cols = L.nc * L.E;
  int col, n;
  if (L.perm == 3) {
    const int64_t q = r / L.E;
    const int e3 = int(r - q * L.E), c3 = int(q / L.LD);
    n = int(q - int64_t(c3) * L.LD);
    col = c3 * L.E + e3;
  } else if (L.perm == 4) {
    n = int(r / cols);
    col = int(r - int64_t(n) * cols);
  } else if (L.perm == 2) {
    const int chunk = int(r >> 5), q = int(r & 31), kc = L.LD >> 2;
    col = (chunk / kc) * 8 + (q >> 2);
    n = (chunk % kc) * 4 + (q & 3);
  } else {
    col = int(r / L.LD);
    n = int(r - int64_t(col) * L.LD);
  }
  if (col >= cols || n >= Np) return false;
  int e;
  if (L.perm == 1) {
    const int gw = 4 * L.nc, g = col / gw, q = col - gw * g;
    e = 4 * g + ((q & 7) >> 1);
  } else if (L.perm == 3) {
    e = col % L.E;
  } else {
    e = col / L.nc;
  }
  return t * L.E + e < K;
}

template <typename T>
__global__ void k_poison_padding(T* __restrict__ buf, int64_t K, int Np, TileLayout L) {
  const int64_t total = L.ntiles(K) * L.TS;
  for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < total; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = w / L.TS;
    if (!tile_word_valid(t, w - t * L.TS, K, Np, L)) buf[w] = T(NAN);
  }
}

// counts[0] += padding words that are not NaN, counts[1] += real DOFs that are not finite
template <typename T>
__global__ void k_check_padding(const T* __restrict__ buf, int64_t K, int Np, TileLayout L,
                                unsigned long long* counts) {
  const int64_t total = L.ntiles(K) * L.TS;
  unsigned long long a = 0, b = 0;
  for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < total; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = w / L.TS;
    const T v = buf[w];
    if (tile_word_valid(t, w - t * L.TS, K, Np, L)) {
      if (!isfinite(double(v))) ++b;
    } else if (!isnan(double(v))) {
      ++a;
    }
  }
  if (a) atomicAdd(counts, a);
  if (b) atomicAdd(counts + 1, b);
}

// device layout L -> [6][K][Np]
template <typename T, typename D>
__global__ void k_tiles_to_cm(const T* __restrict__ src, D* __restrict__ dst, int64_t K, int Np, TileLayout L) {
  const int64_t total = L.nc * K * Np;
  for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < total; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = w / (K * Np);
    const int64_t rem = w - c * K * Np;
    const int64_t k = rem / Np;
    const int n = int(rem - k * Np);
    dst[w] = D(src[L.off(k, int(c), n)]);
  }
}

static unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return unsigned(g);
}

template <typename T>
void poison_padding(T* buf, int64_t K, int Np, const TileLayout& L, void* st) {
  k_poison_padding<T><<<grid_for(L.ntiles(K) * L.TS), 256, 0, static_cast<cudaStream_t>(st)>>>(buf, K, Np, L);
}
template <typename T>
void check_padding(const T* buf, int64_t K, int Np, const TileLayout& L, unsigned long long* counts, void* st) {
  k_check_padding<T><<<grid_for(L.ntiles(K) * L.TS), 256, 0, static_cast<cudaStream_t>(st)>>>(buf, K, Np, L, counts);
}
template void poison_padding<double>(double*, int64_t, int, const TileLayout&, void*);
template void poison_padding<float>(float*, int64_t, int, const TileLayout&, void*);
template void check_padding<double>(const double*, int64_t, int, const TileLayout&, unsigned long long*, void*);
template void check_padding<float>(const float*, int64_t, int, const TileLayout&, unsigned long long*, void*);

template <typename S, typename T>
void cm_to_tiles(const S* src, T* dst, int64_t K, int Np, const TileLayout& L, void* st) {
  k_cm_to_tiles<S, T><<<grid_for(L.ntiles(K) * L.TS), 256, 0, static_cast<cudaStream_t>(st)>>>(src, dst, K, Np, L);
}

template <typename T, typename D>
void tiles_to_cm(const T* src, D* dst, int64_t K, int Np, const TileLayout& L, void* st) {
  k_tiles_to_cm<T, D><<<grid_for(L.nc * K * Np), 256, 0, static_cast<cudaStream_t>(st)>>>(src, dst, K, Np, L);
}

template void cm_to_tiles<double, double>(const double*, double*, int64_t, int, const TileLayout&, void*);
template void cm_to_tiles<double, float>(const double*, float*, int64_t, int, const TileLayout&, void*);
template void cm_to_tiles<float, float>(const float*, float*, int64_t, int, const TileLayout&, void*);
template void tiles_to_cm<double, double>(const double*, double*, int64_t, int, const TileLayout&, void*);
template void tiles_to_cm<float, double>(const float*, double*, int64_t, int, const TileLayout&, void*);
template void tiles_to_cm<float, float>(const float*, float*, int64_t, int, const TileLayout&, void*);

}  // namespace dg

namespace dg {

// Pack the partition-face traces (a6): for send face g, component c, face node j:
// buf[g][c][j] = u[sidx[g][j] + c*Np]  (sender's own face-node order).
template <typename T>
__global__ void k_pack_traces(const T* __restrict__ u, T* __restrict__ buf, const int32_t* __restrict__ sidx,
                              int64_t nfaces, int Nfp, TileLayout L) {
  const int64_t total = nfaces * L.nc * Nfp;
  for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < total; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = w / (L.nc * Nfp);
    const int r = int(w - g * L.nc * Nfp);
    const int c = r / Nfp, j = r - c * Nfp;
    const int32_t si = sidx[g * Nfp + j];
    buf[w] = L.perm == 2 ? u[L.off(si >> 8, c, si & 255)] : u[si + L.cofs(c)];
  }
}

template <typename T>
void pack_traces(const T* u, T* buf, const int32_t* sidx, int64_t nfaces, int Nfp, const TileLayout& L, void* st) {
  k_pack_traces<T><<<grid_for(nfaces * L.nc * Nfp), 256, 0, static_cast<cudaStream_t>(st)>>>(u, buf, sidx, nfaces, Nfp,
                                                                                          L);
}
template void pack_traces<double>(const double*, double*, const int32_t*, int64_t, int, const TileLayout&, void*);
template void pack_traces<float>(const float*, float*, const int32_t*, int64_t, int, const TileLayout&, void*);

}  // namespace dg
