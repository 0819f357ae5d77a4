// BASIC variant: one fused kernel per LSERK stage over element tiles.
//
// One CTA owns EPB consecutive elements.  Per stage it
//   1. stages the element tile u[k][6][Np] in shared memory (coalesced),
//   2. surface (a2+a3): gathers u- from the tile and u+ through gidx, evaluates
//      the upwind/PEC flux x Fscale/2 into a shared face buffer [6][4Nfp]
//      (eq. 5; fig:flux-code a),
//   3. volume (a1): Dr/Ds/Dt contractions + chain rule + curl (eq. 4, eq. 6),
//   4. lift (a4): LIFT x face buffer added to the volume term,
//   5. LSERK update (a5): res = a res + dt rhs; u_out = u + b res, or writes rhs.
// The face buffer never leaves the chip (the paper's D4 facial buffer).
//
// SYS selects the linear system (dg_system): 0 Maxwell (6 fields), 1 acoustics
// (4 fields p, v; NEXT-3): the same four stages, only the flux function, the wall
// mirror state and the combination of the reference derivatives differ.
#pragma once
#include <cuda_runtime.h>

#include "stage_params.h"

namespace dg {

template <int N>
struct Order {
  static constexpr int Np = (N + 1) * (N + 2) * (N + 3) / 6;
  static constexpr int Nfp = (N + 1) * (N + 2) / 2;
  static constexpr int NF = 4 * Nfp;
};

template <typename T, int N>
struct BasicCfg {
  static constexpr int Np = Order<N>::Np;
  static constexpr int NT = Np <= 128 ? 128 : 256;
  static constexpr int EPB = NT / Np > 0 ? NT / Np : 1;
};

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// 2 n.(F - F*) for one face node; jumps d = u+ - u- (reading R1/R2).
template <typename T>
__device__ __forceinline__ void maxwell_flux(T nx, T ny, T nz, T alpha, const T dE[3], const T dH[3],
                                             T out[6]) {
  const T ndotdH = nx * dH[0] + ny * dH[1] + nz * dH[2];
  const T ndotdE = nx * dE[0] + ny * dE[1] + nz * dE[2];
  out[0] = (ny * dH[2] - nz * dH[1]) + alpha * (dE[0] - ndotdE * nx);
  out[1] = (nz * dH[0] - nx * dH[2]) + alpha * (dE[1] - ndotdE * ny);
  out[2] = (nx * dH[1] - ny * dH[0]) + alpha * (dE[2] - ndotdE * nz);
  out[3] = -(ny * dE[2] - nz * dE[1]) + alpha * (dH[0] - ndotdH * nx);
  out[4] = -(nz * dE[0] - nx * dE[2]) + alpha * (dH[1] - ndotdH * ny);
  out[5] = -(nx * dE[1] - ny * dE[0]) + alpha * (dH[2] - ndotdH * nz);
}

// Acoustics (R16): 2 n.(F - F*) = (-A_n + alpha |A_n|) [[u]], u = (p, v).
template <typename T>
__device__ __forceinline__ void acoustic_flux(T nx, T ny, T nz, T alpha, T dp, const T dv[3], T out[4]) {
  const T ndv = nx * dv[0] + ny * dv[1] + nz * dv[2];
  out[0] = alpha * dp - ndv;
  const T q = alpha * ndv - dp;
  out[1] = nx * q;
  out[2] = ny * q;
  out[3] = nz * q;
}

template <int SYS>
struct System;
template <>
struct System<0> { static constexpr int NC = 6; };
template <>
struct System<1> { static constexpr int NC = 4; };

template <typename T, int N, bool UPDATE, int SYS>
__global__ void __launch_bounds__(BasicCfg<T, N>::NT)
    dg_stage_basic(const StageParams<T> p) {
  constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  constexpr int NT = BasicCfg<T, N>::NT, EPB = BasicCfg<T, N>::EPB;
  constexpr int NC = System<SYS>::NC;
  __shared__ T su[EPB * NC * Np];
  __shared__ T sflux[EPB * NC * NF];
  __shared__ int16_t sfm[NF];

  const int tid = threadIdx.x;
  const int64_t k0 = p.k_begin + int64_t(blockIdx.x) * EPB;
  const int64_t kend = p.k_begin + p.K;
  const int ne = int(kend - k0 < EPB ? kend - k0 : EPB);
  const int64_t ES = p.ES;

  for (int m = tid; m < NF; m += NT) sfm[m] = p.fmask[m];
  // 1. element tile -> smem
  for (int w = tid; w < ne * NC * Np; w += NT) {
    const int e = w / (NC * Np), r = w - e * NC * Np;
    su[w] = p.u_in[(k0 + e) * ES + r];
  }
  __syncthreads();

  // 2. surface flux into the on-chip face buffer
  for (int w = tid; w < ne * NF; w += NT) {
    const int e = w / NF, m = w - e * NF, f = m / Nfp;
    const int64_t k = k0 + e;
    const T* g = p.geo + k * GEO_W + 9 + 4 * f;
    const T nx = ldg(g), ny = ldg(g + 1), nz = ldg(g + 2), fs = ldg(g + 3);
    const int nM = sfm[m];
    const T* uM = su + e * NC * Np + nM;
    const int32_t gi = p.gidx[k * NF + m];
    const int64_t cs = (gi >= p.ghost_base) ? Nfp : Np;
    const T* uP = p.u_in + gi;
    const T sc = fs * T(0.5);
    if constexpr (SYS == 0) {
      T dE[3], dH[3];
      if (gi >= 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          dE[c] = ldg(uP + c * cs) - uM[c * Np];
          dH[c] = ldg(uP + (c + 3) * cs) - uM[(c + 3) * Np];
        }
      } else {  // PEC wall: E+ = -E-, H+ = H-
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          dE[c] = T(-2) * uM[c * Np];
          dH[c] = T(0);
        }
      }
      T fl[6];
      maxwell_flux(nx, ny, nz, p.alpha, dE, dH, fl);
#pragma unroll
      for (int c = 0; c < 6; ++c) sflux[(e * NC + c) * NF + m] = fl[c] * sc;
    } else {
      T dp, dv[3];
      if (gi >= 0) {
        dp = ldg(uP) - uM[0];
#pragma unroll
        for (int c = 0; c < 3; ++c) dv[c] = ldg(uP + (c + 1) * cs) - uM[(c + 1) * Np];
      } else {  // rigid wall: p+ = p-, v+ = v- - 2 (n.v-) n
        const T ndv = nx * uM[Np] + ny * uM[2 * Np] + nz * uM[3 * Np];
        dp = T(0);
        dv[0] = T(-2) * ndv * nx;
        dv[1] = T(-2) * ndv * ny;
        dv[2] = T(-2) * ndv * nz;
      }
      T fl[4];
      acoustic_flux(nx, ny, nz, p.alpha, dp, dv, fl);
#pragma unroll
      for (int c = 0; c < 4; ++c) sflux[(e * NC + c) * NF + m] = fl[c] * sc;
    }
  }
  __syncthreads();

  // 3-5. volume + lift + update, one thread per (element, node)
  const T* Dr = p.ops;
  const T* Ds = p.ops + Np * Np;
  const T* Dt = p.ops + 2 * Np * Np;
  const T* LIFT = p.ops + 3 * Np * Np;
  for (int w = tid; w < ne * Np; w += NT) {
    const int e = w / Np, i = w - e * Np;
    const int64_t k = k0 + e;
    const T* ue = su + e * NC * Np;
    T ar[NC], as[NC], at[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) ar[c] = as[c] = at[c] = T(0);
    for (int j = 0; j < Np; ++j) {
      const T dr = ldg(Dr + i * Np + j), ds = ldg(Ds + i * Np + j), dt = ldg(Dt + i * Np + j);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const T v = ue[c * Np + j];
        ar[c] += dr * v;
        as[c] += ds * v;
        at[c] += dt * v;
      }
    }
    const T* g = p.geo + k * GEO_W;
    const T rx = ldg(g + 0), ry = ldg(g + 1), rz = ldg(g + 2);
    const T sx = ldg(g + 3), sy = ldg(g + 4), sz = ldg(g + 5);
    const T tx = ldg(g + 6), ty = ldg(g + 7), tz = ldg(g + 8);
    T dx[NC], dy[NC], dz[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      dx[c] = rx * ar[c] + sx * as[c] + tx * at[c];
      dy[c] = ry * ar[c] + sy * as[c] + ty * at[c];
      dz[c] = rz * ar[c] + sz * as[c] + tz * at[c];
    }
    T rhs[NC];
    if constexpr (SYS == 0) {
      // d_t E = curl H, d_t H = -curl E
      rhs[0] = dy[5] - dz[4];
      rhs[1] = dz[3] - dx[5];
      rhs[2] = dx[4] - dy[3];
      rhs[3] = -(dy[2] - dz[1]);
      rhs[4] = -(dz[0] - dx[2]);
      rhs[5] = -(dx[1] - dy[0]);
    } else {
      // d_t p = -div v, d_t v = -grad p
      rhs[0] = -(dx[1] + dy[2] + dz[3]);
      rhs[1] = -dx[0];
      rhs[2] = -dy[0];
      rhs[3] = -dz[0];
    }
    const T* fe = sflux + e * NC * NF;
    for (int m = 0; m < NF; ++m) {
      const T l = ldg(LIFT + i * NF + m);
#pragma unroll
      for (int c = 0; c < NC; ++c) rhs[c] += l * fe[c * NF + m];
    }
    if (UPDATE) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int64_t idx = k * ES + c * Np + i;
        const T r = (p.first_stage ? T(0) : p.rk_a * p.res[idx]) + p.dt * rhs[c];
        p.res[idx] = r;
        p.u_out[idx] = ue[c * Np + i] + p.rk_b * r;
      }
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) p.rhs_out[k * ES + c * Np + i] = rhs[c];
    }
  }
}

template <typename T, int N>
void launch_stage_basic(const StageParams<T>& p, int mode, cudaStream_t st) {
  using C = BasicCfg<T, N>;
  if (p.K <= 0) return;
  const unsigned grid = unsigned((p.K + C::EPB - 1) / C::EPB);
  if (p.system == 1) {
    if (mode == 1)
      dg_stage_basic<T, N, true, 1><<<grid, C::NT, 0, st>>>(p);
    else
      dg_stage_basic<T, N, false, 1><<<grid, C::NT, 0, st>>>(p);
  } else {
    if (mode == 1)
      dg_stage_basic<T, N, true, 0><<<grid, C::NT, 0, st>>>(p);
    else
      dg_stage_basic<T, N, false, 0><<<grid, C::NT, 0, st>>>(p);
  }
}

}  // namespace dg
