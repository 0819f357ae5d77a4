// MMA variant (FP64): the two dense contractions of a stage on the FP64 tensor
// pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), everything else fused around them.
//
// "View the field vectors in aggregate as a matrix": a CTA owns
// E elements; its 6E element-component columns are the MMA N dimension.
//   volume (a1):  Y_b = D_b . U      D_b in {Dr, Ds, Dt}: [M8 x KV],  U: [KV x 6E]
//   lift   (a4):  R  = curl(Y) + LIFT . Flux                 LIFT: [M8 x NF]
// A operands (operators, zero-padded to M8 rows / KV cols) are read through L1
// (__ldg) — they are shared by every CTA; B operands (the element tile U and the
// face buffer Flux) live in shared memory with a leading dimension = 4 (mod 16)
// doubles so every fragment load is bank-conflict free.  The face buffer
// (a2+a3) never leaves the chip; the LSERK update (a5) is applied straight from
// the lift accumulators.
//
// Work split: task = (node m-tile t of 8 rows, column group g of 4 elements = 24
// columns = 3 n-tiles).  A warp computes all three derivative blocks of its task,
// so the chain rule + curl (eq. 6) need only a per-warp 8x24 scratch exchange.
#pragma once
#include <cuda_runtime.h>

#include "stage_basic.cuh"

namespace dg {

template <int N>
struct MmaCfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  static constexpr int M8 = (Np + 7) / 8 * 8;
  static constexpr int MT = M8 / 8;
  static constexpr int KV = (Np + 3) / 4 * 4;
  static constexpr int KL = NF;  // multiple of 4 for every N
  // leading dimensions = 4 (mod 16) doubles: conflict-free 8x4 fragment loads
  static constexpr int ld4(int x) { return x + ((4 - x % 16) + 16) % 16; }
  static constexpr int LDU = ld4(KV);
  static constexpr int LDF = ld4(KL);
  // elements per CTA (multiple of 4) and warps per CTA, chosen per order so that
  // MT * (E/4) tasks split evenly over the warps
  static constexpr int E = N <= 1 ? 32 : N <= 2 ? 16 : N <= 3 ? 16 : N <= 6 ? 8 : 4;
  static constexpr int G = E / 4;
  static constexpr int TASKS = MT * G;
  static constexpr int NW = N <= 2 ? 8 : N == 3 ? 4 : N == 4 ? 5 : N == 5 ? 7 : N == 6 ? 11 : N == 7 ? 5 : 7;
  static constexpr int NT = NW * 32;
  static constexpr int COLS = 6 * E;
  static constexpr int SCR = 3 * 8 * 24;  // per-warp derivative scratch
  static constexpr size_t SMEM_DOUBLES = size_t(COLS) * LDU + size_t(COLS) * LDF + size_t(E) * GEO_W + size_t(NW) * SCR;
  static constexpr size_t SMEM_BYTES = SMEM_DOUBLES * 8 + NF * 2 + 16;
  // padded operator buffer: Dr|Ds|Dt as [3][M8][KV], then LIFT as [M8][KL]
  static constexpr size_t OPS_DOUBLES = size_t(3) * M8 * KV + size_t(M8) * KL;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int N, bool UPDATE>
__global__ void __launch_bounds__(MmaCfg<N>::NT) dg_stage_mma(const StageParams<double> p, const double* __restrict__ opsA) {
  using C = MmaCfg<N>;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, M8 = C::M8, KV = C::KV, KL = C::KL;
  constexpr int E = C::E, LDU = C::LDU, LDF = C::LDF, NT = C::NT;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;                       // [6E][LDU]  element-component columns
  double* sF = sU + C::COLS * LDU;         // [6E][LDF]  face buffer (flux x Fscale/2)
  double* sG = sF + C::COLS * LDF;         // [E][GEO_W]
  double* sS = sG + E * GEO_W;             // [NW][3][8][24]
  int16_t* sFm = reinterpret_cast<int16_t*>(sS + C::NW * C::SCR);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t k0 = p.k_begin + int64_t(blockIdx.x) * E;
  const int64_t kend = p.k_begin + p.K;
  const int ne = int(kend - k0 < E ? kend - k0 : E);
  const int64_t ES = p.ES;  // = 6 Np for FP64

  // ---- stage the element tile (coalesced: the E tiles are one contiguous chunk)
  const double* ug = p.u_in + k0 * ES;
  for (int w = tid; w < E * 6 * Np; w += NT) {
    const int col = w / Np, n = w - col * Np;
    sU[col * LDU + n] = (col < ne * 6) ? ug[w] : 0.0;
  }
  if constexpr (LDU > Np) {
    constexpr int PAD = LDU - Np;  // zero the K padding (the A operand is zero there too)
    for (int w = tid; w < C::COLS * PAD; w += NT) {
      const int col = w / PAD, n = Np + (w - col * PAD);
      sU[col * LDU + n] = 0.0;
    }
  }
  for (int w = tid; w < E * GEO_W; w += NT) sG[w] = (w < ne * GEO_W) ? p.geo[k0 * GEO_W + w] : 0.0;
  for (int m = tid; m < NF; m += NT) sFm[m] = p.fmask[m];
  __syncthreads();

  // ---- a2 + a3: traces and upwind/PEC flux into the face buffer
  for (int w = tid; w < E * NF; w += NT) {
    const int e = w / NF, m = w - e * NF, f = m / Nfp;
    double fl[6] = {0, 0, 0, 0, 0, 0};
    if (e < ne) {
      const double* g = sG + e * GEO_W + 9 + 4 * f;
      const double nx = g[0], ny = g[1], nz = g[2], fs = g[3];
      const int nM = sFm[m];
      const double* uM = sU + (e * 6) * LDU + nM;
      const int32_t gi = p.gidx[(k0 + e) * NF + m];
      double dE[3], dH[3];
      if (gi >= 0) {
        const int64_t cs = (gi >= p.ghost_base) ? Nfp : Np;
        const double* uP = p.u_in + gi;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          dE[c] = __ldg(uP + c * cs) - uM[c * LDU];
          dH[c] = __ldg(uP + (c + 3) * cs) - uM[(c + 3) * LDU];
        }
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          dE[c] = -2.0 * uM[c * LDU];
          dH[c] = 0.0;
        }
      }
      maxwell_flux<double>(nx, ny, nz, p.alpha, dE, dH, fl);
      const double sc = fs * 0.5;
#pragma unroll
      for (int c = 0; c < 6; ++c) fl[c] *= sc;
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) sF[(e * 6 + c) * LDF + m] = fl[c];
  }
  __syncthreads();

  // ---- a1 + curl + a4 + a5 per warp task
  const double* Dall = opsA;
  const double* Lp = opsA + size_t(3) * M8 * KV;
  double* scr = sS + warp * C::SCR;
  for (int task = warp; task < C::TASKS; task += C::NW) {
    const int t = task % C::MT, g = task / C::MT;
    const int row = 8 * t + gid;
    double acc[3][3][2];
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) acc[b][nt][0] = acc[b][nt][1] = 0.0;
    const double* a0p = Dall + size_t(row) * KV + tig;
    const double* bp = sU + (24 * g + gid) * LDU + tig;
#pragma unroll 4
    for (int kk = 0; kk < KV; kk += 4) {
      const double ar = __ldg(a0p + kk);
      const double as = __ldg(a0p + size_t(M8) * KV + kk);
      const double at = __ldg(a0p + size_t(2) * M8 * KV + kk);
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        const double bv = bp[nt * 8 * LDU + kk];
        dmma(acc[0][nt], ar, bv);
        dmma(acc[1][nt], as, bv);
        dmma(acc[2][nt], at, bv);
      }
    }
    // chain rule (eq. 6) for this thread's 6 columns -> per-warp scratch
#pragma unroll
    for (int nt = 0; nt < 3; ++nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int lc = 8 * nt + 2 * tig + v;          // column within the group
        const double* G = sG + (4 * g + lc / 6) * GEO_W;
        const double ur = acc[0][nt][v], us = acc[1][nt][v], ut = acc[2][nt][v];
        scr[(0 * 8 + gid) * 24 + lc] = G[0] * ur + G[3] * us + G[6] * ut;  // d/dx
        scr[(1 * 8 + gid) * 24 + lc] = G[1] * ur + G[4] * us + G[7] * ut;  // d/dy
        scr[(2 * 8 + gid) * 24 + lc] = G[2] * ur + G[5] * us + G[8] * ut;  // d/dz
      }
    __syncwarp();
    double r[3][2];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int lc = 8 * nt + 2 * tig + v;
        const int base = (lc / 6) * 6, c = lc % 6;
        const double* sx = scr + (0 * 8 + gid) * 24 + base;
        const double* sy = scr + (1 * 8 + gid) * 24 + base;
        const double* sz = scr + (2 * 8 + gid) * 24 + base;
        double val;
        // d_t E = curl H, d_t H = -curl E   (components: 0..2 E, 3..5 H)
        switch (c) {
          case 0: val = sy[5] - sz[4]; break;
          case 1: val = sz[3] - sx[5]; break;
          case 2: val = sx[4] - sy[3]; break;
          case 3: val = -(sy[2] - sz[1]); break;
          case 4: val = -(sz[0] - sx[2]); break;
          default: val = -(sx[1] - sy[0]); break;
        }
        r[nt][v] = val;
      }
    __syncwarp();
    // lift: r += LIFT . Flux
    const double* lp = Lp + size_t(row) * KL + tig;
    const double* fp = sF + (24 * g + gid) * LDF + tig;
#pragma unroll 4
    for (int kk = 0; kk < KL; kk += 4) {
      const double a = __ldg(lp + kk);
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) dmma(r[nt], a, fp[nt * 8 * LDF + kk]);
    }
    // LSERK update / RHS store
    if (row < Np) {
#pragma unroll
      for (int nt = 0; nt < 3; ++nt)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = 24 * g + 8 * nt + 2 * tig + v;
          const int e = col / 6, c = col - 6 * (col / 6);
          if (e < ne) {
            const int64_t idx = (k0 + e) * ES + c * Np + row;
            if (UPDATE) {
              const double rr = (p.first_stage ? 0.0 : p.rk_a * p.res[idx]) + p.dt * r[nt][v];
              p.res[idx] = rr;
              p.u_out[idx] = sU[col * LDU + row] + p.rk_b * rr;
            } else {
              p.rhs_out[idx] = r[nt][v];
            }
          }
        }
    }
  }
}

template <int N>
void launch_stage_mma(const StageParams<double>& p, const double* opsA, int mode, cudaStream_t st) {
  using C = MmaCfg<N>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(dg_stage_mma<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaFuncSetAttribute(dg_stage_mma<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    attr_done = true;
  }
  if (p.K <= 0) return;
  const unsigned grid = unsigned((p.K + C::E - 1) / C::E);
  if (mode == 1)
    dg_stage_mma<N, true><<<grid, C::NT, C::SMEM_BYTES, st>>>(p, opsA);
  else
    dg_stage_mma<N, false><<<grid, C::NT, C::SMEM_BYTES, st>>>(p, opsA);
}

}  // namespace dg
