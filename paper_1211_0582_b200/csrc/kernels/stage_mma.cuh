// MMA variant (FP64): the two dense contractions of a stage on the FP64 tensor
// pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), everything else fused around
// them, in a persistent, software-pipelined kernel.
//
// "View the field vectors in aggregate as a matrix": a tile
// is E elements; its 6E element-component columns are the MMA N dimension.
//   volume (a1):  Y_b = D_b . U      D_b in {Dr, Ds, Dt}: [M8 x KV],  U: [KV x 6E]
//   lift   (a4):  R  = curl(Y) + LIFT . Flux                 LIFT: [M8 x NF]
// A operands (reference operators, zero-padded to M8 rows / KV columns) are
// resident in shared memory where they fit (the paper's "matrix in shared
// memory" strategy), else read through L1.  B operands live in
// shared memory with leading dimension = 4 (mod 16) doubles: conflict-free
// fragment loads.
//
// Column permutation.  Within a group of 4 elements (24 columns = 3 n-tiles) the
// physical column of (element e, component c) is
//     P = 8*(c/2) + 2*e + (c%2),
// so the m8n8k4 accumulator layout (lane holds columns 2*tig+v of each n-tile)
// puts all six components of element e = tig at node row gid into ONE thread:
// the chain rule, the curl (eq. 4, eq. 6) and the LSERK update are thread-local.
//
// Pipeline per CTA (grid = resident CTAs; tiles strided over the grid): while
// computing tile i, cp.async brings tile i+1's U, geometry and gather indices
// into the other buffer; after tile i's MMA phase the exterior traces u+ of tile
// i+1 (a2's irregular gather) are gathered with cp.async
// straight into the face buffer, where the flux phase turns them into
// Fscale/2 * n.(F-F*) in place; the residual of tile i+1 is fetched alongside.
// Every cp.async group is waited on by its issuing thread and followed by a
// block barrier before any other thread reads it.
#pragma once
#include <cuda_runtime.h>

#include "pdl.cuh"
#include "stage_basic.cuh"

namespace dg {

template <int N>
struct MmaCfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  static constexpr int M8 = (Np + 7) / 8 * 8;
  static constexpr int MT = M8 / 8;
  static constexpr int KV = (Np + 3) / 4 * 4;
  static constexpr int KL = NF;  // multiple of 4 for every N
  static constexpr int ld4(int x) { return x + ((4 - x % 16) + 16) % 16; }
  static constexpr int LDU = ld4(KV);
  static constexpr int LDF = ld4(KL);
  static constexpr int LDA = ld4(KV);  // smem-resident operators
  static constexpr int LDL = ld4(KL);
  // per-order tile (elements, multiple of 4), warps, operator residency
  static constexpr int E = N == 1 ? 32 : N == 2 ? 16 : N == 3 ? 8 : 4;
  static constexpr int NW = N == 1 ? 8 : N == 2 ? 8 : N == 3 ? 6 : N == 4 ? 5 : N == 5 ? 7 : N == 6 ? 11 : N == 7 ? 5 : 7;
  static constexpr bool OPS_SMEM = N <= 5;
  static constexpr int G = E / 4;
  static constexpr int TASKS = MT * G;
  static constexpr int NT = NW * 32;
  static constexpr int COLS = 6 * E;
  // shared memory carve-up (doubles)
  static constexpr int U_SZ = COLS * LDU;
  static constexpr int GEO_SZ = E * GEO_W + (E * GEO_W) % 2;
  static constexpr int GIDX_SZ = (E * NF + 1) / 2;  // int32 -> doubles
  static constexpr int F_SZ = COLS * LDF;
  static constexpr int OPS_SZ = OPS_SMEM ? 3 * M8 * LDA + M8 * LDL : 0;
  static constexpr int FM_SZ = (NF + 3) / 4;        // int16 -> doubles
  static constexpr size_t SMEM_DOUBLES =
      size_t(2) * U_SZ + U_SZ /*res*/ + 2 * GEO_SZ + 2 * GIDX_SZ + F_SZ + OPS_SZ + FM_SZ;
  static constexpr size_t SMEM_BYTES = SMEM_DOUBLES * 8;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  // padded operator buffer in global memory: Dr|Ds|Dt as [3][M8][KV], then LIFT [M8][KL]
  static constexpr size_t OPS_DOUBLES = size_t(3) * M8 * KV + size_t(M8) * KL;
};

// physical B-operand column of (element e of the tile, component c)
__device__ __forceinline__ int pcol(int e, int c) { return 24 * (e >> 2) + 8 * (c >> 1) + 2 * (e & 3) + (c & 1); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem_dst))),
               "l"(gmem_src));
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int n>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(n)); }

template <int N, bool UPDATE>
__global__ void __launch_bounds__(MmaCfg<N>::NT)
    dg_stage_mma(const StageParams<double> p, const double* __restrict__ opsA) {
  using C = MmaCfg<N>;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, M8 = C::M8, KV = C::KV, KL = C::KL;
  constexpr int E = C::E, LDU = C::LDU, LDF = C::LDF, NT = C::NT;
  extern __shared__ __align__(16) double smem_mma[];
  double* smem = smem_mma;
  pdl_trigger();
  double* sU0 = smem;
  double* sU1 = sU0 + C::U_SZ;
  double* sR = sU1 + C::U_SZ;                  // residual of the current tile [P][LDU]
  double* sG0 = sR + C::U_SZ;
  double* sG1 = sG0 + C::GEO_SZ;
  int32_t* sI0 = reinterpret_cast<int32_t*>(sG1 + C::GEO_SZ);  // gather indices [e][m] (x2)
  int32_t* sI1 = reinterpret_cast<int32_t*>(sG1 + C::GEO_SZ + C::GIDX_SZ);
  double* sF = sG1 + C::GEO_SZ + 2 * C::GIDX_SZ;  // traces u+, then the face buffer [P][LDF]
  double* sA = sF + C::F_SZ;                   // operators (OPS_SMEM)
  int16_t* sFm = reinterpret_cast<int16_t*>(sA + C::OPS_SZ);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t ES = p.ES;  // = 6 Np for FP64
  const int64_t ntiles = (p.K + E - 1) / E;

  // ---- one-time: operators and Fmask into shared memory
  for (int m = tid; m < NF; m += NT) sFm[m] = p.fmask[m];
  if constexpr (C::OPS_SMEM) {  // cp.async: overlaps with the first tile's loads
    for (int w = tid; w < 3 * M8 * KV; w += NT) {
      const int r = w / KV, k = w - r * KV;
      cp_async8(sA + r * C::LDA + k, opsA + w);
    }
    const double* Lg = opsA + 3 * M8 * KV;
    for (int w = tid; w < M8 * KL; w += NT) {
      const int r = w / KL, k = w - r * KL;
      cp_async8(sA + 3 * M8 * C::LDA + r * C::LDL + k, Lg + w);
    }
  }

  auto tile_count = [&](int64_t tl) -> int {
    const int64_t k0 = p.k_begin + tl * E, kend = p.k_begin + p.K;
    return int(kend - k0 < E ? kend - k0 : E);
  };
  // cp.async of a tile's U (permuted columns), geometry and gather indices;
  // absent elements are zero-filled (their columns still enter the MMAs)
  auto issue_tile = [&](int64_t tl, double* sU, double* sG, int32_t* sI) {
    const int64_t k0 = p.k_begin + tl * E;
    const int ne = tile_count(tl);
    const double* ug = p.u_in + k0 * ES;
    for (int w = tid; w < E * 6 * Np; w += NT) {
      const int ec = w / Np, n = w - ec * Np;
      const int e = ec / 6, c = ec - 6 * e;
      double* dst = sU + pcol(e, c) * LDU + n;
      if (e < ne)
        cp_async8(dst, ug + w);
      else
        *dst = 0.0;
    }
    for (int w = tid; w < E * GEO_W; w += NT) {
      if (w < ne * GEO_W)
        cp_async8(sG + w, p.geo + k0 * GEO_W + w);
      else
        sG[w] = 0.0;
    }
    for (int w = tid; w < E * NF; w += NT) {
      if (w < ne * NF)
        cp_async4(sI + w, p.gidx + k0 * NF + w);
      else
        sI[w] = -1;
    }
  };
  // gather the exterior traces u+ of the tile whose indices are in sI into sF.
  // Each thread handles exactly the index slots it copied itself (no barrier needed).
  auto issue_traces = [&](const int32_t* sI) {
    for (int w = tid; w < E * NF; w += NT) {
      const int32_t gi = sI[w];
      if (gi >= 0) {
        const int e = w / NF, m = w - e * NF;
        const int64_t cs = (gi >= p.ghost_base) ? Nfp : Np;
        const double* src = p.u_in + gi;
#pragma unroll
        for (int c = 0; c < 6; ++c) cp_async8(sF + pcol(e, c) * LDF + m, src + c * cs);
      }
    }
  };
  auto issue_res = [&](int64_t tl) {
    if (!UPDATE || p.first_stage) return;
    const int64_t k0 = p.k_begin + tl * E;
    const int ne = tile_count(tl);
    const double* rg = p.res + k0 * ES;
    for (int w = tid; w < ne * 6 * Np; w += NT) {
      const int ec = w / Np, n = w - ec * Np;
      const int e = ec / 6, c = ec - 6 * e;
      cp_async8(sR + pcol(e, c) * LDU + n, rg + w);
    }
  };
  // zero the K padding of both U buffers once (tile loads never touch it)
  if constexpr (LDU > Np) {
    constexpr int PAD = LDU - Np;
    for (int w = tid; w < C::COLS * PAD; w += NT) {
      const int col = w / PAD, n = Np + (w - col * PAD);
      sU0[col * LDU + n] = 0.0;
      sU1[col * LDU + n] = 0.0;
    }
  }

  pdl_wait();  // the previous stage's fields are complete from here on
  int64_t tile = blockIdx.x;
  if (tile < ntiles) {
    issue_tile(tile, sU0, sG0, sI0);
    cp_commit();
    cp_wait<0>();
    issue_traces(sI0);
    issue_res(tile);
    cp_commit();
  }
  __syncthreads();

  int buf = 0;
  for (; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const double* sU = buf ? sU1 : sU0;
    const double* sG = buf ? sG1 : sG0;
    const int32_t* sI = buf ? sI1 : sI0;
    const int64_t k0 = p.k_begin + tile * E;
    const int ne = tile_count(tile);
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) issue_tile(next, buf ? sU0 : sU1, buf ? sG0 : sG1, buf ? sI0 : sI1);
    cp_commit();
    cp_wait<1>();  // everything but the prefetch: this tile's traces and residual have landed
    __syncthreads();

    // ---- a2 + a3: upwind/PEC flux, in place over the gathered traces
    for (int w = tid; w < E * NF; w += NT) {
      const int e = w / NF, m = w - e * NF, f = m / Nfp;
      double* fcol[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) fcol[c] = sF + pcol(e, c) * LDF + m;
      double fl[6] = {0, 0, 0, 0, 0, 0};
      if (e < ne) {
        const double* g = sG + e * GEO_W + 9 + 4 * f;
        const double nx = g[0], ny = g[1], nz = g[2], fs = g[3];
        const int nM = sFm[m];
        double uM[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) uM[c] = sU[pcol(e, c) * LDU + nM];
        double dE[3], dH[3];
        if (sI[w] >= 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            dE[c] = *fcol[c] - uM[c];
            dH[c] = *fcol[c + 3] - uM[c + 3];
          }
        } else {  // PEC wall: E+ = -E-, H+ = H-
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            dE[c] = -2.0 * uM[c];
            dH[c] = 0.0;
          }
        }
        maxwell_flux<double>(nx, ny, nz, p.alpha, dE, dH, fl);
        const double sc = fs * 0.5;
#pragma unroll
        for (int c = 0; c < 6; ++c) fl[c] *= sc;
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) *fcol[c] = fl[c];
    }
    __syncthreads();

    // ---- a1 + curl + a4 + a5 per warp task (m-tile t, group g); thread = (node row, element 4g+tig)
    for (int task = warp; task < C::TASKS; task += C::NW) {
      const int t = task % C::MT, g = task / C::MT;
      const int row = 8 * t + gid;
      double acc[3][3][2];
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) acc[b][nt][0] = acc[b][nt][1] = 0.0;
      const double* bp = sU + (24 * g + gid) * LDU + tig;
      if constexpr (C::OPS_SMEM) {
        const double* ap = sA + row * C::LDA + tig;
#pragma unroll
        for (int kk = 0; kk < KV; kk += 4) {
          const double ar = ap[kk], as = ap[M8 * C::LDA + kk], at = ap[2 * M8 * C::LDA + kk];
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) {
            const double bv = bp[nt * 8 * LDU + kk];
            dmma(acc[0][nt], ar, bv);
            dmma(acc[1][nt], as, bv);
            dmma(acc[2][nt], at, bv);
          }
        }
      } else {
        const double* ap = opsA + size_t(row) * KV + tig;
#pragma unroll 4
        for (int kk = 0; kk < KV; kk += 4) {
          const double ar = __ldg(ap + kk);
          const double as = __ldg(ap + size_t(M8) * KV + kk);
          const double at = __ldg(ap + size_t(2) * M8 * KV + kk);
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) {
            const double bv = bp[nt * 8 * LDU + kk];
            dmma(acc[0][nt], ar, bv);
            dmma(acc[1][nt], as, bv);
            dmma(acc[2][nt], at, bv);
          }
        }
      }
      // chain rule (eq. 6) + curl, thread-local: acc[b][c/2][c%2] = D_b u_c of element 4g+tig
      double r[3][2];
      {
        const double* Gm = sG + (4 * g + tig) * GEO_W;
        double dx[6], dy[6], dz[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const double ur = acc[0][c >> 1][c & 1], us = acc[1][c >> 1][c & 1], ut = acc[2][c >> 1][c & 1];
          dx[c] = Gm[0] * ur + Gm[3] * us + Gm[6] * ut;
          dy[c] = Gm[1] * ur + Gm[4] * us + Gm[7] * ut;
          dz[c] = Gm[2] * ur + Gm[5] * us + Gm[8] * ut;
        }
        // d_t E = curl H, d_t H = -curl E   (components: 0..2 E, 3..5 H)
        r[0][0] = dy[5] - dz[4];
        r[0][1] = dz[3] - dx[5];
        r[1][0] = dx[4] - dy[3];
        r[1][1] = -(dy[2] - dz[1]);
        r[2][0] = -(dz[0] - dx[2]);
        r[2][1] = -(dx[1] - dy[0]);
      }
      // lift: r += LIFT . Flux  (even/odd k-steps in two accumulator sets: 6 independent DMMA chains)
      const double* fp = sF + (24 * g + gid) * LDF + tig;
      double r2[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      static_assert(KL % 8 == 4 || KL % 8 == 0, "KL multiple of 4");
      if constexpr (C::OPS_SMEM) {
        const double* lp = sA + 3 * M8 * C::LDA + row * C::LDL + tig;
#pragma unroll
        for (int kk = 0; kk < KL; kk += 8) {
          const double a0 = lp[kk];
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dmma(r[nt], a0, fp[nt * 8 * LDF + kk]);
          if (kk + 4 < KL) {
            const double a1 = lp[kk + 4];
#pragma unroll
            for (int nt = 0; nt < 3; ++nt) dmma(r2[nt], a1, fp[nt * 8 * LDF + kk + 4]);
          }
        }
      } else {
        const double* lp = opsA + size_t(3) * M8 * KV + size_t(row) * KL + tig;
#pragma unroll 2
        for (int kk = 0; kk < KL; kk += 8) {
          const double a0 = __ldg(lp + kk);
          const double a1 = (kk + 4 < KL) ? __ldg(lp + kk + 4) : 0.0;
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dmma(r[nt], a0, fp[nt * 8 * LDF + kk]);
          if (kk + 4 < KL) {
#pragma unroll
            for (int nt = 0; nt < 3; ++nt) dmma(r2[nt], a1, fp[nt * 8 * LDF + kk + 4]);
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        r[nt][0] += r2[nt][0];
        r[nt][1] += r2[nt][1];
      }
      // LSERK update / RHS store for (node row, element 4g+tig, component c)
      const int e = 4 * g + tig;
      if (row < Np && e < ne) {
        const int64_t base = (k0 + e) * ES + row;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const int64_t idx = base + c * Np;
          const double rhs = r[c >> 1][c & 1];
          const int col = 24 * g + 8 * (c >> 1) + 2 * tig + (c & 1);
          if (UPDATE) {
            const double rold = p.first_stage ? 0.0 : sR[col * LDU + row];
            const double rr = p.rk_a * rold + p.dt * rhs;
            p.res[idx] = rr;
            p.u_out[idx] = sU[col * LDU + row] + p.rk_b * rr;
          } else {
            p.rhs_out[idx] = rhs;
          }
        }
      }
    }
    // all warps are done with this tile's buffers and face buffer
    cp_wait<0>();
    __syncthreads();
    // exterior traces and residual of the next tile (its indices landed with the prefetch group)
    if (next < ntiles) {
      issue_traces(buf ? sI0 : sI1);
      issue_res(next);
    }
    cp_commit();
  }
  cp_wait<0>();
}

template <int N>
void launch_stage_mma(const StageParams<double>& p, const double* opsA, int mode, cudaStream_t st) {
  using C = MmaCfg<N>;
  static PerDevice pd;
  static int blocks[64] = {0};  // resident CTAs per SM, per device (set with the smem attribute)
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sms_for_device(pd, [&] {
    cudaFuncSetAttribute(dg_stage_mma<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaFuncSetAttribute(dg_stage_mma<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks[dev & 63], dg_stage_mma<N, true>, C::NT, C::SMEM_BYTES);
  });
  const int grid_max = sms * (blocks[dev & 63] > 0 ? blocks[dev & 63] : 1);
  if (p.K <= 0) return;
  const int64_t ntiles = (p.K + C::E - 1) / C::E;
  const unsigned grid = unsigned(ntiles < grid_max ? ntiles : grid_max);
  if (mode == 1)
    launch_pdl(N >= 3, dg_stage_mma<N, true>, grid, C::NT, C::SMEM_BYTES, st, p, opsA);
  else
    launch_pdl(N >= 3, dg_stage_mma<N, false>, grid, C::NT, C::SMEM_BYTES, st, p, opsA);
}

}  // namespace dg
