// WS variant, FP32: the warp-specialized TMA/mbarrier stage kernel of
// stage_ws.cuh with the two contractions on the tensor cores as 3xTF32
// (mma.sync.m16n8k8.tf32 -> SASS HMMA.1688.F32.TF32):
//     A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi      (x_hi = tf32(x), x_lo = tf32(x - x_hi))
// which keeps FP32-level accuracy (plain TF32 fails the 1e-4 FP32 tolerance:
// SURVEY.md §7 hard part 2).  A_hi/A_lo are split once on the host; B (element
// tile, face buffer) is split in registers as fragments are loaded.  The flux,
// chain rule, curl and LSERK update stay on the FFMA pipe, which runs
// concurrently with HMMA (tools/tf32_mma.cu: 518 TF32 FMA/clk/SM ~ 300 TFLOP/s,
// while FFMA warps keep 104 FMA/clk/SM alongside).
//
// m16n8k8 fragments: A a0=(g,t) a1=(g+8,t) a2=(g,t+4) a3=(g+8,t+4); B b0=(k=t,n=g)
// b1=(k=t+4,n=g); C c0=(g,2t) c1=(g,2t+1) c2=(g+8,2t) c3=(g+8,2t+1) with g = lane/4,
// t = lane%4.  Columns 2t+v per n-tile, as for DMMA, so the same column
// permutation gives each thread all six components of element 4g+t — here for
// two node rows (g and g+8 of the 16-row m-tile).
#pragma once
#include <cuda_runtime.h>

#include <cstring>

#include "stage_ws.cuh"

namespace dg {

__host__ __device__ constexpr int ldx8(int x) {  // >= x, = 4 (mod 8): conflict-free 8x4 TF32 fragments
  return (x % 8 == 4) ? x : ldx8(x + 4);
}

template <int N>
struct Ws32Cfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  static constexpr int M16 = (Np + 15) / 16 * 16;
  static constexpr int MT = M16 / 16;
  static constexpr int KV = (Np + 7) / 8 * 8;
  static constexpr int KL = (NF + 7) / 8 * 8;
  static constexpr int LD = ldx8(KV);
  static constexpr int LDF = ldx8(KL);
  static constexpr int LDA = ldx8(KV);
  static constexpr int LDL = ldx8(KL);
  // tuning builds: -DDG_W32_TUNE_N=n with -DDG_W32_{E,S,LA,RES,MW,PW}=v override order n only
#ifdef DG_W32_TUNE_N
  static constexpr bool TUNED = N == DG_W32_TUNE_N;
#else
  static constexpr bool TUNED = false;
#endif
#ifndef DG_W32_E
#define DG_W32_E 0
#endif
#ifndef DG_W32_S
#define DG_W32_S 0
#endif
#ifndef DG_W32_LA
#define DG_W32_LA -1
#endif
#ifndef DG_W32_RES
#define DG_W32_RES -1
#endif
#ifndef DG_W32_MW
#define DG_W32_MW 0
#endif
#ifndef DG_W32_PW
#define DG_W32_PW 0
#endif
  static constexpr int E = (TUNED && DG_W32_E) ? DG_W32_E : N == 1 ? 32 : N == 2 ? 16 : N == 3 ? 8 : 4;
  static constexpr int S = (TUNED && DG_W32_S) ? DG_W32_S : N <= 6 ? 5 : N <= 8 ? 4 : 3;
  static constexpr int LA = (TUNED && DG_W32_LA >= 0) ? DG_W32_LA : S - 2 < 2 ? S - 2 : 2;
  static constexpr bool OPS_SMEM = N <= 4;
  // measured (tools/gpu_tile_sweep.sh, profiles/r1_tile_sweep_f32.jsonl): 11 MMA warps with
  // the residual prefetched into registers win at N = 5, 7, 8 (+6..7 %); N = 3, 4, 6 keep
  // the residual in the ring and 8 MMA warps
  static constexpr bool RES_SMEM = (TUNED && DG_W32_RES >= 0) ? bool(DG_W32_RES) : N <= 4 || N == 6;
  static constexpr int MW = (TUNED && DG_W32_MW) ? DG_W32_MW : (N == 5 || N == 7 || N == 8) ? 11 : 8;
  static constexpr int PW = (TUNED && DG_W32_PW) ? DG_W32_PW : 4;
  // residual from global memory: prefetched into registers at task start while the CTA
  // has at most 16 warps (128 registers per thread; the file is split per SMSP)
  static constexpr bool RES_PREFETCH = !RES_SMEM && MW + 1 + PW <= 16;
  static constexpr int NT = 32 * (MW + 1 + PW);
  static constexpr int PT = 32 * PW;
  static constexpr int G = E / 4;
  static constexpr int T = MT * G;
  static constexpr int TS = 6 * E * LD;  // floats per tile
  static constexpr int GEOT = E * GEO_W;
  static constexpr int IDXT = E * NF;
  static constexpr int OFF_U = 0;
  static constexpr int OFF_R = OFF_U + r16(TS * 4);
  static constexpr int OFF_G = OFF_R + (RES_SMEM ? r16(TS * 4) : 0);
  static constexpr int OFF_I = OFF_G + r16(GEOT * 4);
  static constexpr int OFF_F = OFF_I + r16(IDXT * 4);
  static constexpr int SLOT = OFF_F + r16(6 * E * LDF * 4);
  // operators: hi and lo copies of [3][M16][LDA] + [M16][LDL]
  static constexpr int A_ONE = 3 * M16 * LDA + M16 * LDL;
  static constexpr int A_BYTES = OPS_SMEM ? r16(2 * A_ONE * 4) : 0;
  static constexpr int FM_BYTES = r16(NF * 2);
  static constexpr int BAR_BYTES = 4 * S * 8;
  static constexpr size_t SMEM_BYTES = size_t(S) * SLOT + A_BYTES + FM_BYTES + BAR_BYTES;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  // global operator buffer (floats): hi [3][M16][KV] + [M16][KL], then lo (same shape)
  static constexpr size_t OPS_ONE = size_t(3) * M16 * KV + size_t(M16) * KL;
};

__device__ __forceinline__ unsigned tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// split x into tf32 hi + lo: hi = x with the 13 low mantissa bits cleared (exactly a TF32
// value, so the MMA's own operand conversion cannot alter it), lo = x - hi (exact in FP32,
// |lo| < 2^-10 |x|; the MMA's TF32 conversion of lo costs at most 2^-20 |x|).  Two
// instructions instead of cvt.rna + FADD + cvt.rna.
#ifndef DG_W32_RNA_SPLIT
__device__ __forceinline__ void tf32_split(float x, unsigned& hi, unsigned& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
#else
__device__ __forceinline__ void tf32_split(float x, unsigned& hi, unsigned& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - __uint_as_float(hi));
}
#endif
__device__ __forceinline__ void hmma_tf32(float (&c)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 3xTF32: c += Ahi.Bhi + Ahi.Blo + Alo.Bhi
__device__ __forceinline__ void mma3(float (&c)[4], const unsigned (&ah)[4], const unsigned (&al)[4], unsigned bh0,
                                     unsigned bh1, unsigned bl0, unsigned bl1) {
  hmma_tf32(c, al, bh0, bh1);
  hmma_tf32(c, ah, bl0, bl1);
  hmma_tf32(c, ah, bh0, bh1);
}

template <int N, bool UPDATE, bool BSIG = false>
__global__ void __launch_bounds__(Ws32Cfg<N>::NT, 1)
    dg_stage_ws32(const StageParams<float> p, const float* __restrict__ opsA, int64_t t_begin, int64_t t_count) {
  using C = Ws32Cfg<N>;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, M16 = C::M16, KV = C::KV, KL = C::KL;
  constexpr int E = C::E, LD = C::LD, LDF = C::LDF, S = C::S, TS = C::TS;
  extern __shared__ __align__(128) unsigned char smem_ws32[];
  unsigned char* smem = smem_ws32;
  pdl_trigger();
  float* sA = reinterpret_cast<float*>(smem + size_t(S) * C::SLOT);  // hi then lo
  int16_t* sFm = reinterpret_cast<int16_t*>(smem + size_t(S) * C::SLOT + C::A_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(S) * C::SLOT + C::A_BYTES + C::FM_BYTES);
  uint64_t* bar_load = bars;
  uint64_t* bar_tr = bars + S;
  uint64_t* bar_full = bars + 2 * S;
  uint64_t* bar_empty = bars + 3 * S;
  auto sU = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_U); };
  auto sR = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_R); };
  auto sG = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_G); };
  auto sI = [&](int s) { return reinterpret_cast<int32_t*>(smem + size_t(s) * C::SLOT + C::OFF_I); };
  auto sF = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_F); };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool res_in = UPDATE && !p.first_stage;
  const int64_t J = t_count > blockIdx.x ? (t_count - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t kend = p.k_begin + p.K;
  auto tile_of = [&](int64_t j) { return t_begin + blockIdx.x + j * gridDim.x; };
  auto count_of = [&](int64_t tile) {
    const int64_t k0 = tile * E;
    return int(kend - k0 < E ? kend - k0 : E);
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_load + s, 1);
      mbar_init(bar_tr + s, C::PT);
      mbar_init(bar_full + s, C::PT);
      mbar_init(bar_empty + s, C::MW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int m = tid; m < NF; m += C::NT) sFm[m] = p.fmask[m];
  if constexpr (C::OPS_SMEM) {
    // hi/lo operators into shared memory: 16-byte cp.async chunks (rows are 16-B aligned)
    static_assert(KV % 4 == 0 && KL % 4 == 0 && C::LDA % 4 == 0 && C::LDL % 4 == 0, "16-B operator rows");
    for (int h = 0; h < 2; ++h) {
      const float* src = opsA + size_t(h) * C::OPS_ONE;
      float* dst = sA + h * C::A_ONE;
      for (int w = tid; w < 3 * M16 * KV / 4; w += C::NT) {
        const int r = (4 * w) / KV, k = 4 * w - r * KV;
        cp_async16(dst + r * C::LDA + k, src + 4 * w);
      }
      for (int w = tid; w < M16 * KL / 4; w += C::NT) {
        const int r = (4 * w) / KL, k = 4 * w - r * KL;
        cp_async16(dst + 3 * M16 * C::LDA + r * C::LDL + k, src + 3 * M16 * KV + 4 * w);
      }
    }
    cp_commit();
    cp_wait<0>();
  }
  __syncthreads();
  pdl_wait();  // the previous stage's fields are complete from here on

  if (warp == C::MW) {
    // ===================== TMA loader warp (one lane) =====================
    if (lane == 0) {
      const int64_t nbl = BSIG ? bsig_ctiles(p.bsig_tiles) : 0;  // boundary tiles (multi-rank signal)
      for (int64_t j = 0; j < J; ++j) {
        const int s = int(j % S);
        mbar_wait(bar_empty + s, (unsigned(j / S) & 1) ^ 1);
        if constexpr (BSIG) loader_signal_after_wait(p.bsig, nbl, j, S);
        const int64_t tile = tile_of(j);
        unsigned bytes = TS * 4 + C::GEOT * 4 + C::IDXT * 4;
        if (C::RES_SMEM && res_in) bytes += TS * 4;
        mbar_arrive_tx(bar_load + s, bytes);
        bulk_g2s(sU(s), p.u_in + tile * TS, TS * 4, bar_load + s);
        if (C::RES_SMEM && res_in) bulk_g2s(sR(s), p.res + tile * TS, TS * 4, bar_load + s);
        bulk_g2s(sG(s), p.geo + tile * C::GEOT, C::GEOT * 4, bar_load + s);
        bulk_g2s(sI(s), p.gidx + tile * C::IDXT, C::IDXT * 4, bar_load + s);
      }
      if constexpr (BSIG) loader_signal_tail(bar_empty, p.bsig, nbl, J, S);
    }
  } else if (warp > C::MW) {
    // ============================ flux warps ============================
    const int ptid = tid - 32 * (C::MW + 1);
    auto traces = [&](int64_t j) {
      const int s = int(j % S);
      mbar_wait(bar_load + s, unsigned(j / S) & 1);
      const int32_t* I = sI(s);
      float* F = sF(s);
      for (int w = ptid; w < E * NF; w += C::PT) {
        const int32_t gi = I[w];
        if (gi >= 0) {  // intra-tile faces (negative codes) need no gather
          const int e = w / NF, m = w - e * NF;
          const bool ghost = gi >= p.ghost_base;
          const float* src = p.u_in + gi;
          const int cb = 24 * (e >> 2) + 2 * (e & 3);
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            const int co = 8 * (c >> 1) + (c & 1);
            cp_async4(F + (cb + co) * LDF + m, src + (ghost ? c * Nfp : co * LD));
          }
        }
      }
      cp_async_mbar_arrive(bar_tr + s);
    };
    auto flux = [&](int64_t j) {
      const int s = int(j % S);
      mbar_wait(bar_tr + s, unsigned(j / S) & 1);
      const int ne = count_of(tile_of(j));
      const float* U = sU(s);
      const float* Gm = sG(s);
      const int32_t* I = sI(s);
      float* F = sF(s);
      for (int w = ptid; w < E * NF; w += C::PT) {
        const int e = w / NF, m = w - e * NF, f = m / Nfp;
        const int cb = 24 * (e >> 2) + 2 * (e & 3);
        float fl[6] = {0, 0, 0, 0, 0, 0};
        if (e < ne) {
          const float* g = Gm + e * GEO_W + 9 + 4 * f;
          const float nx = g[0], ny = g[1], nz = g[2], fs = g[3];
          const int nM = sFm[m];
          float uM[6], dE[3], dH[3];
#pragma unroll
          for (int c = 0; c < 6; ++c) uM[c] = U[(cb + 8 * (c >> 1) + (c & 1)) * LD + nM];
          const int32_t gi = I[w];
          if (TileLayout::is_intra(gi)) {  // neighbour in this tile: u+ from shared memory
            const int e2 = TileLayout::intra_e(gi), n2 = TileLayout::intra_n(gi);
            const int cb2 = 24 * (e2 >> 2) + 2 * (e2 & 3);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              dE[c] = U[(cb2 + 8 * (c >> 1) + (c & 1)) * LD + n2] - uM[c];
              dH[c] = U[(cb2 + 8 * ((c + 3) >> 1) + ((c + 3) & 1)) * LD + n2] - uM[c + 3];
            }
          } else if (gi >= 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              dE[c] = F[(cb + 8 * (c >> 1) + (c & 1)) * LDF + m] - uM[c];
              dH[c] = F[(cb + 8 * ((c + 3) >> 1) + ((c + 3) & 1)) * LDF + m] - uM[c + 3];
            }
          } else {  // PEC wall: E+ = -E-, H+ = H-
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              dE[c] = -2.0f * uM[c];
              dH[c] = 0.0f;
            }
          }
          maxwell_flux<float>(nx, ny, nz, p.alpha, dE, dH, fl);
          const float sc = fs * 0.5f;
#pragma unroll
          for (int c = 0; c < 6; ++c) fl[c] *= sc;
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) F[(cb + 8 * (c >> 1) + (c & 1)) * LDF + m] = fl[c];
      }
      // zero the K padding of the face buffer (lift K = KL >= NF)
      if constexpr (KL > NF) {
        for (int w = ptid; w < 6 * E * (KL - NF); w += C::PT) {
          const int col = w / (KL - NF), k = NF + (w - col * (KL - NF));
          F[col * LDF + k] = 0.0f;
        }
      }
      mbar_arrive(bar_full + s);
    };
    for (int64_t t = 0; t < C::LA && t < J; ++t) traces(t);
    for (int64_t j = 0; j < J; ++j) {
      if (C::LA == 0) {
        traces(j);
        flux(j);
      } else {
        flux(j);
        if (j + C::LA < J) traces(j + C::LA);
      }
    }
  } else {
    // ============================= MMA warps =============================
    const int gid = lane >> 2, tig = lane & 3;
    const int64_t total = J * C::T;
    int64_t released = 0, waited = -1, lwaited = -1;
    auto release = [&](int64_t jj) {
      if (waited < jj) {
        mbar_wait(bar_full + int(jj % S), unsigned(jj / S) & 1);
        waited = jj;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + int(jj % S));
    };
    const float* Ahi = C::OPS_SMEM ? sA : opsA;
    const float* Alo = C::OPS_SMEM ? sA + C::A_ONE : opsA + C::OPS_ONE;
    constexpr int lda = C::OPS_SMEM ? C::LDA : KV;
    constexpr int ldl = C::OPS_SMEM ? C::LDL : KL;
    constexpr int l0 = 3 * M16 * lda;  // LIFT offset within an operator copy
    auto ldA = [&](const float* base, int idx) -> float {
      if constexpr (C::OPS_SMEM)
        return base[idx];
      else
        return __ldg(base + idx);
    };
    for (int64_t q = warp; q < total; q += C::MW) {
      const int64_t j = q / C::T;
      const int task = int(q - j * C::T);
      while (released < j) release(released++);
      const int s = int(j % S);
      // volume needs only the loaded tile (load[s]); the face buffer (full[s]) is waited for
      // before the lift (see stage_ws.cuh)
      if (lwaited < j) {
        if (waited < j) mbar_wait(bar_load + s, unsigned(j / S) & 1);
        lwaited = j;
      }
      const int64_t tile = tile_of(j);
      const int ne = count_of(tile);
      const int t = task % C::MT, g = task / C::MT;
      const int r0 = 16 * t + gid;  // rows r0 and r0 + 8
      const float* U = sU(s);
      const float* F = sF(s);
      float acc[3][3][4];
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) acc[b][nt][0] = acc[b][nt][1] = acc[b][nt][2] = acc[b][nt][3] = 0.0f;
      float rpre[2][6];  // residual prefetch (RES_PREFETCH): rows r0, r0 + 8
      if constexpr (UPDATE && C::RES_PREFETCH) {
        const int e = 4 * g + tig;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 6; ++c)
            rpre[h][c] = (res_in && r0 + 8 * h < Np && e < ne)
                             ? p.res[tile * TS + r0 + 8 * h +
                                     int64_t(24 * g + 8 * (c >> 1) + 2 * tig + (c & 1)) * LD]
                             : 0.0f;
      }
      const float* bp = U + (24 * g + gid) * LD + tig;
#ifndef DG_W32_GUNROLL
#define DG_W32_GUNROLL (N == 8 ? 4 : 8)  // measured, profiles/r1_unroll_sweep.jsonl (2/2 before: N = 4 -3 %, N = 5 -2 %)
#endif
      constexpr int kVolUnroll = DG_W32_GUNROLL;
#pragma unroll kVolUnroll
      for (int kk = 0; kk < KV; kk += 8) {
        unsigned bh[3][2], bl[3][2];
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) {
          // node rows k >= Np are layout padding: masked (NaN-poisoned padding test)
          tf32_split((kk + 4 <= Np || kk + tig < Np) ? bp[nt * 8 * LD + kk] : 0.0f, bh[nt][0], bl[nt][0]);
          tf32_split((kk + 8 <= Np || kk + 4 + tig < Np) ? bp[nt * 8 * LD + kk + 4] : 0.0f, bh[nt][1], bl[nt][1]);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int rb = b * M16 + r0;
          unsigned ah[4], al[4];
          ah[0] = __float_as_uint(ldA(Ahi, rb * lda + kk + tig));
          ah[1] = __float_as_uint(ldA(Ahi, (rb + 8) * lda + kk + tig));
          ah[2] = __float_as_uint(ldA(Ahi, rb * lda + kk + tig + 4));
          ah[3] = __float_as_uint(ldA(Ahi, (rb + 8) * lda + kk + tig + 4));
          al[0] = __float_as_uint(ldA(Alo, rb * lda + kk + tig));
          al[1] = __float_as_uint(ldA(Alo, (rb + 8) * lda + kk + tig));
          al[2] = __float_as_uint(ldA(Alo, rb * lda + kk + tig + 4));
          al[3] = __float_as_uint(ldA(Alo, (rb + 8) * lda + kk + tig + 4));
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) mma3(acc[b][nt], ah, al, bh[nt][0], bh[nt][1], bl[nt][0], bl[nt][1]);
        }
      }
      // chain rule + curl for rows r0 (h=0) and r0+8 (h=1), element 4g+tig
      float r[3][4];
      {
        const float* Gm = sG(s) + (4 * g + tig) * GEO_W;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float dx[6], dy[6], dz[6];
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            const int i = 2 * h + (c & 1);
            const float ur = acc[0][c >> 1][i], us = acc[1][c >> 1][i], ut = acc[2][c >> 1][i];
            dx[c] = Gm[0] * ur + Gm[3] * us + Gm[6] * ut;
            dy[c] = Gm[1] * ur + Gm[4] * us + Gm[7] * ut;
            dz[c] = Gm[2] * ur + Gm[5] * us + Gm[8] * ut;
          }
          r[0][2 * h + 0] = dy[5] - dz[4];
          r[0][2 * h + 1] = dz[3] - dx[5];
          r[1][2 * h + 0] = dx[4] - dy[3];
          r[1][2 * h + 1] = -(dy[2] - dz[1]);
          r[2][2 * h + 0] = -(dz[0] - dx[2]);
          r[2][2 * h + 1] = -(dx[1] - dy[0]);
        }
      }
      if (waited < j) {
        mbar_wait(bar_full + s, unsigned(j / S) & 1);
        waited = j;
      }
      // lift: r += LIFT . Flux  (3xTF32)
      const float* fp = F + (24 * g + gid) * LDF + tig;
#ifndef DG_W32_LUNROLL
#define DG_W32_LUNROLL (N == 8 ? 4 : 8)
#endif
      constexpr int kLiftUnroll = DG_W32_LUNROLL;
#pragma unroll kLiftUnroll
      for (int kk = 0; kk < KL; kk += 8) {
        unsigned ah[4], al[4];
        ah[0] = __float_as_uint(ldA(Ahi, l0 + r0 * ldl + kk + tig));
        ah[1] = __float_as_uint(ldA(Ahi, l0 + (r0 + 8) * ldl + kk + tig));
        ah[2] = __float_as_uint(ldA(Ahi, l0 + r0 * ldl + kk + tig + 4));
        ah[3] = __float_as_uint(ldA(Ahi, l0 + (r0 + 8) * ldl + kk + tig + 4));
        al[0] = __float_as_uint(ldA(Alo, l0 + r0 * ldl + kk + tig));
        al[1] = __float_as_uint(ldA(Alo, l0 + (r0 + 8) * ldl + kk + tig));
        al[2] = __float_as_uint(ldA(Alo, l0 + r0 * ldl + kk + tig + 4));
        al[3] = __float_as_uint(ldA(Alo, l0 + (r0 + 8) * ldl + kk + tig + 4));
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) {
          unsigned bh0, bl0, bh1, bl1;
          tf32_split(fp[nt * 8 * LDF + kk], bh0, bl0);
          tf32_split(fp[nt * 8 * LDF + kk + 4], bh1, bl1);
          mma3(r[nt], ah, al, bh0, bh1, bl0, bl1);
        }
      }
      // LSERK update / RHS store (tiled layout), rows r0 and r0+8
      const int e = 4 * g + tig;
      if (e < ne) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = r0 + 8 * h;
          if (row < Np) {
            const int64_t tb = tile * TS + row;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              const int col = 24 * g + 8 * (c >> 1) + 2 * tig + (c & 1);
              const int64_t idx = tb + int64_t(col) * LD;
              const float rhs = r[c >> 1][2 * h + (c & 1)];
              if (UPDATE) {
                float rold = 0.0f;
                if constexpr (C::RES_SMEM) {
                  if (res_in) rold = sR(s)[col * LD + row];
                } else if constexpr (C::RES_PREFETCH) {
                  rold = rpre[h][c];
                } else {
                  if (res_in) rold = p.res[idx];
                }
                const float rr = p.rk_a * rold + p.dt * rhs;
                p.res[idx] = rr;
                p.u_out[idx] = U[col * LD + row] + p.rk_b * rr;
              } else {
                p.rhs_out[idx] = rhs;
              }
            }
          }
        }
      }
    }
    while (released < J) release(released++);
  }
}

template <int N>
void launch_stage_ws32(const StageParams<float>& p, const float* opsA, int mode, cudaStream_t st) {
  using C = Ws32Cfg<N>;
  static PerDevice pd;
  const int sms = sms_for_device(pd, [] {
      cudaFuncSetAttribute(dg_stage_ws32<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
      cudaFuncSetAttribute(dg_stage_ws32<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
      cudaFuncSetAttribute(dg_stage_ws32<N, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
  });
  if (p.K <= 0) return;
  const int64_t t0 = p.k_begin / C::E;
  const int64_t tc = (p.k_begin + p.K + C::E - 1) / C::E - t0;
  const int cap = sms - p.sm_reserve > 1 ? sms - p.sm_reserve : 1;  // SMs left to concurrent NCCL kernels
  const unsigned grid = unsigned(tc < cap ? tc : cap);
  if (mode == 1 && p.bsig)
    launch_pdl(true, dg_stage_ws32<N, true, true>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
  else if (mode == 1)
    launch_pdl(true, dg_stage_ws32<N, true>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
  else
    launch_pdl(true, dg_stage_ws32<N, false>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
}

template <int N>
TileLayout ws32_layout() {
  using C = Ws32Cfg<N>;
  TileLayout L;
  L.E = C::E;
  L.LD = C::LD;
  L.perm = 1;
  L.TS = C::TS;
  return L;
}

// host: padded 3xTF32 operator buffer (hi then lo), from row-major FP64 Dr|Ds|Dt ([Np][Np]) and LIFT ([Np][4Nfp])
template <int N>
void ws32_ops(const double* Dr, const double* Ds, const double* Dt, const double* LIFT, float* out) {
  using C = Ws32Cfg<N>;
  constexpr int Np = C::Np, NF = C::NF, M16 = C::M16, KV = C::KV, KL = C::KL;
  auto tf32 = [](double v) -> float {  // round-to-nearest into 10 explicit mantissa bits (matches cvt.rna)
    float f = float(v);
    unsigned u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) {
      u += 0x1000u;
      u &= 0xffffe000u;
    }
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  for (size_t i = 0; i < 2 * C::OPS_ONE; ++i) out[i] = 0.0f;
  const double* D[3] = {Dr, Ds, Dt};
  for (int b = 0; b < 3; ++b)
    for (int i = 0; i < Np; ++i)
      for (int k = 0; k < Np; ++k) {
        const double v = D[b][i * Np + k];
        const float hi = tf32(v);
        out[(size_t(b) * M16 + i) * KV + k] = hi;
        out[C::OPS_ONE + (size_t(b) * M16 + i) * KV + k] = tf32(v - double(hi));
      }
  for (int i = 0; i < Np; ++i)
    for (int k = 0; k < NF; ++k) {
      const double v = LIFT[i * NF + k];
      const float hi = tf32(v);
      out[size_t(3) * M16 * KV + size_t(i) * KL + k] = hi;
      out[C::OPS_ONE + size_t(3) * M16 * KV + size_t(i) * KL + k] = tf32(v - double(hi));
    }
}

}  // namespace dg
