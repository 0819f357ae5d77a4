// TC variant (FP32, N <= 4): the stage kernel on the 5th-generation tensor cores.
// tcgen05.mma kind::tf32 with operands in shared memory (K-major, SWIZZLE_NONE
// canonical core-matrix layout, described by UMMA smem descriptors) and the FP32
// accumulators in tensor memory, as 3xTF32:
//     A.B ~= A_hi.B + A_lo.B + A_hi.B_lo        (B_lo = B - trunc_tf32(B))
// The hardware truncates FP32 operands to TF32 (measured: tools/tcgen05_probe.cu),
// so B itself serves as B_hi.  Validated numerics: 1e-6 relative vs FP64.
//
//   volume (a1): D_V[M_V x 6E] = [Dr;Ds;Dt] (rows b*Np+i, M_V = 64|128) . U (K = KV)
//   lift   (a4): D_L[64 x 6E]  = LIFT (rows i) . Flux (K = KL)
// Columns = element-components (col = 6e + c), the paper's "fields in aggregate as
// a matrix".  The field tiles in HBM are stored as the smem image
// of the B operand (TileLayout perm = 2), so one bulk copy moves a tile.
//
// Warp roles (one persistent CTA per SM, S-slot smem ring, mbarrier handshakes):
//   warp 0            TMA loader (lane 0): U, residual, geometry, gather indices
//   warps 1..8        flux (PW = 8): cp.async trace gather (LA tiles ahead) -> upwind/PEC
//                     flux in place (a2+a3) -> B_lo splits of U and Flux ->
//                     fence.proxy.async -> full[s]
//   warp 9            TMEM allocator + MMA issuer (lane 0): 3 x (KV/8 + KL/8)
//                     tcgen05.mma per tile into a double-buffered accumulator,
//                     tcgen05.commit -> acc_full[a]
//   warps 10..17      epilogue (EW = 8, two per TMEM lane quarter): tcgen05.ld rows ->
//                     smem staging (Y_V, Y_L), then per (node, element): chain rule +
//                     curl + lift + LSERK update (a5) into smem, bulk store of the
//                     u_out / res tiles, release acc_empty[a] and the ring slot empty[s].
#pragma once
#include <cuda_runtime.h>

#include "stage_ws32.cuh"

namespace dg {

template <int N>
struct TcCfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  static_assert(3 * Np <= 128 && Np <= 64, "TC kernel covers N <= 4");
  static constexpr int KV = (Np + 7) / 8 * 8;     // volume K (tf32 MMA K = 8)
  static constexpr int KL = (NF + 7) / 8 * 8;     // lift K
  static constexpr int MV = 3 * Np <= 64 ? 64 : 128;
  static constexpr int ML = 64;
  static constexpr int E = N <= 2 ? 16 : 8;       // 6E % 16 == 0
  static constexpr int COLS = 6 * E;
  static constexpr int S = N <= 3 ? 3 : 2;        // ring slots (smem budget)
  static constexpr int LA = S - 2;                 // trace lookahead
  static constexpr int PW = 8;                     // flux warps
  static constexpr int EW = 8;                     // epilogue warps (two per TMEM lane quarter)
  static constexpr int W_LOAD = 0, W_FLUX0 = 1, W_MMA = 1 + PW, W_EPI0 = 2 + PW;
  static constexpr int NT = 32 * (W_EPI0 + EW);
  static constexpr int PT = 32 * PW;
  static constexpr int ET = 32 * EW;
  static constexpr int TS = COLS * KV;             // floats per field tile (B image)
  static constexpr int FS = COLS * KL;             // floats per face-buffer tile
  static constexpr int GEOT = E * GEO_W;
  static constexpr int IDXT = E * NF;
  static constexpr int TMEM_COLS = 2 * 2 * COLS <= 256 ? 256 : 512;
  // slot carve-up (bytes; 128-B aligned pieces for the descriptors)
  static constexpr int al128(int b) { return (b + 127) / 128 * 128; }
  static constexpr int OFF_U = 0;
  static constexpr int OFF_UL = OFF_U + al128(TS * 4);
  static constexpr int OFF_R = OFF_UL + al128(TS * 4);
  static constexpr int OFF_F = OFF_R + al128(TS * 4);
  static constexpr int OFF_FL = OFF_F + al128(FS * 4);
  static constexpr int OFF_G = OFF_FL + al128(FS * 4);
  static constexpr int OFF_I = OFF_G + al128(GEOT * 4);
  static constexpr int SLOT = OFF_I + al128(IDXT * 4);
  // shared: operators (hi, lo), epilogue staging Y_V [MV][COLS], Y_L [Np][COLS]
  static constexpr int AV = MV * KV, AL = ML * KL;  // floats per operator copy
  static constexpr int OFF_A = S * SLOT;
  static constexpr int OFF_YV = OFF_A + al128(2 * (AV + AL) * 4);
  static constexpr int OFF_YL = OFF_YV + al128(MV * (COLS + 1) * 4);
  static constexpr int OFF_FM = OFF_YL + al128(Np * (COLS + 1) * 4);
  static constexpr int OFF_BAR = OFF_FM + al128(NF * 2);
  static constexpr int NBAR = 4 * S + 4;
  static constexpr size_t SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  // global operator buffer (floats): [A_V hi | A_V lo | A_L hi | A_L lo], core-matrix layout
  static constexpr size_t OPS_FLOATS = size_t(2) * (AV + AL);
};

__device__ __forceinline__ int cm_off(int r, int k, int K) {  // K-major SWIZZLE_NONE canonical placement
  return ((r >> 3) * (K >> 2) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t umma_desc_kmajor(const void* smem, int K) {
  // LBO = 128 B (adjacent core matrices along K), SBO = (K/4)*128 B (adjacent 8-row groups)
  uint64_t d = uint64_t((smem_u32(smem) >> 4) & 0x3FFF);
  d |= uint64_t(128 >> 4) << 16;
  d |= uint64_t(((K / 4) * 128) >> 4) << 32;
  d |= uint64_t(1) << 46;  // sm100 descriptor version
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

#ifdef DG_WS_PROFILE
// 0 load wait empty | 1 flux wait load | 2 flux traces issue | 3 flux wait traces | 4 flux compute | 5 flux lo-split
// 6 mma wait full | 7 mma wait acc_empty | 8 mma issue | 9 epi wait acc_full | 10 epi pass1 | 11 epi pass2
// 12 epi store+release | 13 tiles (lane-0 of epilogue warp 0)
__device__ unsigned long long g_tc_prof[16];
#define TC_T(v) long long v = clock64()
#define TC_A(i, t0) \
  do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_tc_prof[i], (unsigned long long)(clock64() - (t0))); } while (0)
#else
#define TC_T(v) \
  do {          \
  } while (0)
#define TC_A(i, t0) \
  do {              \
  } while (0)
#endif

template <int N, bool UPDATE>
__global__ void __launch_bounds__(TcCfg<N>::NT, 1)
    dg_stage_tc(const StageParams<float> p, const float* __restrict__ opsA, int64_t t_begin, int64_t t_count) {
  using C = TcCfg<N>;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, KV = C::KV, KL = C::KL, E = C::E, COLS = C::COLS;
  constexpr int S = C::S, TS = C::TS;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  unsigned char* smem = smem_tc;
  pdl_trigger();
  auto sU = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_U); };
  auto sUL = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_UL); };
  auto sR = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_R); };
  auto sF = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_F); };
  auto sFL = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_FL); };
  auto sG = [&](int s) { return reinterpret_cast<float*>(smem + size_t(s) * C::SLOT + C::OFF_G); };
  auto sI = [&](int s) { return reinterpret_cast<int32_t*>(smem + size_t(s) * C::SLOT + C::OFF_I); };
  float* sAV = reinterpret_cast<float*>(smem + C::OFF_A);  // hi, then lo
  float* sAL = sAV + 2 * C::AV;                             // hi, then lo
  float* YV = reinterpret_cast<float*>(smem + C::OFF_YV);   // [MV][COLS+1]
  float* YL = reinterpret_cast<float*>(smem + C::OFF_YL);   // [Np][COLS+1]
  int16_t* sFm = reinterpret_cast<int16_t*>(smem + C::OFF_FM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* bar_load = bars;
  uint64_t* bar_tr = bars + S;
  uint64_t* bar_full = bars + 2 * S;
  uint64_t* bar_empty = bars + 3 * S;
  uint64_t* acc_full = bars + 4 * S;
  uint64_t* acc_empty = bars + 4 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

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
      mbar_init(bar_empty + s, C::EW);  // epilogue warps
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);   // tcgen05.commit
      mbar_init(acc_empty + a, C::EW);  // epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == C::W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int m = tid; m < NF; m += C::NT) sFm[m] = p.fmask[m];
  for (int w = tid; w < int(C::OPS_FLOATS); w += C::NT) cp_async4(sAV + w, opsA + w);
  cp_commit();
  cp_wait<0>();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the previous stage's fields are complete from here on

  if (warp == C::W_LOAD) {
    // ============================ loader ============================
    if (lane == 0) {
      for (int64_t j = 0; j < J; ++j) {
        const int s = int(j % S);
        TC_T(t0);
        mbar_wait(bar_empty + s, (unsigned(j / S) & 1) ^ 1);
        TC_A(0, t0);
        const int64_t tile = tile_of(j);
        unsigned bytes = TS * 4 + C::GEOT * 4 + C::IDXT * 4;
        if (res_in) bytes += TS * 4;
        mbar_arrive_tx(bar_load + s, bytes);
        bulk_g2s(sU(s), p.u_in + tile * TS, TS * 4, bar_load + s);
        if (res_in) bulk_g2s(sR(s), p.res + tile * TS, TS * 4, bar_load + s);
        bulk_g2s(sG(s), p.geo + tile * C::GEOT, C::GEOT * 4, bar_load + s);
        bulk_g2s(sI(s), p.gidx + tile * C::IDXT, C::IDXT * 4, bar_load + s);
      }
    }
  } else if (warp >= C::W_FLUX0 && warp < C::W_MMA) {
    // ============================= flux =============================
    const int ptid = tid - 32 * C::W_FLUX0;
    auto traces = [&](int64_t j) {
      const int s = int(j % S);
      TC_T(t0);
      mbar_wait(bar_load + s, unsigned(j / S) & 1);
      TC_A(1, t0);
      TC_T(t1);
      const int32_t* I = sI(s);
      float* F = sF(s);
      for (int w = ptid; w < E * NF; w += C::PT) {  // element-fastest: <= 2-way bank conflicts
        const int m = w / E, e = w - m * E;
        const int32_t gi = I[e * NF + m];
        if (gi >= 0) {  // intra-tile faces (negative codes) need no gather
          if (gi & TileLayout::GHOST_FLAG) {
            const float* src = p.u_in + p.ghost_base + (gi & ~TileLayout::GHOST_FLAG);
#pragma unroll
            for (int c = 0; c < 6; ++c) cp_async4(F + cm_off(6 * e + c, m, KL), src + c * Nfp);
          } else {
            const int k2 = gi >> 8, n2 = gi & 255;
            const float* src = p.u_in + int64_t(k2 / E) * TS;
            const int col0 = 6 * (k2 % E);
#pragma unroll
            for (int c = 0; c < 6; ++c) cp_async4(F + cm_off(6 * e + c, m, KL), src + cm_off(col0 + c, n2, KV));
          }
        }
      }
      cp_async_mbar_arrive(bar_tr + s);
      // B_lo split of the element tile for 3xTF32 (padding is zero, so is its split)
      const float* U = sU(s);
      float* UL = sUL(s);
      for (int w = ptid; w < TS; w += C::PT) UL[w] = tf32_lo(U[w]);
      TC_A(2, t1);
    };
    auto flux = [&](int64_t j) {
      const int s = int(j % S);
      TC_T(t0);
      mbar_wait(bar_tr + s, unsigned(j / S) & 1);
      TC_A(3, t0);
      TC_T(t1);
      const int ne = count_of(tile_of(j));
      const float* U = sU(s);
      const float* Gm = sG(s);
      const int32_t* I = sI(s);
      float* F = sF(s);
      for (int w = ptid; w < E * NF; w += C::PT) {  // element-fastest
        const int m = w / E, e = w - m * E, f = m / Nfp;
        float fl[6] = {0, 0, 0, 0, 0, 0};
        if (e < ne) {
          const float* g = Gm + e * GEO_W + 9 + 4 * f;
          const float nx = g[0], ny = g[1], nz = g[2], fs = g[3];
          const int nM = sFm[m];
          float uM[6], dE[3], dH[3];
#pragma unroll
          for (int c = 0; c < 6; ++c) uM[c] = U[cm_off(6 * e + c, nM, KV)];
          const int32_t gi = I[e * NF + m];
          if (TileLayout::is_intra(gi)) {  // neighbour in this tile: u+ from shared memory
            const int e2 = TileLayout::intra_e(gi), n2 = TileLayout::intra_n(gi);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              dE[c] = U[cm_off(6 * e2 + c, n2, KV)] - uM[c];
              dH[c] = U[cm_off(6 * e2 + c + 3, n2, KV)] - uM[c + 3];
            }
          } else if (gi >= 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              dE[c] = F[cm_off(6 * e + c, m, KL)] - uM[c];
              dH[c] = F[cm_off(6 * e + c + 3, m, KL)] - uM[c + 3];
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
        float* FL = sFL(s);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const int o = cm_off(6 * e + c, m, KL);
          F[o] = fl[c];
          FL[o] = tf32_lo(fl[c]);  // B_lo split for 3xTF32
        }
      }
      if constexpr (KL > NF) {  // zero the lift K padding (and its split)
        float* FL = sFL(s);
        for (int w = ptid; w < COLS * (KL - NF); w += C::PT) {
          const int cl = w / (KL - NF), k = NF + (w - cl * (KL - NF));
          F[cm_off(cl, k, KL)] = 0.0f;
          FL[cm_off(cl, k, KL)] = 0.0f;
        }
      }
      TC_A(4, t1);
      TC_T(t2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05.mma operands
      TC_A(5, t2);
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
  } else if (warp == C::W_MMA) {
    // ========================= MMA issuer =========================
    if (lane == 0) {
      constexpr uint32_t idv = idesc_tf32_f32(C::MV, COLS), idl = idesc_tf32_f32(C::ML, COLS);
      for (int64_t j = 0; j < J; ++j) {
        const int s = int(j % S), a = int(j & 1);
        TC_T(t0);
        mbar_wait(bar_full + s, unsigned(j / S) & 1);
        TC_A(6, t0);
        TC_T(t1);
        mbar_wait(acc_empty + a, (unsigned(j >> 1) & 1) ^ 1);
        TC_A(7, t1);
        TC_T(t2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dV = tmem + uint32_t(a * 2 * COLS), dL = dV + COLS;
        const float* U = sU(s);
        const float* UL = sUL(s);
        const float* F = sF(s);
        const float* FL = sFL(s);
        uint32_t acc = 0;
        for (int kk = 0; kk < KV; kk += 8) {
          const int o = (kk >> 2) * 32;  // two core matrices per K=8 step
          umma_tf32(dV, umma_desc_kmajor(sAV + o, KV), umma_desc_kmajor(U + o, KV), idv, acc);
          acc = 1;
          umma_tf32(dV, umma_desc_kmajor(sAV + C::AV + o, KV), umma_desc_kmajor(U + o, KV), idv, 1);
          umma_tf32(dV, umma_desc_kmajor(sAV + o, KV), umma_desc_kmajor(UL + o, KV), idv, 1);
        }
        acc = 0;
        for (int kk = 0; kk < KL; kk += 8) {
          const int o = (kk >> 2) * 32;
          umma_tf32(dL, umma_desc_kmajor(sAL + o, KL), umma_desc_kmajor(F + o, KL), idl, acc);
          acc = 1;
          umma_tf32(dL, umma_desc_kmajor(sAL + C::AL + o, KL), umma_desc_kmajor(F + o, KL), idl, 1);
          umma_tf32(dL, umma_desc_kmajor(sAL + o, KL), umma_desc_kmajor(FL + o, KL), idl, 1);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(acc_full + a))
                     : "memory");
        TC_A(8, t2);
      }
    }
  } else {
    // =========================== epilogue ===========================
    const int q = warp & 3;           // TMEM lane quarter of this warp
    const int half = (warp - C::W_EPI0) >> 2;  // which of the two warps of this quarter
    const int et = tid - 32 * C::W_EPI0;
    for (int64_t j = 0; j < J; ++j) {
      const int s = int(j % S), a = int(j & 1);
      const int64_t tile = tile_of(j);
      const int ne = count_of(tile);
      TC_T(t0);
      mbar_wait(acc_full + a, unsigned(j >> 1) & 1);
      TC_A(9, t0);
      TC_T(t1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // pass 1: TMEM rows -> shared staging (M=128: row = lane; M=64: row = 16*q + lane, lane < 16)
      const uint32_t colV = uint32_t(a * 2 * COLS), colL = colV + COLS;
      const int rowV = C::MV == 128 ? 32 * q + lane : (lane < 16 ? 16 * q + lane : -1);
      const int rowL = lane < 16 ? 16 * q + lane : -1;
#pragma unroll 1
      for (int c0 = 8 * half; c0 < COLS; c0 += 8 * (C::EW / 4)) {
        uint32_t v[8], l[8];
        const uint32_t base = tmem + (uint32_t(32 * q) << 16);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(base + colV + c0));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(l[0]), "=r"(l[1]), "=r"(l[2]), "=r"(l[3]), "=r"(l[4]), "=r"(l[5]), "=r"(l[6]), "=r"(l[7])
                     : "r"(base + colL + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (rowV >= 0 && rowV < 3 * Np)
#pragma unroll
          for (int i = 0; i < 8; ++i) YV[rowV * (COLS + 1) + c0 + i] = __uint_as_float(v[i]);
        if (rowL >= 0 && rowL < Np)
#pragma unroll
          for (int i = 0; i < 8; ++i) YL[rowL * (COLS + 1) + c0 + i] = __uint_as_float(l[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + a);
      asm volatile("bar.sync 2, %0;" ::"n"(C::ET) : "memory");  // staging complete
      TC_A(10, t1);
      TC_T(t2);
      // pass 2: per (node i, element e): chain rule + curl (eq. 4, 6) + lift + LSERK update.
      // Results overwrite the slot's tile images (u_out into U, res/rhs into R), which
      // are then written back with one bulk copy each.
      float* U = sU(s);
      float* R = sR(s);
      const float* Gm = sG(s);
      for (int pr = et; pr < Np * E; pr += C::ET) {  // element-fastest: <= 2-way bank conflicts
        const int i = pr / E, e = pr - i * E;
        const float* g = Gm + e * GEO_W;
        float dx[6], dy[6], dz[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const int col = 6 * e + c;
          const float ur = YV[i * (COLS + 1) + col], us = YV[(Np + i) * (COLS + 1) + col],
                      ut = YV[(2 * Np + i) * (COLS + 1) + col];
          dx[c] = g[0] * ur + g[3] * us + g[6] * ut;
          dy[c] = g[1] * ur + g[4] * us + g[7] * ut;
          dz[c] = g[2] * ur + g[5] * us + g[8] * ut;
        }
        float rhs[6];
        rhs[0] = dy[5] - dz[4];
        rhs[1] = dz[3] - dx[5];
        rhs[2] = dx[4] - dy[3];
        rhs[3] = -(dy[2] - dz[1]);
        rhs[4] = -(dz[0] - dx[2]);
        rhs[5] = -(dx[1] - dy[0]);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const int col = 6 * e + c;
          const float r = rhs[c] + YL[i * (COLS + 1) + col];
          const int o = cm_off(col, i, KV);
          if (UPDATE) {
            const float rold = res_in ? R[o] : 0.0f;
            const float rr = p.rk_a * rold + p.dt * r;
            R[o] = rr;
            U[o] = U[o] + p.rk_b * rr;
          } else {
            R[o] = r;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> bulk-store reads
      asm volatile("bar.sync 2, %0;" ::"n"(C::ET) : "memory");     // staging and slot tile images done
      TC_A(11, t2);
      TC_T(t3);
      if (et == 0) {
        // absent elements of a partial tile hold zero fields -> zero results; padding rows stay zero
        if (UPDATE) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.u_out + tile * TS),
                       "r"(smem_u32(U)), "r"(unsigned(TS * 4))
                       : "memory");
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.res + tile * TS),
                       "r"(smem_u32(R)), "r"(unsigned(TS * 4))
                       : "memory");
        } else {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.rhs_out + tile * TS),
                       "r"(smem_u32(R)), "r"(unsigned(TS * 4))
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem may be reused after this
      }
      asm volatile("bar.sync 2, %0;" ::"n"(C::ET) : "memory");
      if (lane == 0) mbar_arrive(bar_empty + s);
      TC_A(12, t3);
#ifdef DG_WS_PROFILE
      if (et == 0) atomicAdd(&g_tc_prof[13], 1ull);
#endif
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == C::W_MMA) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

#ifdef DG_WS_PROFILE
inline void tc_prof_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_tc_prof, sizeof(g_tc_prof)); }
inline void tc_prof_reset() {
  static unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
}
#endif

template <int N>
void launch_stage_tc(const StageParams<float>& p, const float* opsA, int mode, cudaStream_t st) {
  using C = TcCfg<N>;
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(dg_stage_tc<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaFuncSetAttribute(dg_stage_tc<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (p.K <= 0) return;
  const int64_t t0 = p.k_begin / C::E;
  const int64_t tc = (p.k_begin + p.K + C::E - 1) / C::E - t0;
  const unsigned grid = unsigned(tc < sms ? tc : sms);
  if (mode == 1)
    launch_pdl(true, dg_stage_tc<N, true>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
  else
    launch_pdl(true, dg_stage_tc<N, false>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
}

template <int N>
TileLayout tc_layout() {
  using C = TcCfg<N>;
  TileLayout L;
  L.E = C::E;
  L.LD = C::KV;
  L.perm = 2;
  L.TS = C::TS;
  return L;
}

// host: operators in the core-matrix layout, split for 3xTF32 with hardware truncation
// (hi = trunc_tf32(float(v)), lo = float(v - hi)): [A_V hi | A_V lo | A_L hi | A_L lo].
template <int N>
void tc_ops(const double* Dr, const double* Ds, const double* Dt, const double* LIFT, float* out) {
  using C = TcCfg<N>;
  constexpr int Np = C::Np, NF = C::NF, KV = C::KV, KL = C::KL;
  auto cm = [](int r, int k, int K) { return ((r >> 3) * (K >> 2) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); };
  auto trunc32 = [](double v) -> float {
    float f = float(v);
    unsigned u;
    std::memcpy(&u, &f, 4);
    u &= 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  for (size_t i = 0; i < C::OPS_FLOATS; ++i) out[i] = 0.0f;
  float* avh = out;
  float* avl = out + C::AV;
  float* alh = out + 2 * C::AV;
  float* all = alh + C::AL;
  const double* D[3] = {Dr, Ds, Dt};
  for (int b = 0; b < 3; ++b)
    for (int i = 0; i < Np; ++i)
      for (int k = 0; k < Np; ++k) {
        const double v = D[b][i * Np + k];
        const float hi = trunc32(v);
        avh[cm(b * Np + i, k, KV)] = hi;
        avl[cm(b * Np + i, k, KV)] = float(v - double(hi));
      }
  for (int i = 0; i < Np; ++i)
    for (int k = 0; k < NF; ++k) {
      const double v = LIFT[i * NF + k];
      const float hi = trunc32(v);
      alh[cm(i, k, KL)] = hi;
      all[cm(i, k, KL)] = float(v - double(hi));
    }
}

}  // namespace dg
