// WS variant (FP64, default): warp-specialized, mbarrier-pipelined stage kernel.
//
// One persistent CTA per SM walks its element tiles through an S-slot ring:
//
//   producer warps (PW):  TMA bulk copies of the tile's U, residual, geometry and
//                         gather indices (one elected thread, complete_tx on
//                         `load[s]`)  ->  cp.async gather of the exterior traces u+
//                         straight into the face buffer (a2, PAPER.md:236-255,
//                         1266-1270; completion tracked by `tr[s]`)  ->  upwind/PEC
//                         flux x Fscale/2 in place (a3, fig:flux-code a)  ->
//                         arrive `full[s]`.
//   MMA warps (MW, one or two per SMSP):  stream (m-tile, 4-element group) tasks
//                         continuously across tiles: [Dr;Ds;Dt] . U on DMMA (a1),
//                         chain rule + curl thread-local, LIFT . Flux on DMMA
//                         (a4), LSERK update (a5) from the accumulators; arrive
//                         `empty[s]` after their last task of a tile.
//
// The field arrays use the tiled layout of TileLayout (perm = 1): each tile is the
// shared-memory image of the MMA B operand, so its load is a single bulk copy.
// Column permutation: see stage_mma.cuh — every accumulator thread owns all six
// components of one element at one node row.
//
// Measured B200 DMMA.8x8x4: 26-cycle latency, one issue per 16 cycles per SMSP;
// four warps (one per SMSP) with >= 2 independent chains saturate the FP64 tensor
// pipe (tools/dmma_lat.cu), hence MW = 4 when the operators sit in shared memory.
#pragma once
#include <cuda_runtime.h>

#include "stage_mma.cuh"

namespace dg {

__host__ __device__ constexpr int ldx(int x) {  // smallest >= x with x % 16 in {4, 12}: conflict-free 8x4 fragments
  return (x % 16 == 4 || x % 16 == 12) ? x : ldx(x + 4);
}
__host__ __device__ constexpr int r16(int bytes) { return (bytes + 15) / 16 * 16; }

template <int N, int NC = 6>
struct WsCfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  // NC fields per element (6 Maxwell; 4 linear acoustics, NEXT-3): a 4-element column group is
  // GW = 4 NC columns = NC / 2 DMMA n-tiles, thread (gid, tig) owning all NC components of
  // element 4g + tig at node row 8t + gid
  static constexpr int GW = 4 * NC, NT3 = NC / 2;
  static constexpr int M8 = (Np + 7) / 8 * 8;
  static constexpr int MT = M8 / 8;
  static constexpr int KV = (Np + 3) / 4 * 4;
  static constexpr int KL = NF;
  static constexpr int LD = ldx(KV);
  static constexpr int LDF = ldx(NF);
  static constexpr int LDA = ldx(KV);
  static constexpr int LDL = ldx(NF);
  // per-order configuration: tile size, ring depth, warp roles,
  // operator residency, residual staging
  // tuning builds (tools/tune_ws.sh, NEXT-4): -DDG_WS_TUNE_N=n -DDG_WS_E=e -DDG_WS_S=s override
  // the tile size / ring depth of order n only
#ifdef DG_WS_TUNE_N
  static constexpr bool TUNED = N == DG_WS_TUNE_N;
#else
  static constexpr bool TUNED = false;
#endif
#ifdef DG_WS_E
  static constexpr int E_TUNE = DG_WS_E;
#else
  static constexpr int E_TUNE = 0;
#endif
#ifdef DG_WS_S
  static constexpr int S_TUNE = DG_WS_S;
#else
  static constexpr int S_TUNE = 0;
#endif
  // measured (NEXT-4 sweeps, profiles/r1_tile_sweep*.jsonl): N=3 E=4/S=8 beats E=8/S=5 by 6 %;
  // N=4 with the residual out of the ring (register prefetch) fits S=8 and a 4-tile trace
  // look-ahead (+3.4 %); N=7/8 prefer shallower rings with 11 MMA warps
  static constexpr int E = (TUNED && E_TUNE) ? E_TUNE : N == 1 ? 32 : N == 2 ? 16 : 4;
  static constexpr int S = (TUNED && S_TUNE) ? S_TUNE
                           : N == 2 ? 4 : N == 3 ? 8 : N == 4 ? 8 : N == 5 ? 3 : N == 6 ? 3 : N == 7 ? 3 : 2;
#ifdef DG_WS_LA
  static constexpr int LA_TUNE = DG_WS_LA;
#else
  static constexpr int LA_TUNE = 0;
#endif
  // trace gathers issued LA tiles ahead of the flux (LA <= S - 2: the slot of tile j+LA
  // must have been released by the MMA warps, which may still be on tile j-1)
  static constexpr int LA = (TUNED && LA_TUNE) ? LA_TUNE : N == 4 ? 4 : S - 2 < 2 ? S - 2 : 2;
  static_assert(LA <= S - 2 || S <= 2, "look-ahead beyond the ring");
#ifdef DG_WS_OPS
  static constexpr bool OPS_SMEM = TUNED ? bool(DG_WS_OPS) : N <= 5;
#else
  static constexpr bool OPS_SMEM = N <= 5;
#endif
#ifdef DG_WS_RES
  static constexpr bool RES_SMEM = TUNED ? bool(DG_WS_RES) : N <= 3;
#else
  static constexpr bool RES_SMEM = N <= 3;
#endif
  // warp roles (measured, tools/gpu_tile_sweep.sh): >= 2 MMA warps per SMSP so one's epilogue
  // hides under the other's DMMAs; 11 for N >= 5, which keeps the CTA at 16 warps (a 17th
  // warp would cap registers at 96 per thread and force the residual prefetch off)
#ifdef DG_WS_MW
  static constexpr int MW = DG_WS_MW;
#else
  static constexpr int MW = N >= 5 ? 11 : 8;
#endif
#ifdef DG_WS_PW
  static constexpr int PW = DG_WS_PW;  // flux warps (trace gather + flux); plus one dedicated TMA loader warp
#else
  static constexpr int PW = N <= 3 ? 6 : 4;  // N = 1, 2: +9 % over 4 flux warps
#endif
  // residual from global memory: prefetched into registers at task start, unless a
  // 17-warp CTA (register cap 96 per thread: the file is split per SMSP) would spill
  static constexpr bool RES_PREFETCH = !RES_SMEM && (N <= 5 || MW + 1 + PW <= 16);
  static constexpr int NT = 32 * (MW + 1 + PW);
  static constexpr int PT = 32 * PW;
  // MMA warps start the volume contraction once the tile is loaded and wait for the flux
  // only before the lift; measured (profiles/r1_early_volume.jsonl): N = 5 +4.6 %, N = 4
  // +1.3 %, N = 3 -4.4 % (kept off there), others within noise
#ifdef DG_WS_EARLY
  static constexpr bool EARLY_VOL = TUNED ? bool(DG_WS_EARLY) : N != 3;
#else
  static constexpr bool EARLY_VOL = N != 3;
#endif
  static constexpr int G = E / 4;
  static constexpr int T = MT * G;  // tasks per tile
  static constexpr int TS = NC * E * LD;
  static constexpr int GEOT = E * GEO_W;
  static constexpr int IDXT = E * NF;
  // slot carve-up (bytes, 16-B aligned pieces)
  static constexpr int OFF_U = 0;
  static constexpr int OFF_R = OFF_U + r16(TS * 8);
  static constexpr int OFF_G = OFF_R + (RES_SMEM ? r16(TS * 8) : 0);
  static constexpr int OFF_I = OFF_G + r16(GEOT * 8);
  static constexpr int OFF_F = OFF_I + r16(IDXT * 4);
  static constexpr int SLOT = OFF_F + r16(NC * E * LDF * 8);
  static constexpr int A_BYTES = OPS_SMEM ? r16((3 * M8 * LDA + M8 * LDL) * 8) : 0;
  static constexpr int FM_BYTES = r16(NF * 2);
  // mbarriers load/tr/full/empty [S]
  static constexpr int BAR_BYTES = 4 * S * 8;
  static constexpr size_t SMEM_BYTES = size_t(S) * SLOT + A_BYTES + FM_BYTES + BAR_BYTES;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(E % 4 == 0, "tile = whole 4-element column groups");
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Multi-rank stages ("boundary-first stage"): the tiles [0, p.bsig_tiles) of the
// launch hold the partition-boundary elements.  bsig_ctiles() is the number of them this CTA
// processes (its first tiles, j < nb).  Once the CTA has written all of them, one thread adds nb to
// *p.bsig (GPU-scope fence first); the comm stream waits for the total (cuStreamWaitValue32: a
// front-end wait, no SM is held) and then packs and sends the next stage's traces while the interior
// tiles are still running.  No kernel ever waits on it.
__device__ __forceinline__ int64_t bsig_ctiles(int64_t nbt) {
  return nbt > int64_t(blockIdx.x) ? (nbt - int64_t(blockIdx.x) + gridDim.x - 1) / gridDim.x : 0;
}
// Ring kernels (WS, WS32, FFMA): the TMA loader lane signals instead of the store warps.  The store
// warps release tile jj with an mbarrier arrive (release, CTA scope) after their last store of it; the
// loader acquires that phase (its slot-reuse wait, or an explicit wait after its loop), then fences at
// GPU scope (cumulative over the acquired stores) and adds nb.  A named barrier in the store warps'
// release path cost 3-6 % at N = 1..3 even when not taken, so the signal lives here, and only in the
// BSIG = true kernel instances (multi-rank stages; the code alone cost ~2 % in the single-rank ones).
// Call right after the loader's slot-reuse wait for tile j, which acquired the release of tile j - S.
__device__ __forceinline__ void loader_signal_after_wait(unsigned* bsig, int64_t nb, int64_t j, int S) {
  if (bsig && j - S == nb - 1) {
    __threadfence();
    atomicAdd(bsig, unsigned(nb));
  }
}
// after the loader's loop: boundary tiles among the CTA's last S tiles were never re-waited
__device__ __forceinline__ void loader_signal_tail(uint64_t* bar_empty, unsigned* bsig, int64_t nb, int64_t J, int S) {
  if (bsig && nb > 0 && nb - 1 + S >= J) {
    mbar_wait(bar_empty + int((nb - 1) % S), unsigned((nb - 1) / S) & 1);
    __threadfence();
    atomicAdd(bsig, unsigned(nb));
  }
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// ---------------------------------------------------------------- profiling (DG_WS_PROFILE builds only)
#ifdef DG_WS_PROFILE
// per-role cycle counters summed over all CTAs:
// 0 prod wait empty, 1 prod wait load, 2 prod wait traces, 3 prod flux compute, 4 prod trace issue,
// 5 cons wait full, 6 cons task compute, 7 tiles, 8 tasks, 9 prod total, 10 cons total
__device__ unsigned long long g_ws_prof[16];
#define DG_T0() long long _t0 = clock64()
#define DG_ACC(i)                                                     \
  do {                                                                \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_ws_prof[i], (unsigned long long)(clock64() - _t0)); \
  } while (0)
#define DG_CNT(i, v)                                                  \
  do {                                                                \
    if (threadIdx.x == 0) atomicAdd(&g_ws_prof[i], (unsigned long long)(v)); \
  } while (0)
#else
#define DG_T0() \
  do {          \
  } while (0)
#define DG_ACC(i) \
  do {            \
  } while (0)
#define DG_CNT(i, v) \
  do {               \
  } while (0)
#endif

// ---------------------------------------------------------------- kernel
// Tiles [t_begin, t_begin + t_count) of the tiled arrays; p.k_begin/p.K give the
// element range (tile-aligned start) used to count elements in the last tile.
template <int N, bool UPDATE, int SYS = 0, bool BSIG = false>
__global__ void __launch_bounds__(WsCfg<N, System<SYS>::NC>::NT, 1)
    dg_stage_ws(const StageParams<double> p, const double* __restrict__ opsA, int64_t t_begin, int64_t t_count) {
  constexpr int NC = System<SYS>::NC, GW = 4 * NC, NT3 = NC / 2;
  using C = WsCfg<N, NC>;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, M8 = C::M8, KV = C::KV, KL = C::KL;
  constexpr int E = C::E, LD = C::LD, LDF = C::LDF, S = C::S, TS = C::TS;
  extern __shared__ __align__(128) unsigned char smem_ws[];
  unsigned char* smem = smem_ws;
  pdl_trigger();
  double* sA = reinterpret_cast<double*>(smem + size_t(S) * C::SLOT);
  int16_t* sFm = reinterpret_cast<int16_t*>(smem + size_t(S) * C::SLOT + C::A_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(S) * C::SLOT + C::A_BYTES + C::FM_BYTES);
  uint64_t* bar_load = bars;
  uint64_t* bar_tr = bars + S;
  uint64_t* bar_full = bars + 2 * S;
  uint64_t* bar_empty = bars + 3 * S;
  constexpr int NTK = C::NT;
  auto sU = [&](int s) { return reinterpret_cast<double*>(smem + size_t(s) * C::SLOT + C::OFF_U); };
  auto sR = [&](int s) { return reinterpret_cast<double*>(smem + size_t(s) * C::SLOT + C::OFF_R); };
  auto sG = [&](int s) { return reinterpret_cast<double*>(smem + size_t(s) * C::SLOT + C::OFF_G); };
  auto sI = [&](int s) { return reinterpret_cast<int32_t*>(smem + size_t(s) * C::SLOT + C::OFF_I); };
  auto sF = [&](int s) { return reinterpret_cast<double*>(smem + size_t(s) * C::SLOT + C::OFF_F); };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tiles of this CTA: t_begin + blockIdx.x + j * gridDim.x, j < J
  const int64_t J = t_count > blockIdx.x ? (t_count - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t JJ = J;
  const int64_t kend = p.k_begin + p.K;
  auto tile_of = [&](int64_t jj) { return t_begin + blockIdx.x + jj * gridDim.x; };
  const bool res_in = UPDATE && !p.first_stage;
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
  for (int m = tid; m < NF; m += NTK) sFm[m] = p.fmask[m];
  if constexpr (C::OPS_SMEM) {
    // 16-byte cp.async chunks (rows of KV, KL, LDA, LDL doubles are 16-B aligned)
    static_assert(KV % 2 == 0 && KL % 2 == 0 && C::LDA % 2 == 0 && C::LDL % 2 == 0, "16-B operator rows");
    for (int w = tid; w < 3 * M8 * KV / 2; w += NTK) {
      const int r = (2 * w) / KV, k = 2 * w - r * KV;
      cp_async16(sA + r * C::LDA + k, opsA + 2 * w);
    }
    const double* Lg = opsA + 3 * M8 * KV;
    for (int w = tid; w < M8 * KL / 2; w += NTK) {
      const int r = (2 * w) / KL, k = 2 * w - r * KL;
      cp_async16(sA + 3 * M8 * C::LDA + r * C::LDL + k, Lg + 2 * w);
    }
    cp_commit();
    cp_wait<0>();
  }
  __syncthreads();
  pdl_wait();  // the previous stage's fields are complete from here on

  if (warp == C::MW) {
    // ====================== TMA loader warp (one lane) ======================
    // Runs ahead of everybody, bounded only by free ring slots: tile j's bulk
    // loads are issued as soon as the MMA warps release tile j - S.
    if (lane == 0) {
      DG_T0();
      const int64_t nbl = BSIG ? bsig_ctiles(p.bsig_tiles) : 0;  // boundary tiles (multi-rank signal)
      for (int64_t j = 0; j < JJ; ++j) {
        const int s = int(j % S);
        const unsigned u = unsigned(j / S);
        {
          DG_T0();
          mbar_wait(bar_empty + s, (u & 1) ^ 1);
          DG_ACC(0);
        }
        if constexpr (BSIG) loader_signal_after_wait(p.bsig, nbl, j, S);
        const int64_t tile = tile_of(j);
        unsigned bytes = TS * 8 + C::GEOT * 8 + C::IDXT * 4;
        if (C::RES_SMEM && res_in) bytes += TS * 8;
        mbar_arrive_tx(bar_load + s, bytes);
        bulk_g2s(sU(s), p.u_in + tile * TS, TS * 8, bar_load + s);
        if (C::RES_SMEM && res_in) bulk_g2s(sR(s), p.res + tile * TS, TS * 8, bar_load + s);
        bulk_g2s(sG(s), p.geo + tile * C::GEOT, C::GEOT * 8, bar_load + s);
        bulk_g2s(sI(s), p.gidx + tile * C::IDXT, C::IDXT * 4, bar_load + s);
      }
      if constexpr (BSIG) loader_signal_tail(bar_empty, p.bsig, nbl, JJ, S);
    }
  } else if (warp > C::MW) {
    // ============================= flux warps =============================
    const int ptid = tid - 32 * (C::MW + 1);
    auto traces = [&](int64_t j) {  // all flux threads
      const int s = int(j % S);
      {
        DG_T0();
        mbar_wait(bar_load + s, unsigned(j / S) & 1);
        DG_ACC(1);
      }
      DG_T0();
      const int32_t* I = sI(s);
      double* F = sF(s);
      const double* uin = p.u_in;
      for (int w = ptid; w < E * NF; w += C::PT) {
        const int32_t gi = I[w];
        if (gi >= 0) {  // intra-tile faces (negative codes) need no gather
          const int e = w / NF, m = w - e * NF;
          const bool ghost = gi >= p.ghost_base;
          const double* src = uin + gi;
          const int cb = GW * (e >> 2) + 2 * (e & 3);
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int co = 8 * (c >> 1) + (c & 1);
            cp_async8(F + (cb + co) * LDF + m, src + (ghost ? c * Nfp : co * LD));
          }
        }
      }
      cp_async_mbar_arrive(bar_tr + s);
      DG_ACC(4);
    };
    auto flux = [&](int64_t j) {  // all flux threads
      const int s = int(j % S);
      {
        DG_T0();
        mbar_wait(bar_tr + s, unsigned(j / S) & 1);
        DG_ACC(2);
      }
      DG_T0();
      const int ne = count_of(tile_of(j));
      const double* U = sU(s);
      const double* Gm = sG(s);
      const int32_t* I = sI(s);
      double* F = sF(s);
      for (int w = ptid; w < E * NF; w += C::PT) {
        const int e = w / NF, m = w - e * NF, f = m / Nfp;
        const int cb = GW * (e >> 2) + 2 * (e & 3);
        auto col = [&](int base, int c) { return base + 8 * (c >> 1) + (c & 1); };
        double fl[6] = {0, 0, 0, 0, 0, 0};
        if (e < ne) {
          const double* g = Gm + e * GEO_W + 9 + 4 * f;
          const double nx = g[0], ny = g[1], nz = g[2], fs = g[3];
          const int nM = sFm[m];
          double uM[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) uM[c] = U[col(cb, c) * LD + nM];
          const int32_t gi = I[w];
          if constexpr (SYS == 0) {
            double dE[3], dH[3];
            if (TileLayout::is_intra(gi)) {  // neighbour in this tile: u+ from shared memory
              const int e2 = TileLayout::intra_e(gi), n2 = TileLayout::intra_n(gi);
              const int cb2 = GW * (e2 >> 2) + 2 * (e2 & 3);
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                dE[c] = U[col(cb2, c) * LD + n2] - uM[c];
                dH[c] = U[col(cb2, c + 3) * LD + n2] - uM[c + 3];
              }
            } else if (gi >= 0) {
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                dE[c] = F[col(cb, c) * LDF + m] - uM[c];
                dH[c] = F[col(cb, c + 3) * LDF + m] - uM[c + 3];
              }
            } else {  // PEC wall: E+ = -E-, H+ = H-
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                dE[c] = -2.0 * uM[c];
                dH[c] = 0.0;
              }
            }
            maxwell_flux<double>(nx, ny, nz, p.alpha, dE, dH, fl);
          } else {  // rigid wall (R17): p+ = p-, v+ = v- - 2 (n.v-) n
            double uP[NC];
            const bool wall = !TileLayout::is_intra(gi) && gi < 0;
            if (TileLayout::is_intra(gi)) {
              const int e2 = TileLayout::intra_e(gi), n2 = TileLayout::intra_n(gi);
              const int cb2 = GW * (e2 >> 2) + 2 * (e2 & 3);
#pragma unroll
              for (int c = 0; c < NC; ++c) uP[c] = U[col(cb2, c) * LD + n2];
            } else {
#pragma unroll
              for (int c = 0; c < NC; ++c) uP[c] = wall ? uM[c] : F[col(cb, c) * LDF + m];
            }
            const double ndv = nx * uM[1] + ny * uM[2] + nz * uM[3];
            const double dp = wall ? 0.0 : uP[0] - uM[0];
            double dv[3];
            dv[0] = wall ? -2.0 * ndv * nx : uP[1] - uM[1];
            dv[1] = wall ? -2.0 * ndv * ny : uP[2] - uM[2];
            dv[2] = wall ? -2.0 * ndv * nz : uP[3] - uM[3];
            acoustic_flux<double>(nx, ny, nz, p.alpha, dp, dv, fl);
          }
          const double sc = fs * 0.5;
#pragma unroll
          for (int c = 0; c < NC; ++c) fl[c] *= sc;
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) F[col(cb, c) * LDF + m] = fl[c];
      }
      DG_ACC(3);
      mbar_arrive(bar_full + s);
    };
    // flux warps: tile j's flux, then tile j+LA's trace gather (its bulk load was issued
    // by the loader warp as soon as a slot was free)
    DG_T0();
    DG_CNT(7, JJ);
    int64_t issued = 0;  // traces issued for positions < issued
    auto issue_upto = [&](int64_t lim) {
      while (issued < lim) traces(issued++);
    };
    for (int64_t j = 0; j < JJ; ++j) {
      const int64_t end = JJ;
      const bool first = j == 0;
      issue_upto(first ? (j + C::LA < end ? (C::LA > 0 ? j + C::LA : j + 1) : end) : j + 1);
      flux(j);
      issue_upto(j + 1 + C::LA < end ? j + 1 + C::LA : end);
    }
    DG_ACC(9);
  } else {
    // ============================= MMA warps =============================
    const int gid = lane >> 2, tig = lane & 3;
    const int64_t total = JJ * C::T;
    int64_t released = 0, waited = -1, lwaited = -1;
    auto release = [&](int64_t jj) {  // this warp is done with tile jj (waits for it to exist first)
      if (waited < jj) {
        mbar_wait(bar_full + int(jj % S), unsigned(jj / S) & 1);
        waited = jj;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + int(jj % S));
    };
    DG_T0();
    for (int64_t q = warp; q < total; q += C::MW) {
      const int64_t j = q / C::T;
      const int task = int(q - j * C::T);
      while (released < j) release(released++);
      const int s = int(j % S);
      // the volume contraction needs only the loaded tile (load[s]); the face buffer
      // (full[s]) is waited for just before the lift, so the first tile of a stage
      // overlaps its flux with the volume work.  (load[s] cannot be a phase ahead or
      // behind: this warp has passed full[] of tile j-S and not released tile j.)
      if (lwaited < j) {
        if (waited < j) mbar_wait((C::EARLY_VOL ? bar_load : bar_full) + s, unsigned(j / S) & 1);
        lwaited = j;
      }
#ifdef DG_WS_PROFILE
      long long _tc = clock64();
      if (lane == 0) atomicAdd(&g_ws_prof[8], 1ull);
#endif
      const int64_t tile = tile_of(j);
      const int ne = count_of(tile);
      const double rk_a = p.rk_a, rk_b = p.rk_b;
      double* const u_out = p.u_out;
      const int t = task % C::MT, g = task / C::MT;
      const int row = 8 * t + gid;
      const double* U = sU(s);
      const double* F = sF(s);
      double acc[3][NT3][2];
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int nt = 0; nt < NT3; ++nt) acc[b][nt][0] = acc[b][nt][1] = 0.0;
      // residual through global memory (!RES_SMEM): prefetched into registers now, used
      // in the update after the contractions (hides the load latency behind the DMMAs)
      double rpre[NC];
      if constexpr (UPDATE && C::RES_PREFETCH) {
        const int e = 4 * g + tig;
        const int64_t tb = tile * TS + 8 * t + gid;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          rpre[c] = (res_in && 8 * t + gid < Np && e < ne)
                        ? p.res[tb + int64_t(GW * g + 8 * (c >> 1) + 2 * tig + (c & 1)) * LD]
                        : 0.0;
      }
      const double* bp = U + (GW * g + gid) * LD + tig;
      if constexpr (C::OPS_SMEM) {
        const double* ap = sA + row * C::LDA + tig;
#pragma unroll
        for (int kk = 0; kk < KV; kk += 4) {
          const double ar = ap[kk], as = ap[M8 * C::LDA + kk], at = ap[2 * M8 * C::LDA + kk];
#pragma unroll
          for (int nt = 0; nt < NT3; ++nt) {
            // node rows k >= Np are layout padding: masked, so the K padding never multiplies
            // whatever the padding holds (NaN-poisoned padding test)
            const double bv = (kk + 4 <= Np || kk + tig < Np) ? bp[nt * 8 * LD + kk] : 0.0;
            dmma(acc[0][nt], ar, bv);
            dmma(acc[1][nt], as, bv);
            dmma(acc[2][nt], at, bv);
          }
        }
      } else {
        const double* ap = opsA + size_t(row) * KV + tig;
        // operators streamed through L1/L2 (N >= 6): deeper unrolling keeps more operator loads in
        // flight (profiles/r1_unroll_sweep.jsonl: N = 6 +4.5 %, 7 +7 %, 8 +10 %, 9 +4 % over 4/2)
#ifndef DG_WS_GUNROLL
        constexpr int GU = (N == 7 || N == 9) ? 16 : (N == 6 || N == 8) ? 12 : 4;
#else
        constexpr int GU = DG_WS_GUNROLL;
#endif
#pragma unroll GU
        for (int kk = 0; kk < KV; kk += 4) {
          const double ar = __ldg(ap + kk);
          const double as = __ldg(ap + size_t(M8) * KV + kk);
          const double at = __ldg(ap + size_t(2) * M8 * KV + kk);
#pragma unroll
          for (int nt = 0; nt < NT3; ++nt) {
            // node rows k >= Np are layout padding: masked, so the K padding never multiplies
            // whatever the padding holds (NaN-poisoned padding test)
            const double bv = (kk + 4 <= Np || kk + tig < Np) ? bp[nt * 8 * LD + kk] : 0.0;
            dmma(acc[0][nt], ar, bv);
            dmma(acc[1][nt], as, bv);
            dmma(acc[2][nt], at, bv);
          }
        }
      }
      // chain rule (eq. 6) + curl (Maxwell) / -div v, -grad p (acoustics), thread-local
      // (element 4g+tig, node row); component c lives in r[c >> 1][c & 1]
      double r[NT3][2];
      {
        const double* Gm = sG(s) + (4 * g + tig) * GEO_W;
        double dx[NC], dy[NC], dz[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double ur = acc[0][c >> 1][c & 1], us = acc[1][c >> 1][c & 1], ut = acc[2][c >> 1][c & 1];
          dx[c] = Gm[0] * ur + Gm[3] * us + Gm[6] * ut;
          dy[c] = Gm[1] * ur + Gm[4] * us + Gm[7] * ut;
          dz[c] = Gm[2] * ur + Gm[5] * us + Gm[8] * ut;
        }
        if constexpr (SYS == 0) {
          r[0][0] = dy[5] - dz[4];     // d_t Ex = (curl H)_x
          r[0][1] = dz[3] - dx[5];     // d_t Ey
          r[1][0] = dx[4] - dy[3];     // d_t Ez
          r[1][1] = -(dy[2] - dz[1]);  // d_t Hx = -(curl E)_x
          r[2][0] = -(dz[0] - dx[2]);  // d_t Hy
          r[2][1] = -(dx[1] - dy[0]);  // d_t Hz
        } else {
          r[0][0] = -(dx[1] + dy[2] + dz[3]);  // d_t p = -div v
          r[0][1] = -dx[0];                    // d_t v = -grad p
          r[1][0] = -dy[0];
          r[1][1] = -dz[0];
        }
      }
      if (waited < j) {
        long long _tw = clock64();
        mbar_wait(bar_full + s, unsigned(j / S) & 1);
#ifdef DG_WS_PROFILE
        if (lane == 0) atomicAdd(&g_ws_prof[5], (unsigned long long)(clock64() - _tw));
#else
        (void)_tw;
#endif
        waited = j;
      }
      // lift: r += LIFT . Flux  (two accumulator sets: 6 independent DMMA chains)
      const double* fp = F + (GW * g + gid) * LDF + tig;
      double r2[NT3][2];
#pragma unroll
      for (int nt = 0; nt < NT3; ++nt) r2[nt][0] = r2[nt][1] = 0.0;
      if constexpr (C::OPS_SMEM) {
        const double* lp = sA + 3 * M8 * C::LDA + row * C::LDL + tig;
#pragma unroll
        for (int kk = 0; kk < KL; kk += 8) {
          const double a0 = lp[kk];
#pragma unroll
          for (int nt = 0; nt < NT3; ++nt) dmma(r[nt], a0, fp[nt * 8 * LDF + kk]);
          if (kk + 4 < KL) {
            const double a1 = lp[kk + 4];
#pragma unroll
            for (int nt = 0; nt < NT3; ++nt) dmma(r2[nt], a1, fp[nt * 8 * LDF + kk + 4]);
          }
        }
      } else {
        const double* lp = opsA + size_t(3) * M8 * KV + size_t(row) * KL + tig;
#ifndef DG_WS_LUNROLL
        constexpr int LU = (N == 7 || N == 9) ? 8 : (N == 6 || N == 8) ? 6 : 2;
#else
        constexpr int LU = DG_WS_LUNROLL;
#endif
#pragma unroll LU
        for (int kk = 0; kk < KL; kk += 8) {
          const double a0 = __ldg(lp + kk);
          const double a1 = (kk + 4 < KL) ? __ldg(lp + kk + 4) : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT3; ++nt) dmma(r[nt], a0, fp[nt * 8 * LDF + kk]);
          if (kk + 4 < KL) {
#pragma unroll
            for (int nt = 0; nt < NT3; ++nt) dmma(r2[nt], a1, fp[nt * 8 * LDF + kk + 4]);
          }
        }
      }
      // LSERK update / RHS store (tiled layout)
      const int e = 4 * g + tig;
      if (row < Np && e < ne) {
        const int64_t tb = tile * TS + row;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int col = GW * g + 8 * (c >> 1) + 2 * tig + (c & 1);
          const int64_t idx = tb + int64_t(col) * LD;
          const double rhs = r[c >> 1][c & 1] + r2[c >> 1][c & 1];
          if (UPDATE) {
            double rold = 0.0;
            if constexpr (C::RES_SMEM) {
              if (res_in) rold = sR(s)[col * LD + row];
            } else if constexpr (C::RES_PREFETCH) {
              rold = rpre[c];
            } else {
              if (res_in) rold = p.res[idx];
            }
            const double rr = rk_a * rold + p.dt * rhs;
            p.res[idx] = rr;
            u_out[idx] = U[col * LD + row] + rk_b * rr;
          } else {
            p.rhs_out[idx] = rhs;
          }
        }
      }
#ifdef DG_WS_PROFILE
      if (lane == 0) atomicAdd(&g_ws_prof[6], (unsigned long long)(clock64() - _tc));
#endif
    }
    while (released < JJ) release(released++);
    DG_ACC(10);
  }
}

template <int N, int SYS>
void launch_stage_ws_sys(const StageParams<double>& p, const double* opsA, int mode, cudaStream_t st) {
  using C = WsCfg<N, System<SYS>::NC>;
  static PerDevice pd;
  const int sms = sms_for_device(pd, [] {
      cudaFuncSetAttribute(dg_stage_ws<N, true, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
      cudaFuncSetAttribute(dg_stage_ws<N, false, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
      cudaFuncSetAttribute(dg_stage_ws<N, true, SYS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
  });
  if (p.K <= 0) return;
  // element range [k_begin, k_begin+K) must start on a tile boundary
  const int64_t t0 = p.k_begin / C::E;
  const int64_t tc = (p.k_begin + p.K + C::E - 1) / C::E - t0;
  const int cap = sms - p.sm_reserve > 1 ? sms - p.sm_reserve : 1;  // SMs left to concurrent NCCL kernels
  const unsigned grid = unsigned(tc < cap ? tc : cap);
  if (mode == 1 && p.bsig)
    launch_pdl(true, dg_stage_ws<N, true, SYS, true>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
  else if (mode == 1)
    launch_pdl(true, dg_stage_ws<N, true, SYS>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
  else
    launch_pdl(true, dg_stage_ws<N, false, SYS>, grid, C::NT, C::SMEM_BYTES, st, p, opsA, t0, tc);
}
template <int N>
void launch_stage_ws(const StageParams<double>& p, const double* opsA, int mode, cudaStream_t st) {
  if (p.system == 1)
    launch_stage_ws_sys<N, 1>(p, opsA, mode, st);
  else
    launch_stage_ws_sys<N, 0>(p, opsA, mode, st);
}

#ifdef DG_WS_PROFILE
inline void ws_prof_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_ws_prof, sizeof(g_ws_prof)); }
inline void ws_prof_reset() {
  static unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_ws_prof, z, sizeof(z));
}
#endif

template <int N>
TileLayout ws_layout() {
  using C = WsCfg<N>;
  TileLayout L;
  L.E = C::E;
  L.LD = C::LD;
  L.perm = 1;
  L.TS = C::TS;
  return L;
}

}  // namespace dg
