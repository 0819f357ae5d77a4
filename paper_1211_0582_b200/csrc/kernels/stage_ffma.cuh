// FFMA variant, FP32: the warp-specialized TMA/mbarrier stage kernel of
// stage_ws.cuh with both contractions as register-tiled FFMA (no tensor cores).
//
// Why a SIMT path at all: the north_star asks for the FP32 contraction's
// TF32-or-FFMA choice to be justified by measurement.  3xTF32 costs three MMAs
// per product plus the hi/lo split of every B value, and pads M to 16; the
// algorithmic FP32 work at N = 4 is 38 K FMA per element and stage, which the
// FFMA pipe (128 FMA/clk/SM, 72 TF/s measured) retires in ~300 cycles — the
// same order as the 3xTF32 tensor time, with no padding and no splits.
//
// Tile layout (TileLayout perm = 3): element e, component c, node n of a tile at
// (c*LD + n)*E + e — elements fastest, so that
//   * a warp's 32 lanes (E elements x RG row groups) read B values U[c][k][e] for
//     consecutive e: one conflict-free shared-memory wavefront;
//   * the LSERK update stores u_out/res for consecutive e: coalesced 128-B rows;
//   * one bulk copy (TMA) still moves a whole tile (the tile is its smem image).
// Operators are stored transposed, A^T[b][k][m] and LIFT^T[j][m] (m fastest,
// padded to MR rows), so a thread's RB = 4 consecutive rows are one float4
// load that the whole warp shares (broadcast).
//
// Register tile per thread: 4 node rows x 6 components x {r,s,t} = 72 volume
// accumulators (9 loads per 72 FFMA), then chain rule + curl in registers
// (4 x 6 values), then LIFT . Flux (7 loads per 24 FFMA), then the update.  The
// residual is cp.async'ed into a per-warp staging buffer at task start (its
// latency hides behind the contractions without holding 24 registers).
// Roles (as stage_ws.cuh): 1 TMA loader warp, PW flux warps (trace gather with
// cp.async LA tiles ahead, upwind/PEC flux in place), CW compute warps streaming
// (tile, row block) tasks.
//
// FP64 (DFMA) instance: the same kernel with T = double and RB = 2 rows per thread (one
// 16-byte operator load still covers a thread's rows): 36 volume accumulators.
#pragma once
#include <cuda_runtime.h>

#include <cstring>

#include "stage_ws.cuh"

namespace dg {

// 16-byte vector of T (a thread's RB operator rows in one shared-memory load)
template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
  static __device__ __forceinline__ void unpack(const float4& v, float (&a)[4]) {
    a[0] = v.x;
    a[1] = v.y;
    a[2] = v.z;
    a[3] = v.w;
  }
};
template <>
struct V16<double> {
  using type = double2;
  static __device__ __forceinline__ void unpack(const double2& v, double (&a)[2]) {
    a[0] = v.x;
    a[1] = v.y;
  }
};
template <typename T>
__device__ __forceinline__ void cp_async_w(T* dst, const T* src) {
  if constexpr (sizeof(T) == 8)
    cp_async8(dst, src);
  else
    cp_async4(dst, src);
}

template <typename T, int N, int NC = 6>
struct FfCfg {
  static constexpr int W = int(sizeof(T));
  static constexpr bool F64 = W == 8;
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
#ifndef DG_FF_TUNE_W
#define DG_FF_TUNE_W 4
#endif
#ifdef DG_FF_TUNE_N
  static constexpr bool TUNED = N == DG_FF_TUNE_N && W == DG_FF_TUNE_W;
#else
  static constexpr bool TUNED = false;
#endif
#ifndef DG_FF_E
#define DG_FF_E 0
#endif
#ifndef DG_FF_S
#define DG_FF_S 0
#endif
#ifndef DG_FF_LA
#define DG_FF_LA -1
#endif
#ifndef DG_FF_CW
#define DG_FF_CW 0
#endif
#ifndef DG_FF_PW
#define DG_FF_PW 0
#endif
#ifndef DG_FF_OPS
#define DG_FF_OPS -1
#endif
  // elements per tile = elements per task (lanes = E elements x RG row groups); measured
  // (tools/gpu_ffma_tune.sh): smaller tiles win where they cost little row padding, since
  // 20 250 / (E x 148) tiles per CTA sets the tail imbalance and the ring depth
  static constexpr int E = (TUNED && DG_FF_E) ? DG_FF_E
                           : F64 ? (N <= 3 ? 16 : N <= 6 ? 8 : 4)
                                 : N <= 3 ? 32 : (N == 4 || N == 6) ? 16 : 8;
  static_assert(E == 4 || E == 8 || E == 16 || E == 32, "tile = 4, 8, 16 or 32 elements");
#ifndef DG_FF_EPL
#define DG_FF_EPL 0
#endif
  // elements per lane: 2 where the operators stream from L2 (FP32 N >= 6; ncu at N = 7: L1 hit rate 10 %,
  // 41 % long-scoreboard stalls): each operator load then feeds twice the FFMAs
  static constexpr int EPL = (TUNED && DG_FF_EPL) ? DG_FF_EPL : 1;
  static_assert(!F64 || EPL == 1, "EPL = 2 is an FP32-only tuning option (FP64 would not fit 216 registers)");
  static constexpr int EL = E / EPL;       // distinct elements per warp (lanes = EL x RG)
  static_assert(EL >= 4 && E % EPL == 0, "elements per lane");
  static constexpr int RG = 32 / EL;
  static constexpr int RB = 16 / W;        // node rows per thread (one 16-byte operator load)
  static constexpr int RT = RB * RG;       // node rows per task
  static constexpr int MB = (Np + RT - 1) / RT;  // row blocks = tasks per tile
  static constexpr int MR = MB * RT;       // padded rows of the transposed operators
  static constexpr int LD = Np;            // node stride of a component (no padding)
  static constexpr int TS = NC * LD * E;   // words per tile (NC fields: 6 Maxwell, 4 acoustics)
  static constexpr int GEOT = E * GEO_W;
  static constexpr int IDXT = E * NF;
  static constexpr int A_FLOATS = 3 * Np * MR + NF * MR;  // operator words
  static constexpr bool OPS_SMEM =
      (TUNED && DG_FF_OPS >= 0) ? bool(DG_FF_OPS) : (F64 ? A_FLOATS * W <= 64 * 1024 : N <= 5);
  static constexpr int A_BYTES = OPS_SMEM ? r16(A_FLOATS * W) : 0;
  static constexpr int OFF_U = 0;
  static constexpr int OFF_G = OFF_U + r16(TS * W);
  static constexpr int OFF_I = OFF_G + r16(GEOT * W);
  static constexpr int OFF_F = OFF_I + r16(IDXT * 4);
  static constexpr int SLOT = OFF_F + r16(NC * NF * E * W);
  static constexpr int FM_BYTES = r16(NF * 2);
  // residual staging: each compute warp cp.async's its task's residual (6 x RB values per
  // lane) into shared memory at task start, so no registers are held across the contractions
  static constexpr int STG_FLOATS = EPL * NC * RB * 32;
  static constexpr int STG_BYTES = 8 * STG_FLOATS * W;  // up to 8 compute warps (CW <= 8)
  static constexpr int FIXED = A_BYTES + FM_BYTES + STG_BYTES + 4 * 8 * 8;
  static constexpr int S_FIT = (227 * 1024 - FIXED) / SLOT;
  static constexpr int S_DEF = S_FIT > 6 ? 6 : S_FIT;
  // FP32 N = 4: a 3-slot ring with look-ahead 1 beats 4 slots / look-ahead 2 (0.307 vs 0.326 ms,
  // profiles/r1_ffma_tune.jsonl)
  // FP64 N = 1: 16-element tiles in an 8-slot ring with a 4-tile trace look-ahead beat 32 / 6 / 2
  // (C4 1.525 vs 1.590 ms, C2 0.0514 vs 0.0556 ms per step; profiles/r2_ffma_lown.jsonl)
  // FP32 N = 1: 8 slots / look-ahead 4 (C4 0.952 vs 1.002 ms, C2 -4 %); FP32 N = 2: 32-element tiles in a 4-slot
  // ring (C4 2.47 vs 3.27 ms, C2 0.078 vs 0.086 ms; profiles/r2_ffma_lown2.txt)
  static constexpr int S = (TUNED && DG_FF_S) ? DG_FF_S
                           : (!F64 && N == 4) ? 3
                           : (N == 1) ? 8
                           : (!F64 && N == 2) ? 4 : S_DEF;
  static_assert(S >= 2, "two ring slots at least");
  static constexpr int LA = (TUNED && DG_FF_LA >= 0) ? DG_FF_LA : (N == 1) ? 4 : S - 2 < 2 ? S - 2 : 2;
  static_assert(LA <= S - 2 || (S == 2 && LA == 0), "look-ahead beyond the ring");
#ifndef DG_FF_SPLIT
#define DG_FF_SPLIT -1
#endif
  // Register split (setmaxnreg): 16 warps = 4 warpgroups; the two compute warpgroups grow
  // to REG_HI registers, the producer warpgroups (loader + 7 flux warps) shrink to REG_LO.
  // Without it, 12 warps (3 per SMSP) leave 168 registers for the 72-accumulator tile but
  // only 3 flux warps, which cannot keep up at N <= 4 (ncu: compute warps wait on full[s]).
  // measured (profiles/r1_ffma_tune.jsonl): N = 1, 2, 3 gain 11-18 %, N = 4 is even, N >= 5 lose 1-5 %
  // FP64 (RB = 2, 36 accumulators) fits 128 registers: 16 warps without a split.
  // EPL = 2 (twice the accumulators): 12 warps, compute warpgroups at 224 registers, loader + 3 flux at 64.
  static constexpr bool SPLIT = (TUNED && DG_FF_SPLIT >= 0) ? bool(DG_FF_SPLIT) : (!F64 && N <= 4) || EPL == 2;
  static constexpr int REG_HI = EPL == 2 ? 216 : 192, REG_LO = 64;
  static constexpr int CW = SPLIT || F64 ? 8 : (TUNED && DG_FF_CW) ? DG_FF_CW : 8;
  static constexpr int PW = EPL == 2 ? 3 : SPLIT || F64 ? 7 : (TUNED && DG_FF_PW) ? DG_FF_PW : 3;
  // setmaxnreg.inc blocks until the CTA's pool has the registers, and the pool is what the launch
  // allocated: (warps x the launch-bound register count), so the split must fit inside it
  static constexpr int LAUNCH_REGS = (65536 / (32 * (CW + 1 + PW)) / 8) * 8 > 255 ? 255
                                     : (65536 / (32 * (CW + 1 + PW)) / 8) * 8;
  static_assert(!SPLIT || (CW % 4 == 0 && (CW + 1 + PW) % 4 == 0 &&
                           CW * REG_HI + (1 + PW) * REG_LO <= (CW + 1 + PW) * LAUNCH_REGS),
                "warpgroup register split exceeds the launch allocation (setmaxnreg.inc would block)");
  static constexpr int NT = 32 * (CW + 1 + PW);
  static constexpr int PT = 32 * PW;
  static constexpr int BAR_BYTES = 4 * S * 8;
  static_assert(CW <= 8, "residual staging sized for 8 compute warps");
  static constexpr size_t SMEM_BYTES = size_t(S) * SLOT + A_BYTES + FM_BYTES + STG_BYTES + BAR_BYTES;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert((TS * W) % 16 == 0 && (GEOT * W) % 16 == 0 && (IDXT * 4) % 16 == 0, "16-B bulk copies");
};

template <typename T, int N, bool UPDATE, int SYS, bool BSIG = false>
__global__ void __launch_bounds__(FfCfg<T, N, System<SYS>::NC>::NT, 1)
    dg_stage_ffma(const StageParams<T> p, const T* __restrict__ opsT, int64_t t_begin, int64_t t_count) {
  constexpr int NC = System<SYS>::NC;
  using C = FfCfg<T, N, NC>;
  using V = typename V16<T>::type;
  constexpr int W = C::W;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, E = C::E, LD = C::LD, S = C::S, TS = C::TS;
  constexpr int MR = C::MR, RB = C::RB;
  extern __shared__ __align__(128) unsigned char smem_ff[];
  unsigned char* smem = smem_ff;
  pdl_trigger();
  T* sA = reinterpret_cast<T*>(smem + size_t(S) * C::SLOT);
  int16_t* sFm = reinterpret_cast<int16_t*>(smem + size_t(S) * C::SLOT + C::A_BYTES);
  T* sStg = reinterpret_cast<T*>(smem + size_t(S) * C::SLOT + C::A_BYTES + C::FM_BYTES);
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + size_t(S) * C::SLOT + C::A_BYTES + C::FM_BYTES + C::STG_BYTES);
  uint64_t* bar_load = bars;
  uint64_t* bar_tr = bars + S;
  uint64_t* bar_full = bars + 2 * S;
  uint64_t* bar_empty = bars + 3 * S;
  auto sU = [&](int s) { return reinterpret_cast<T*>(smem + size_t(s) * C::SLOT + C::OFF_U); };
  auto sG = [&](int s) { return reinterpret_cast<T*>(smem + size_t(s) * C::SLOT + C::OFF_G); };
  auto sI = [&](int s) { return reinterpret_cast<int32_t*>(smem + size_t(s) * C::SLOT + C::OFF_I); };
  auto sF = [&](int s) { return reinterpret_cast<T*>(smem + size_t(s) * C::SLOT + C::OFF_F); };

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
      mbar_init(bar_empty + s, C::CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int m = tid; m < NF; m += C::NT) sFm[m] = p.fmask[m];
  if constexpr (C::OPS_SMEM) {
    constexpr int PER16 = 16 / W;
    static_assert(MR % PER16 == 0, "16-B operator rows");
    for (int w = tid; w < C::A_FLOATS / PER16; w += C::NT) cp_async16(sA + PER16 * w, opsT + PER16 * w);
    cp_commit();
    cp_wait<0>();
  }
  __syncthreads();
  pdl_wait();  // the previous stage's fields are complete from here on

  // role branches: producers (loader + flux warps) first, so that each warpgroup executes one
  // and the same setmaxnreg instruction (.aligned) and ptxas sees every role's register limit
  if (warp >= C::CW) {
  if constexpr (C::SPLIT) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::REG_LO));
  if (warp == C::CW) {
    // ===================== TMA loader warp (one lane) =====================
    if (lane == 0) {
      const int64_t nbl = BSIG ? bsig_ctiles(p.bsig_tiles) : 0;  // boundary tiles (multi-rank signal)
      for (int64_t j = 0; j < J; ++j) {
        const int s = int(j % S);
        mbar_wait(bar_empty + s, (unsigned(j / S) & 1) ^ 1);
        if constexpr (BSIG) loader_signal_after_wait(p.bsig, nbl, j, S);
        const int64_t tile = tile_of(j);
        mbar_arrive_tx(bar_load + s, TS * W + C::GEOT * W + C::IDXT * 4);
        bulk_g2s(sU(s), p.u_in + tile * TS, TS * W, bar_load + s);
        bulk_g2s(sG(s), p.geo + tile * C::GEOT, C::GEOT * W, bar_load + s);
        bulk_g2s(sI(s), p.gidx + tile * C::IDXT, C::IDXT * 4, bar_load + s);
      }
      if constexpr (BSIG) loader_signal_tail(bar_empty, p.bsig, nbl, J, S);
    }
  } else if (warp > C::CW) {
    // ============================ flux warps ============================
    // work item w = m*E + e (elements fastest: conflict-free face-buffer writes;
    // the gather index of a perm-3 tile is stored [m][e] for the same reason)
    const int ptid = tid - 32 * (C::CW + 1);
    auto traces = [&](int64_t j) {
      const int s = int(j % S);
      mbar_wait(bar_load + s, unsigned(j / S) & 1);
      const int32_t* I = sI(s);
      T* F = sF(s);
      for (int w = ptid; w < E * NF; w += C::PT) {
        const int32_t gi = I[w];
        if (gi >= 0) {  // intra-tile faces (negative codes) need no gather
          const bool ghost = gi >= p.ghost_base;
          const T* src = p.u_in + gi;
#pragma unroll
          for (int c = 0; c < NC; ++c) cp_async_w(F + c * NF * E + w, src + (ghost ? c * Nfp : c * LD * E));
        }
      }
      cp_async_mbar_arrive(bar_tr + s);
    };
    // flux of IT items per thread at once, branch-free, so the shared-memory loads of
    // independent items overlap (a single flux warp per SMSP is latency-bound otherwise).
    // u+ comes from the tile (intra-tile face), the gathered face buffer, or — on a PEC
    // wall — u- itself with the E jump negated (E+ = -E-, H+ = H-).  Items of elements
    // beyond the launch range are computed too (harmless: the compute warps skip them).
    auto flux = [&](int64_t j) {
      constexpr int IT = 2;  // (FP64: 16 warps x 128 registers also hold two items)
      constexpr int NIT = (E * NF + C::PT - 1) / C::PT;
      const int s = int(j % S);
      mbar_wait(bar_tr + s, unsigned(j / S) & 1);
      const T* U = sU(s);
      const T* Gm = sG(s);
      const int32_t* I = sI(s);
      T* F = sF(s);
#pragma unroll 1
      for (int it = 0; it < NIT; it += IT) {
        T uM[IT][NC], uP[IT][NC], g[IT][4], sE[IT];
        int wv[IT];
#pragma unroll
        for (int q = 0; q < IT; ++q) {
          const int w0 = ptid + (it + q) * C::PT;
          const bool ok = (it + q < NIT) && w0 < E * NF;
          const int w = ok ? w0 : ptid;
          wv[q] = ok ? w : -1;
          const int m = w / E, e = w - m * E, f = m / Nfp;
          const int nM = sFm[m];
          const int32_t gi = I[w];
          const T* pm = U + nM * E + e;
          const T* pp = pm;
          int cs = LD * E;
          sE[q] = T(-1);
          if (TileLayout::is_intra(gi)) {
            sE[q] = T(1);
            pp = U + TileLayout::intra_n(gi) * E + TileLayout::intra_e(gi);
          } else if (gi >= 0) {
            sE[q] = T(1);
            pp = F + w;
            cs = NF * E;
          }
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uM[q][c] = pm[c * LD * E];
            uP[q][c] = pp[c * cs];
          }
          const T* gp = Gm + e * GEO_W + 9 + 4 * f;
#pragma unroll
          for (int i = 0; i < 4; ++i) g[q][i] = gp[i];
        }
#pragma unroll
        for (int q = 0; q < IT; ++q) {
          T fl[NC];
          if constexpr (SYS == 0) {
            T dE[3], dH[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              dE[c] = sE[q] * uP[q][c] - uM[q][c];
              dH[c] = uP[q][c + 3] - uM[q][c + 3];
            }
            maxwell_flux<T>(g[q][0], g[q][1], g[q][2], p.alpha, dE, dH, fl);
          } else {  // acoustics; rigid wall (sE = -1, u+ = u-): p+ = p-, v+ = v- - 2 (n.v-) n
            const T nx = g[q][0], ny = g[q][1], nz = g[q][2];
            const T wall = sE[q] < T(0) ? T(1) : T(0);
            const T ndv = nx * uM[q][1] + ny * uM[q][2] + nz * uM[q][3];
            const T dp = uP[q][0] - uM[q][0];
            T dv[3];
            dv[0] = uP[q][1] - uM[q][1] - wall * T(2) * ndv * nx;
            dv[1] = uP[q][2] - uM[q][2] - wall * T(2) * ndv * ny;
            dv[2] = uP[q][3] - uM[q][3] - wall * T(2) * ndv * nz;
            acoustic_flux<T>(nx, ny, nz, p.alpha, dp, dv, fl);
          }
          const T sc = g[q][3] * T(0.5);
          if (wv[q] >= 0) {
#pragma unroll
            for (int c = 0; c < NC; ++c) F[c * NF * E + wv[q]] = fl[c] * sc;
          }
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
  }
  } else {
    if constexpr (C::SPLIT) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REG_HI));
    // =========================== compute warps ===========================
    constexpr int EPL = C::EPL, EL = C::EL;
    const int el = lane % EL, rg = lane / EL;  // elements el + ep * EL, ep < EPL
    const int64_t total = J * C::MB;
    int64_t released = 0, waited = -1, lwaited = -1;
    auto release = [&](int64_t jj) {
      if (waited < jj) {
        mbar_wait(bar_full + int(jj % S), unsigned(jj / S) & 1);
        waited = jj;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + int(jj % S));
    };
    const T* A = C::OPS_SMEM ? sA : opsT;
    auto ld4 = [&](int idx) -> V {  // RB consecutive operator rows, 16 bytes
      if constexpr (C::OPS_SMEM)
        return *reinterpret_cast<const V*>(A + idx);
      else
        return __ldg(reinterpret_cast<const V*>(A + idx));
    };
    for (int64_t q = warp; q < total; q += C::CW) {
      const int64_t j = q / C::MB;
      const int mb = int(q - j * C::MB);
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
      const int row0 = mb * C::RT + rg * RB;
      const T* U = sU(s) + el;
      const T* F = sF(s) + el;
      const int64_t tb = tile * TS + el;
      T* stg = sStg + warp * C::STG_FLOATS + lane;  // [ep][c][i][lane]
      if (UPDATE && res_in) {  // residual -> staging (coalesced over elements), consumed by the update
#pragma unroll
        for (int ep = 0; ep < EPL; ++ep)
          if (el + ep * EL < ne) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
              for (int i = 0; i < RB; ++i)
                if (row0 + i < Np)
                  cp_async_w(stg + ((ep * NC + c) * RB + i) * 32,
                             p.res + tb + ep * EL + int64_t(c * LD + row0 + i) * E);
          }
        cp_commit();
      }
      // ---- a1: [Dr;Ds;Dt] . U, RB rows x 6 components x 3 operators, EPL elements
      T acc[EPL][3][NC][RB];
#pragma unroll
      for (int ep = 0; ep < EPL; ++ep)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int i = 0; i < RB; ++i) acc[ep][b][c][i] = T(0);
#ifndef DG_FF_VUNROLL
#define DG_FF_VUNROLL (C::OPS_SMEM ? 5 : 10)  // operators through L1/L2 (N >= 6): +10..18 %
#endif
      constexpr int kVolUnroll = DG_FF_VUNROLL;
#pragma unroll kVolUnroll
      for (int k = 0; k < Np; ++k) {
        T a[3][RB];
#pragma unroll
        for (int b = 0; b < 3; ++b) V16<T>::unpack(ld4((b * Np + k) * MR + row0), a[b]);
#pragma unroll
        for (int ep = 0; ep < EPL; ++ep)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const T bv = U[(c * LD + k) * E + ep * EL];
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
              for (int i = 0; i < RB; ++i) acc[ep][b][c][i] = fma(a[b][i], bv, acc[ep][b][c][i]);
          }
      }
      // ---- chain rule + curl (thread-local: all components of one element and row)
      T r[EPL][NC][RB];
#pragma unroll
      for (int ep = 0; ep < EPL; ++ep) {
        const T* Gm = sG(s) + (el + ep * EL) * GEO_W;
        T gm[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) gm[i] = Gm[i];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          T dx[NC], dy[NC], dz[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const T ur = acc[ep][0][c][i], us = acc[ep][1][c][i], ut = acc[ep][2][c][i];
            dx[c] = gm[0] * ur + gm[3] * us + gm[6] * ut;
            dy[c] = gm[1] * ur + gm[4] * us + gm[7] * ut;
            dz[c] = gm[2] * ur + gm[5] * us + gm[8] * ut;
          }
          if constexpr (SYS == 0) {  // d_t E = curl H, d_t H = -curl E
            r[ep][0][i] = dy[5] - dz[4];
            r[ep][1][i] = dz[3] - dx[5];
            r[ep][2][i] = dx[4] - dy[3];
            r[ep][3][i] = -(dy[2] - dz[1]);
            r[ep][4][i] = -(dz[0] - dx[2]);
            r[ep][5][i] = -(dx[1] - dy[0]);
          } else {  // d_t p = -div v, d_t v = -grad p
            r[ep][0][i] = -(dx[1] + dy[2] + dz[3]);
            r[ep][1][i] = -dx[0];
            r[ep][2][i] = -dy[0];
            r[ep][3][i] = -dz[0];
          }
        }
      }
      if (waited < j) {
        mbar_wait(bar_full + s, unsigned(j / S) & 1);
        waited = j;
      }
      // ---- a4: r += LIFT . Flux
#ifndef DG_FF_LUNROLL
#define DG_FF_LUNROLL (C::OPS_SMEM ? 4 : 8)
#endif
      constexpr int kLiftUnroll = DG_FF_LUNROLL;
#pragma unroll kLiftUnroll
      for (int jn = 0; jn < NF; ++jn) {
        T l[RB];
        V16<T>::unpack(ld4(3 * Np * MR + jn * MR + row0), l);
#pragma unroll
        for (int ep = 0; ep < EPL; ++ep)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const T fv = F[(c * NF + jn) * E + ep * EL];
#pragma unroll
            for (int i = 0; i < RB; ++i) r[ep][c][i] = fma(l[i], fv, r[ep][c][i]);
          }
      }
      // ---- a5: LSERK update (or RHS store), coalesced over elements
      if (UPDATE && res_in) cp_wait<0>();
#pragma unroll
      for (int ep = 0; ep < EPL; ++ep) {
        if (el + ep * EL < ne) {
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int i = 0; i < RB; ++i) {
              const int row = row0 + i;
              if (row < Np) {
                const int64_t idx = tb + ep * EL + int64_t(c * LD + row) * E;
                if (UPDATE) {
                  const T rold = res_in ? stg[((ep * NC + c) * RB + i) * 32] : T(0);
                  const T rr = p.rk_a * rold + p.dt * r[ep][c][i];
                  p.res[idx] = rr;
                  p.u_out[idx] = U[(c * LD + row) * E + ep * EL] + p.rk_b * rr;
                } else {
                  p.rhs_out[idx] = r[ep][c][i];
                }
              }
            }
        }
      }
    }
    while (released < J) release(released++);
  }
}

template <typename T, int N, int SYS>
void launch_stage_ffma_sys(const StageParams<T>& p, const T* opsT, int mode, cudaStream_t st) {
  using C = FfCfg<T, N, System<SYS>::NC>;
  static PerDevice pd;
  const int sms = sms_for_device(pd, [] {
      cudaFuncSetAttribute(dg_stage_ffma<T, N, true, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(C::SMEM_BYTES));
      cudaFuncSetAttribute(dg_stage_ffma<T, N, false, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(C::SMEM_BYTES));
      cudaFuncSetAttribute(dg_stage_ffma<T, N, true, SYS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(C::SMEM_BYTES));
  });
  if (p.K <= 0) return;
  const int64_t t0 = p.k_begin / C::E;
  const int64_t tc = (p.k_begin + p.K + C::E - 1) / C::E - t0;
  const int cap = sms - p.sm_reserve > 1 ? sms - p.sm_reserve : 1;  // SMs left to concurrent NCCL kernels
  const unsigned grid = unsigned(tc < cap ? tc : cap);
  if (mode == 1 && p.bsig)
    launch_pdl(true, dg_stage_ffma<T, N, true, SYS, true>, grid, C::NT, C::SMEM_BYTES, st, p, opsT, t0, tc);
  else if (mode == 1)
    launch_pdl(true, dg_stage_ffma<T, N, true, SYS>, grid, C::NT, C::SMEM_BYTES, st, p, opsT, t0, tc);
  else
    launch_pdl(true, dg_stage_ffma<T, N, false, SYS>, grid, C::NT, C::SMEM_BYTES, st, p, opsT, t0, tc);
}

// p.system selects the linear system (dg_system): 0 Maxwell, 1 acoustics (NEXT-3)
template <typename T, int N>
void launch_stage_ffma(const StageParams<T>& p, const T* opsT, int mode, cudaStream_t st) {
  if (p.system == 1)
    launch_stage_ffma_sys<T, N, 1>(p, opsT, mode, st);
  else
    launch_stage_ffma_sys<T, N, 0>(p, opsT, mode, st);
}

template <typename T, int N>
TileLayout ffma_layout() {
  using C = FfCfg<T, N>;
  TileLayout L;
  L.E = C::E;
  L.LD = C::LD;
  L.perm = 3;
  L.TS = C::TS;
  return L;
}

// host: transposed, row-padded operators A^T[3][Np][MR] (A^T[b][k][m] = D_b[m][k]) and
// LIFT^T[NF][MR], from row-major FP64 Dr|Ds|Dt ([Np][Np]) and LIFT ([Np][NF]); padding zero
template <typename T, int N>
void ffma_ops(const double* Dr, const double* Ds, const double* Dt, const double* LIFT, T* out) {
  using C = FfCfg<T, N>;
  constexpr int Np = C::Np, NF = C::NF, MR = C::MR;
  for (int i = 0; i < C::A_FLOATS; ++i) out[i] = T(0);
  const double* D[3] = {Dr, Ds, Dt};
  for (int b = 0; b < 3; ++b)
    for (int m = 0; m < Np; ++m)
      for (int k = 0; k < Np; ++k) out[(size_t(b) * Np + k) * MR + m] = T(D[b][m * Np + k]);
  for (int m = 0; m < Np; ++m)
    for (int jn = 0; jn < NF; ++jn) out[size_t(3) * Np * MR + size_t(jn) * MR + m] = T(LIFT[m * NF + jn]);
}

}  // namespace dg
