// TC variant (FP32, N = 1..9): the stage kernel on the 5th-generation tensor cores.
//
// One tile = E = 21 elements = 126 (element, output-component) rows of a 128-row
// tcgen05 MMA.  The whole semi-discrete right-hand side of a tile is ONE K-chunked
// GEMM accumulated in tensor memory (eq. 4; eq. 6, PAPER.md:290-308;
// "fields in aggregate as a matrix"):
//
//   D[row = 6e+c][n] = sum_k  G[row][k] . Op[k][n],      n = output node (MMA N = Np -> NP16)
//
//   volume K (a1): k = (node m, derivative d):  Op = D_d^T,  G = the chain rule and the
//                  curl folded into the operand: rhsE = curl H, rhsH = -curl E gives, e.g.
//                  for row Ex:  G = g[d][y]*Hz(m) - g[d][z]*Hy(m)   (g[d][a] = dr_d/dx_a)
//   lift K (a4):   k = face node m:  Op = LIFT^T,  G = Fscale/2 * upwind/PEC flux (a2+a3)
//
// so the epilogue is only the LSERK update (a5) of D.  Operands are fp32 in shared
// memory in the K-major SWIZZLE_NONE canonical layout, 8-k chunks (LBO 128 B, SBO 256 B);
// the accumulation is 3xTF32:  G.Op ~= G.Op + G_lo.Op + G.Op_lo, where the hardware
// truncates fp32 operands to TF32 (tools/tcgen05_probe.cu), so x itself is x_hi and only
// x_lo = x - trunc(x) is stored (operators: split once on the host).
//
// Warp roles (one persistent CTA per SM; all handshakes are mbarriers):
//   warps 0..3   epilogue: warp q reads TMEM lanes 32q..32q+31 (row = lane), LSERK update
//                straight from the accumulator to global memory (coalesced along rows)
//   warp 4       loaders: lane 0 streams node-octet slabs of the tile (8 nodes x 126 rows,
//                one bulk copy each; the field layout is node-major per tile) through an
//                RS-slot ring; lane 1 streams the operator chunks in MMA order through an
//                RB-slot ring (N >= 5), or copies all of them once (N <= 4, resident)
//   warp 5       TMEM allocator + MMA issuer (one thread): per 8-k chunk three
//                tcgen05.mma.kind::tf32 (M=128, N=NP16, K=8) into a double-buffered
//                accumulator; tcgen05.commit frees ring slots and signals the epilogue
//   warps 6..9   volume generators: row = thread; per octet slab 3 chunks (d = r,s,t)
//   warps 10..15 flux generators (PW warps): item = (element, face node); u- and u+
//                gathered from global/L2 (the per-face (neighbour base, orientation code)
//                connectivity + 24 smem orientation tables replace the per-node index),
//                upwind/PEC flux x Fscale/2, one 8-k chunk at a time, one chunk look-ahead
// The MMA consumes the volume and flux chunk streams in a fixed proportional merge
// (tc_is_vol), so the accumulation order is deterministic and partition-invariant.
#pragma once
#include <cuda_runtime.h>

#include <cstring>

#include "stage_ws.cuh"

#ifndef DG_TC_WB
#define DG_TC_WB 0
#endif
#ifndef DG_TC_RA
#define DG_TC_RA 12
#endif
#ifndef DG_TC_RB
#define DG_TC_RB 12
#endif
#ifndef DG_TC_LF
#define DG_TC_LF 0
#endif
#ifndef DG_TC_RS
#define DG_TC_RS 0
#endif
#ifndef DG_TC_LT
#define DG_TC_LT 0
#endif
#ifndef DG_TC_RM
#define DG_TC_RM 0
#endif
// Diagnostic knock-outs (timing experiments only; results are wrong when set, never in libdg.so):
// DG_TC_X = bit mask: 1 flux warps skip the trace gathers and the flux arithmetic (zeros),
// 2 operand writers skip the slab reads and the G arithmetic, 4 writers skip tcgen05.st,
// 8 epilogue skips the global loads and stores, 16 the MMA issuer does not wait for its operand
// chunks (pure issue rate; hangs: kept out of the sweeps), 32 the MMA issuer skips its tcgen05.fence::after_thread_sync.  Which removal speeds the kernel up tells which
// role bounds it (tools/gpu_tc_knockout.sh).
#ifndef DG_TC_X
#define DG_TC_X 0
#endif

namespace dg {

// the MMA's fixed interleave of the NV volume and NFQ flux chunks of a tile
__host__ __device__ constexpr bool tc_is_vol(int v, int f, int NV, int NFQ) {
  return f >= NFQ || (v < NV && v * NFQ <= f * NV);
}

template <int N, int SYS = 0>
struct TcCfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  // SYS 0 Maxwell (6 fields), 1 linear acoustics (4 fields, NEXT-3): the same GEMM with the system's
  // operand generator and flux.  Acoustics uses 24 elements = 96 rows: 8 x 24 = 192 flux items, one
  // per flux thread and chunk (32 elements would need 256 flux threads).
  static constexpr int NC = System<SYS>::NC;
  static constexpr int E = SYS == 0 ? 21 : 24;      // elements per tile
  static constexpr int ROWS = NC * E;               // 126 (Maxwell) / 96 (acoustics) of the 128 MMA rows
  static constexpr int NP16 = (Np + 15) / 16 * 16;  // MMA N
  static constexpr int NO = (Np + 7) / 8;           // node octets
  static constexpr int NV = 3 * NO;                 // volume chunks
  static constexpr int NFQ = (NF + 7) / 8;          // flux chunks
  static constexpr int NQ = NV + NFQ;
  static constexpr int TS = (ROWS * Np + 7) / 8 * 8;  // floats per tile (node-major)
  static constexpr int GEOT = tc_geot(E);           // floats per tile of geometry (E x 26, padded to 16 B)
  static constexpr int CONNT = TC_CONNT;            // int32 per tile: fbase [E][4] | fcode [E] (4 x u8) | pad
  static constexpr int MSLOT = (GEOT * 4 + CONNT * 4 + 127) / 128 * 128;  // meta ring slot (bytes)
  static_assert(E * GEO_W <= GEOT && 5 * E <= CONNT, "per-tile records");
  static constexpr int SLABF = 1024;                // floats per slab slot (8 x 126 used)
  static constexpr int OPC = 2 * 8 * NP16;          // floats per operator chunk (hi | lo)
  static constexpr int ITEMS = 8 * E;               // flux items (element, face-node slot) per chunk
  static constexpr int PW = 6;                      // flux warps: one item per thread and chunk
  static constexpr int FTH = 32 * PW;
  // ring depths (0 = per-order default; measured, profiles/r2_tc_tune.jsonl): shallower flux staging and trace
  // pipelines (LF 4, LT 3) at N = 4, 5, 6, 9 and shallower slab/meta rings at N = 5 (-1..4 %), round-2 defaults otherwise
  static constexpr bool SHALLOW = N == 4 || N == 5 || N == 6 || N == 9;
  static constexpr int LT = DG_TC_LT ? DG_TC_LT : SHALLOW ? 3 : 4;  // per-thread cp.async trace pipeline depth (chunks)
  static constexpr int TRC = FTH * 2 * NC;          // floats per trace-staging chunk: [NC pairs][FTH][2] (u-, u+)
  static constexpr int LF = DG_TC_LF ? DG_TC_LF : SHALLOW ? 4 : 6;  // flux staging ring (chunks) [128 rows][8]
  static constexpr int FSC = 128 * 8;
  static constexpr int RS = DG_TC_RS ? DG_TC_RS : N == 5 ? 3 : 4, RM = DG_TC_RM ? DG_TC_RM : N == 5 ? 3 : 4;
  // operand chunks per writer batch (one tcgen05.wait::st): 3, or 4 at N = 6, 8, 9 (measured on C2,
  // tools/gpu_tc_tune.sh: N = 6 -3.5 %, N = 8 -3.5 %, N = 9 -2 %; N = 3, 4 +1.5 % with 4, N = 7 +0.4 %)
  static constexpr int WB = DG_TC_WB ? DG_TC_WB : (N == 6 || N == 8 || N == 9) ? 4 : 3;
  static constexpr int WUNR = NQ <= 36 ? (NQ + WB - 1) / WB : 1;
  // generated operand G in TENSOR memory (kind::tf32 A operand: lane = row, one column per k):
  // ring slots of 16 columns (8 G | 8 G_lo) after the two accumulators
#ifdef DG_TC_ONEACC
  static constexpr int NACC = 1;                    // accumulators (tiles in flight between MMA and epilogue)
#else
  static constexpr int NACC = 2;
#endif
  // 3xTF32 with two MMAs per chunk where the instruction floor dominates (N <= 6, measured
  // ~45-60 cycles per M = 128 kind::tf32 MMA up to N ~ 96, tools/tcgen05_peak.cu):
  //   G . [Op | Op_lo] as ONE MMA of width 2 NP16 (the chunk's hi and lo blocks are adjacent
  //   8-row core-matrix groups, so they form one B operand), then G_lo . Op into the first half;
  //   the epilogue adds the halves.  N >= 7: three MMAs of width NP16 (2 NP16 > 192; the pipe is
  //   throughput-bound there, so fusing would gain nothing).
#ifdef DG_TC_NOFUSE
  static constexpr bool FUSE_LO = false;
#else
  static constexpr bool FUSE_LO = 2 * NP16 <= 192;
#endif
  static constexpr int DW = FUSE_LO ? 2 * NP16 : NP16;  // accumulator columns per tile
  static constexpr int ACC1 = DW;                   // column of accumulator 1
  static constexpr int NA = (512 - NACC * DW) / 16;
  static constexpr int RA_T = NA < DG_TC_RA ? NA : DG_TC_RA;
  static __host__ __device__ constexpr int a_col(int k) { return NACC * DW + 16 * k; }
  static constexpr int al1k(int b) { return (b + 1023) / 1024 * 1024; }
  static constexpr int NTAB = NF + 24 * Nfp + 6 * Nfp + 8 * NFQ;  // int16: Fmask | node | ghost | chunk-slot tables
  static constexpr int FIXED = RS * SLABF * 4 + RM * MSLOT + LT * TRC * 4 + LF * FSC * 4 +
                               (NTAB * 2 + 15) / 16 * 16 + 1024;
  static constexpr bool OP_RES = FIXED + al1k(NQ * OPC * 4) <= 226 * 1024;  // operators resident in smem
  static constexpr int RB_MAX = (226 * 1024 - FIXED) / (OPC * 4);
  static constexpr int RA = RA_T & ~1;  // even: slots are released in pairs
  static constexpr int RB = OP_RES ? NQ : (RB_MAX < DG_TC_RB ? RB_MAX : DG_TC_RB);
  // 16 warps: 4 per SMSP, so every thread can have 128 registers
  static constexpr int W_LD = 4, W_MMA = 5, W_VG0 = 6, W_FG0 = 10;
  static constexpr int NW = W_FG0 + PW;
  static constexpr int NT = 32 * NW;
  static constexpr int TMEM_COLS = 512;
  static constexpr int OFF_B = 0;
  static constexpr int OFF_S = OFF_B + al1k(RB * OPC * 4);
  static constexpr int OFF_M = OFF_S + RS * SLABF * 4;   // meta ring: [RM][geo GEOT floats | conn CONNT ints]
  static constexpr int OFF_TR = OFF_M + RM * MSLOT;     // trace staging ring [LT][TRC]
  static constexpr int OFF_FS = OFF_TR + LT * TRC * 4;  // flux staging ring [LF][FSC]
  static constexpr int OFF_T = OFF_FS + LF * FSC * 4;
  static constexpr int OFF_BAR = OFF_T + (NTAB * 2 + 15) / 16 * 16;
  static constexpr int NBAR = 2 * RB + 2 * RA + 2 * LF + 2 * RS + 2 * RM + 4;
  static constexpr size_t SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
  static_assert(RA >= 4, "TMEM operand ring depth");
  static_assert(Nfp <= 64 && Np <= 256, "chunk-slot table packing");
  static_assert(RB >= 3, "operator ring depth");
  static_assert(8 * ROWS <= SLABF && ROWS <= 128, "slab slot / MMA rows");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(FTH >= ITEMS, "one flux item per thread and chunk");
  static_assert(ITEMS <= 2 * 32 * PW, "at most two flux items per thread and chunk");
  static constexpr size_t OPS_FLOATS = size_t(NQ) * OPC;
};

__device__ __forceinline__ uint64_t tc_desc(const void* smem) {  // K-major, 8-k chunk: LBO 128 B, SBO 256 B
  uint64_t d = uint64_t((smem_u32(smem) >> 4) & 0x3FFF);
  d |= uint64_t(128 >> 4) << 16;
  d |= uint64_t(256 >> 4) << 32;
  d |= uint64_t(1) << 46;  // sm100 descriptor version
  return d;
}
__host__ __device__ constexpr uint32_t tc_idesc(int m, int n) {  // kind::tf32, fp32 accumulate, both K-major
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// mbarrier wait with a suspend-time hint: a waiting warp sleeps until the phase completes
// instead of spinning try_wait and stealing issue slots from the producer warps
__device__ __forceinline__ void tc_wait(uint64_t* b, unsigned parity) {
#ifdef DG_TC_SPIN
  mbar_wait(b, parity);
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// one lane of a converged warp (elect.sync): the MMA issuer's single issuing thread
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n.reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(p));
  return p != 0;
}
// the MMA issuer's waits (DG_TC_MMASPIN: spin instead of the suspend-hint wait, experiment)
__device__ __forceinline__ void tc_wait_mma(uint64_t* b, unsigned parity) {
#ifdef DG_TC_MMASPIN
  mbar_wait(b, parity);
#else
  tc_wait(b, parity);
#endif
}
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
// word offset of (row, kk) inside an 8-k chunk of the canonical K-major layout
__host__ __device__ constexpr int tc_cm(int r, int kk) { return ((r >> 3) * 2 + (kk >> 2)) * 32 + (r & 7) * 4 + (kk & 3); }

#ifdef DG_WS_PROFILE
// per-role cycle counters (lane 0 of each warp, summed over CTAs; tools/tc_profile.py):
// 0 epi wait acc_full | 1 epi work | 2 VG wait slab | 3 VG wait A slot | 4 VG work | 5 FG wait A slot |
// 6 FG work (loads + flux) | 7 MMA wait V chunk | 8 MMA wait F chunk | 9 MMA wait operator chunk |
// 10 MMA issue | 11 slab loader wait | 12 tiles (epilogue warp 0) | 13 CTA cycles (epilogue warp 0)
__device__ unsigned long long g_tc_prof[16];
__device__ float* g_tc_dbg = nullptr;  // debug dump of the generated operand G [tile][NQ][128][8]
inline void tc_dbg_set(float* p) { cudaMemcpyToSymbol(g_tc_dbg, &p, sizeof(p)); }
#define TC_T(v) long long v = clock64()
#define TC_A(i, t0)                                             \
  do {                                                          \
    tcp[i] += (unsigned long long)(clock64() - (t0));           \
  } while (0)
inline void tc_prof_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_tc_prof, sizeof(g_tc_prof)); }
inline void tc_prof_reset() {
  static unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
}
#else
#define TC_T(v) \
  do {          \
  } while (0)
#define TC_A(i, t0) \
  do {              \
  } while (0)
#endif

template <int N, bool UPDATE, int SYS, bool BSIG = false>
__global__ void __launch_bounds__(TcCfg<N, SYS>::NT, 1)
    dg_stage_tc(const StageParams<float> p, const float* __restrict__ ops, int t_begin64, int t_count64) {
  // per-CTA counters and word offsets fit 32 bits (dg_mesh_upload bounds a rank's state below 2^31 words)
  const int t_begin = int(t_begin64), t_count = int(t_count64);
  using C = TcCfg<N, SYS>;
  constexpr int NC = C::NC;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, E = C::E, ROWS = C::ROWS, NP16 = C::NP16;
  constexpr int NO = C::NO, NV = C::NV, NFQ = C::NFQ, NQ = C::NQ, TS = C::TS;
  constexpr int RB = C::RB, RS = C::RS, RA = C::RA, LF = C::LF, RM = C::RM, LT = C::LT, ITEMS = C::ITEMS;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  unsigned char* smem = smem_tc;
  pdl_trigger();
#ifdef DG_WS_PROFILE
  unsigned long long tcp[12] = {0};  // per-thread role counters, flushed once at the end
#endif
  float* sB = reinterpret_cast<float*>(smem + C::OFF_B);
  float* sFS = reinterpret_cast<float*>(smem + C::OFF_FS);
  float* sS = reinterpret_cast<float*>(smem + C::OFF_S);
  float* sTR = reinterpret_cast<float*>(smem + C::OFF_TR);
  int16_t* sFm = reinterpret_cast<int16_t*>(smem + C::OFF_T);
  const int16_t* sNP = sFm + NF;          // [24][Nfp] neighbour node of face node i, by f2*6 + orientation
  const int16_t* sGP = sNP + 24 * Nfp;    // [6][Nfp]  ghost record position, by orientation
  auto sGeo = [&](int j) { return reinterpret_cast<const float*>(smem + C::OFF_M + int(j % RM) * C::MSLOT); };
  auto sConn = [&](int j) {
    return reinterpret_cast<const int32_t*>(smem + C::OFF_M + int(j % RM) * C::MSLOT + C::GEOT * 4);
  };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* b_full = bars;
  uint64_t* b_empty = b_full + RB;
  uint64_t* a_full = b_empty + RB;   // TMEM operand ring (writers -> MMA)
  uint64_t* a_empty = a_full + RA;   // (MMA commit -> writers)
  uint64_t* f_full = a_empty + RA;   // flux staging ring (flux warps -> writers)
  uint64_t* f_empty = f_full + LF;   // (writers -> flux warps)
  uint64_t* s_full = f_empty + LF;
  uint64_t* s_empty = s_full + RS;
  uint64_t* m_full = s_empty + RS;
  uint64_t* m_empty = m_full + RM;
  uint64_t* acc_full = m_empty + RM;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int J = t_count > blockIdx.x ? (t_count - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int kend = int(p.k_begin + p.K);
  auto tile_of = [&](int j) { return t_begin + blockIdx.x + j * gridDim.x; };
  auto count_of = [&](int tile) {
    const int k0 = tile * E;
    return int(kend - k0 < E ? kend - k0 : E);
  };

  if (tid == 0) {
    for (int i = 0; i < RB; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    for (int i = 0; i < RA; ++i) {
      mbar_init(a_full + i, 4);
      mbar_init(a_empty + i, 1);  // (only the first RA / 2: one per slot pair)
    }
    for (int i = 0; i < LF; ++i) {
      mbar_init(f_full + i, C::PW);
      mbar_init(f_empty + i, 4);
    }
    for (int i = 0; i < RS; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 4);
    }
    for (int i = 0; i < RM; ++i) {
      mbar_init(m_full + i, 1);
      mbar_init(m_empty + i, 4 + C::PW);  // operand writers + flux warps
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (C::OP_RES) {  // resident operators (N <= 5): fetched while the previous stage drains
      mbar_arrive_tx(b_full, unsigned(C::OPS_FLOATS * 4));
      bulk_g2s(sB, ops, unsigned(C::OPS_FLOATS * 4), b_full);
    }
  }
  if (warp == C::W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int w = tid; w < NF + 30 * Nfp; w += C::NT) sFm[w] = p.ftab[w];
  for (int w = tid; w < 8 * NFQ; w += C::NT) {  // chunk slot w -> face node m = w: f | i << 2 | Fmask[m] << 8
    const int f = w / Nfp, i = w - f * Nfp;
    sFm[NF + 30 * Nfp + w] = int16_t(w < NF ? (f | (i << 2) | (int(p.ftab[w]) << 8)) : 0xffff);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the previous stage's fields are complete from here on

  if (warp < 4) {
    // =========================== epilogue (a5) ===========================
    // u and res of a 16-node column group do not depend on the accumulator: they are loaded
    // one group ahead (the first group before waiting for the MMA), so their latency hides
    // behind the MMA / the previous group instead of serializing with the stores.
    const int r = 32 * warp + lane, e = r / NC;
    const bool res_in = UPDATE && !p.first_stage;
    TC_T(tcta);
    for (int j = 0; j < J; ++j) {
      const int a = j % C::NACC;
      const int tile = tile_of(j);
      const bool valid = r < ROWS && e < count_of(tile);
      const int base = tile * TS + r;
      auto ld_grp = [&](int c0, float (&uv)[16], float (&rv)[16]) {
        const float* up = p.u_in + base + c0 * ROWS;
        const float* rp = p.res + base + c0 * ROWS;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const bool ok = UPDATE && valid && c0 + i < Np && !(DG_TC_X & 8);
          uv[i] = ok ? __ldg(up + i * ROWS) : 0.0f;
          rv[i] = ok && res_in ? rp[i * ROWS] : 0.0f;
        }
      };
      auto ld16 = [&](uint32_t col, uint32_t (&v)[16]) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + (uint32_t(32 * warp) << 16) + col));
      };
      auto process = [&](int c0, const float (&uv)[16], const float (&rv)[16]) {
        uint32_t v[16];
        ld16(uint32_t(a * C::ACC1 + c0), v);
        if constexpr (C::FUSE_LO) {  // D = G.Op_hi + G_lo.Op_hi (first half) + G.Op_lo (second half)
          uint32_t w[16];
          ld16(uint32_t(a * C::ACC1 + NP16 + c0), w);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(w[i]));
        } else {
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (valid && !(DG_TC_X & 8)) {
          float* rp = p.res + base + c0 * ROWS;
          float* op = (UPDATE ? p.u_out : p.rhs_out) + base + c0 * ROWS;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (c0 + i < Np) {
              const float d = __uint_as_float(v[i]);
              if (UPDATE) {
                const float rr = p.rk_a * rv[i] + p.dt * d;
                rp[i * ROWS] = rr;
                op[i * ROWS] = uv[i] + p.rk_b * rr;
              } else {
                op[i * ROWS] = d;
              }
            }
          }
        }
      };
      float ua[16], ra[16], ub[16], rb[16];
      ld_grp(0, ua, ra);
      TC_T(t0);
      tc_wait(acc_full + a, unsigned(j / C::NACC) & 1);
      TC_A(0, t0);
      TC_T(t1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c0 = 0; c0 < NP16; c0 += 32) {
        if (c0 + 16 < NP16) ld_grp(c0 + 16, ub, rb);
        process(c0, ua, ra);
        if (c0 + 16 < NP16) {
          if (c0 + 32 < NP16) ld_grp(c0 + 32, ua, ra);
          process(c0 + 16, ub, rb);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + a);
      TC_A(1, t1);
#ifdef DG_WS_PROFILE
      if (tid == 0) atomicAdd(&g_tc_prof[12], 1ull);
#endif
    }
#ifdef DG_WS_PROFILE
    if (tid == 0) atomicAdd(&g_tc_prof[13], (unsigned long long)(clock64() - tcta));
#endif
  } else if (warp == C::W_LD) {
    if (lane == 0) {
      // ===== loader: one thread drives both copy streams with non-blocking barrier tests =====
      // stream 1: per tile, geometry + connectivity (meta ring), then its node-octet slabs;
      // stream 2: the operator chunks in MMA order (streamed orders; resident: one copy, issued in the
      // prologue before the programmatic-dependency wait: the operators do not depend on the previous stage)
      const int T2 = C::OP_RES ? 0 : J * NQ;
      int j1 = 0, o1 = -1, g1 = 0, g2 = 0;
      while (j1 < J || g2 < T2) {
        bool moved = false;
        if (j1 < J) {
          const int tile = tile_of(j1);
          if (o1 < 0) {
            const int ms = j1 % RM;
            if (mbar_test(m_empty + ms, (unsigned(j1 / RM) & 1) ^ 1)) {
              mbar_arrive_tx(m_full + ms, unsigned(C::GEOT * 4 + C::CONNT * 4));
              bulk_g2s(smem + C::OFF_M + ms * C::MSLOT, p.geo + tile * C::GEOT, unsigned(C::GEOT * 4), m_full + ms);
              bulk_g2s(smem + C::OFF_M + ms * C::MSLOT + C::GEOT * 4, p.gidx + tile * C::CONNT, unsigned(C::CONNT * 4),
                       m_full + ms);
              o1 = 0;
              moved = true;
            }
          } else {
            const int s = g1 % RS;
            if (mbar_test(s_empty + s, (unsigned(g1 / RS) & 1) ^ 1)) {
              const int nodes = Np - 8 * o1 < 8 ? Np - 8 * o1 : 8;
              unsigned bytes = unsigned(nodes * ROWS * 4);
              bytes = (bytes + 15) & ~15u;  // an odd node count ends 8 B short; the tile padding covers it
              mbar_arrive_tx(s_full + s, bytes);
              bulk_g2s(sS + s * C::SLABF, p.u_in + tile * TS + 8 * o1 * ROWS, bytes, s_full + s);
              ++g1;
              if (++o1 == NO) {
                o1 = -1;
                ++j1;
              }
              moved = true;
            }
          }
        }
        if (g2 < T2) {
          const int b = g2 % RB;
          if (mbar_test(b_empty + b, (unsigned(g2 / RB) & 1) ^ 1)) {
            mbar_arrive_tx(b_full + b, unsigned(C::OPC * 4));
            bulk_g2s(sB + b * C::OPC, ops + (g2 % NQ) * C::OPC, unsigned(C::OPC * 4), b_full + b);
            ++g2;
            moved = true;
          }
        }
        if (!moved) __nanosleep(64);
      }
    }
  } else if (warp == C::W_MMA) {
    // ============================ MMA issuer ============================
    // The whole warp runs the schedule (warp-uniform control flow: ring positions and phases are
    // kept as incrementing counters, the operand addresses stay in uniform registers) and one
    // elected lane issues the MMAs and commits.  Round 2 measurement: issued from `if (lane == 0)`
    // with modulo ring arithmetic, every chunk cost ~70 SASS instructions (R2UR moves, divisions,
    // an ELECT retry loop per MMA) in one dependent chain, ~450 cycles per chunk at every order.
    constexpr uint32_t idesc = tc_idesc(128, NP16);
    constexpr uint32_t idesc2 = tc_idesc(128, C::FUSE_LO ? 2 * NP16 : NP16);  // G . [Op | Op_lo]
    // descriptor of operator slot/chunk 0; other chunks differ only in the start-address
    // field (bits 0..13, address >> 4), so they are db0 + (byte offset >> 4)
    const uint64_t db0 = tc_desc(sB);
    constexpr uint64_t DLO = uint64_t(8 * NP16 * 4) >> 4;  // hi -> lo half of a chunk
    constexpr uint64_t DCH = uint64_t(C::OPC * 4) >> 4;    // next chunk / slot
    const bool leader = elect_one();
    // multi-rank boundary signal (stage_ws.cuh): the epilogue releases tile j's accumulator after its
    // stores; this warp acquires that release before reusing the accumulator for tile j + NACC
    const int nbl = BSIG ? int(bsig_ctiles(p.bsig_tiles)) : 0;
    if constexpr (C::OP_RES) tc_wait_mma(b_full, 0);
    int slot = 0, bsl = 0;       // operand ring (TMEM) and operator ring positions
    unsigned aph = 0, bph = 0;   // their phases
    for (int j = 0; j < J; ++j) {
      const int a = j % C::NACC;
      tc_wait_mma(acc_empty + a, (unsigned(j / C::NACC) & 1) ^ 1);
      if constexpr (BSIG)
        if (leader) loader_signal_after_wait(p.bsig, nbl, j, C::NACC);
      const uint32_t d = tmem + uint32_t(a * C::ACC1);
      int wb = 0;  // position in the writers' batch of WB chunks
      for (int s = 0; s < NQ; ++s) {
        TC_T(t0);
        // N <= 6: the writers publish a batch of WB chunks together (one tcgen05.wait::st, arrivals
        // in chunk order), so the batch's last chunk being complete implies the others: one wait +
        // one fence per batch.  N >= 7, where the writers bound the pipe, waiting per chunk lets the
        // MMA start earlier.
        const bool bstart = !C::FUSE_LO || wb == 0;
        if (bstart) {
          int ls = slot;
          unsigned lph = aph;
          if constexpr (C::FUSE_LO) {
            ls += (NQ - s < C::WB ? NQ - s : C::WB) - 1;
            if (ls >= RA) {
              ls -= RA;
              lph ^= 1u;
            }
          }
          tc_wait_mma(a_full + ls, lph);
        }
        TC_A(7, t0);
        uint64_t db;
        if constexpr (C::OP_RES) {
          db = db0 + uint64_t(s) * DCH;
        } else {
          TC_T(t2);
          tc_wait_mma(b_full + bsl, bph);
          TC_A(9, t2);
          db = db0 + uint64_t(bsl) * DCH;
        }
        TC_T(t1);
        if (bstart && !(DG_TC_X & 32)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem + uint32_t(C::a_col(slot));  // G at ta, G_lo at ta + 8
        if (leader) {
          if constexpr (C::FUSE_LO) {
            tc_mma_ts(d, ta, db, idesc2, s > 0 ? 1u : 0u);         // G . [Op | Op_lo]  (2 NP16 columns)
            tc_mma_ts(d, ta + 8, db, idesc, 1u);                   // G_lo . Op         (first NP16)
          } else {
            tc_mma_ts(d, ta, db, idesc, s > 0 ? 1u : 0u);          // G . Op
            tc_mma_ts(d, ta + 8, db, idesc, 1u);                   // G_lo . Op
            tc_mma_ts(d, ta, db + DLO, idesc, 1u);                 // G . Op_lo
          }
          // frees the TMEM operand slots in pairs (one commit per two chunks: ~45 cycles each)
          if (slot & 1) tc_commit(a_empty + (slot >> 1));
          if constexpr (!C::OP_RES) tc_commit(b_empty + bsl);       // frees the operator slot
          if (s == NQ - 1) tc_commit(acc_full + a);                 // accumulator complete
        }
        __syncwarp();
        TC_A(10, t1);
        if (++slot == RA) {
          slot = 0;
          aph ^= 1u;
        }
        if constexpr (!C::OP_RES) {
          if (++bsl == RB) {
            bsl = 0;
            bph ^= 1u;
          }
        }
        if (++wb == C::WB) wb = 0;
      }
    }
    if constexpr (BSIG)
      if (leader) loader_signal_tail(acc_empty, p.bsig, nbl, J, C::NACC);
  } else if (warp < C::W_FG0) {
    // ============ operand writers: G chunks into the TMEM ring, in MMA order ============
    // Lane-owning warps (warp % 4 = TMEM lane quarter): row r = 32 (warp % 4) + lane.
    // Volume chunk (octet o, derivative d) (a1): G = al_d u_f1 + be_d u_f2 from the slab;
    // flux chunk (a2 + a3): G = the flux warps' values from the staging ring.  Written with
    // tcgen05.st (no generic->async proxy fence on the path), G_lo = G - trunc_tf32(G).
    const int r = 32 * (warp & 3) + lane, e = r / NC, out = r - NC * (r / NC);
    // Maxwell: row -> (first field, its derivative direction, second field, its direction, sign):
    // rhsE = curl H, rhsH = -curl E;  out: Ex Ey Ez Hx Hy Hz
    // Acoustics (R16): rhs_p = -div v -> fields vx, vy, vz with directions x, y, z;
    // rhs_va = -d_a p -> field p with direction a (one term; the others have zero coefficients)
    int f1, f2, f3 = 0, x1, x2, x3 = 0;
    float sg;
    if constexpr (SYS == 0) {
      f1 = out < 3 ? (out == 0 ? 5 : out == 1 ? 3 : 4) : (out == 3 ? 2 : out == 4 ? 0 : 1);
      f2 = out < 3 ? (out == 0 ? 4 : out == 1 ? 5 : 3) : (out == 3 ? 1 : out == 4 ? 2 : 0);
      x1 = out % 3 == 0 ? 1 : out % 3 == 1 ? 2 : 0;  // curl_x = d_y(.) - d_z(.), cyclic
      x2 = out % 3 == 0 ? 2 : out % 3 == 1 ? 0 : 1;
      sg = out < 3 ? 1.0f : -1.0f;
    } else {
      f1 = out == 0 ? 1 : 0, f2 = out == 0 ? 2 : 0, f3 = out == 0 ? 3 : 0;
      x1 = out == 0 ? 0 : out - 1, x2 = 1, x3 = 2;
      sg = -1.0f;
    }
    const uint32_t trow = tmem + (uint32_t(32 * (warp & 3)) << 16);
    int ga = 0, gs = 0, gf = 0;
    for (int j = 0; j < J; ++j) {
      const int tile = tile_of(j);
      const bool valid = r < ROWS && e < count_of(tile);
      static_assert(C::RA >= C::WB, "TMEM ring holds a writer batch");
      float al[3], be[3], gm3[3];
      tc_wait(m_full + j % RM, unsigned(j / RM) & 1);
      {
        const float* g = sGeo(j) + (valid ? e : 0) * GEO_W;
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {  // g[3 d + a] = d r_d / d x_a (eq. 6)
          if constexpr (SYS == 0) {
            al[dd] = valid ? sg * g[3 * dd + x1] : 0.0f;
            be[dd] = valid ? -sg * g[3 * dd + x2] : 0.0f;
            gm3[dd] = 0.0f;
          } else {
            al[dd] = valid ? sg * g[3 * dd + x1] : 0.0f;
            be[dd] = valid && out == 0 ? sg * g[3 * dd + x2] : 0.0f;
            gm3[dd] = valid && out == 0 ? sg * g[3 * dd + x3] : 0.0f;
          }
        }
      }
      // generic-proxy reads of a TMA-written (async-proxy) buffer must be ordered before the
      // next TMA write into it: proxy fence before releasing the slot (cross-proxy WAR)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(m_empty + j % RM);
      float u1[8], u2[8], u3[8];
      int v = 0, f = 0;
      TC_T(t1);
      // WB steps per batch: one tcgen05.wait::st for WB chunk stores.  For small NQ the whole
      // tile schedule is unrolled, so the volume/flux interleave is resolved at compile time.
#pragma unroll(C::WUNR)
      for (int s0 = 0; s0 < NQ; s0 += C::WB) {
        const int nb = NQ - s0 < C::WB ? NQ - s0 : C::WB;
        float vv[C::WB][8];
#pragma unroll
        for (int bq = 0; bq < C::WB; ++bq) {
          if (bq < nb) {
            if (tc_is_vol(v, f, NV, NFQ)) {
              const int o = v / 3, dd = v - 3 * o;
              if (dd == 0) {  // a new octet slab: its two fields for this row
                const int ss = gs % RS;
                TC_T(t0);
                tc_wait(s_full + ss, unsigned(gs / RS) & 1);
                TC_A(2, t0);
                const float* sl = sS + ss * C::SLABF + NC * e;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  const bool ok = valid && 8 * o + jj < Np && !(DG_TC_X & 2);
                  u1[jj] = ok ? sl[jj * ROWS + f1] : 0.0f;
                  u2[jj] = ok ? sl[jj * ROWS + f2] : 0.0f;
                  if constexpr (SYS == 1) u3[jj] = ok ? sl[jj * ROWS + f3] : 0.0f;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cross-proxy WAR (see above)
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty + ss);
                ++gs;
              }
              const float a1 = dd == 0 ? al[0] : dd == 1 ? al[1] : al[2];
              const float b1 = dd == 0 ? be[0] : dd == 1 ? be[1] : be[2];
              if constexpr (SYS == 0) {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) vv[bq][jj] = a1 * u1[jj] + b1 * u2[jj];
              } else {
                const float c1 = dd == 0 ? gm3[0] : dd == 1 ? gm3[1] : gm3[2];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) vv[bq][jj] = a1 * u1[jj] + b1 * u2[jj] + c1 * u3[jj];
              }
              ++v;
            } else {
              const int fs = gf % LF;
              TC_T(t0);
              tc_wait(f_full + fs, unsigned(gf / LF) & 1);
              TC_A(2, t0);
              const float4* src = reinterpret_cast<const float4*>(sFS + fs * C::FSC + 8 * r);
              const float4 x = src[0], y = src[1];
              const bool ok = r < ROWS;  // rows ROWS..127 of the MMA are padding: keep them zero
              vv[bq][0] = ok ? x.x : 0.0f;
              vv[bq][1] = ok ? x.y : 0.0f;
              vv[bq][2] = ok ? x.z : 0.0f;
              vv[bq][3] = ok ? x.w : 0.0f;
              vv[bq][4] = ok ? y.x : 0.0f;
              vv[bq][5] = ok ? y.y : 0.0f;
              vv[bq][6] = ok ? y.z : 0.0f;
              vv[bq][7] = ok ? y.w : 0.0f;
              __syncwarp();
              if (lane == 0) mbar_arrive(f_empty + fs);
              ++gf;
              ++f;
            }
          }
        }
        TC_A(4, t1);
        TC_T(t2);
#pragma unroll
        for (int bq = 0; bq < C::WB; ++bq) {
          if (bq < nb) {
            const int slot = (ga + bq) % RA;
            tc_wait(a_empty + (slot >> 1), (unsigned((ga + bq) / RA) & 1) ^ 1);  // the slot pair's release
            // orders this store after the MMAs that read the slot (their commit completed the wait)
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef DG_WS_PROFILE
            if (g_tc_dbg) {
              float* dp = g_tc_dbg + ((size_t(tile) * NQ + (s0 + bq)) * 128 + r) * 8;
              for (int jj = 0; jj < 8; ++jj) dp[jj] = vv[bq][jj];
            }
#endif
            uint32_t w[16];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              w[jj] = __float_as_uint(vv[bq][jj]);
              w[8 + jj] = __float_as_uint(tf32_lo(vv[bq][jj]));
            }
            if (!(DG_TC_X & 4))
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::
                    "r"(trow + uint32_t(C::a_col(slot))),
                "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),
                "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
                : "memory");
          }
        }
        TC_A(3, t2);
#ifdef DG_WS_PROFILE
        t1 = clock64();
#endif
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0)
          for (int bq = 0; bq < nb; ++bq) mbar_arrive(a_full + (ga + bq) % RA);
        ga += nb;
      }
      TC_A(4, t1);
    }
  } else {
    // ============ flux (a2 + a3): upwind/PEC flux x Fscale/2 -> flux staging ============
    // Item (element e, face-node slot kk) per thread and chunk.  Its traces u- and u+ are
    // cp.async'ed LT - 1 chunks ahead into this thread's own staging slots (per-thread
    // cp.async groups: no cross-thread synchronisation); the flux goes to the staging ring
    // as plain shared stores, which the operand writers pick up.
    const int ft = tid - 32 * C::W_FG0;
    const int kk = ft & 7, e = ft >> 3;
    const bool item = ft < ITEMS;
    const int TOT = J * NFQ;
    const uint16_t* sQ = reinterpret_cast<const uint16_t*>(sGP + 6 * Nfp);  // [NFQ][8]: f | i << 2 | Fmask << 8
    float* const stg0 = sTR + 2 * ft;   // this thread's staging words: + (slot * NC + pair) * 2 * FTH
    constexpr int PST = 2 * C::FTH;     // floats between pairs
    constexpr int PH = NC / 2;          // component pairs per side (u- pairs 0..PH-1, u+ pairs PH..NC-1)
    // issue side: (tile, chunk) = (ji, qi), staging slot si
    int ji = 0, qi = 0, si = 0;
    bool act_i = false;
    const float* uT_i = p.u_in;
    const int32_t* cn_i = nullptr;
    int codes_i = 0;
    auto issue = [&]() {
      if (qi == 0) {
        tc_wait(m_full + ji % RM, unsigned(ji / RM) & 1);
        const int tile = tile_of(ji);
        act_i = item && e < count_of(tile);
        uT_i = p.u_in + tile * TS + NC * e;
        cn_i = sConn(ji) + 4 * e;
        codes_i = sConn(ji)[4 * E + e];
      }
      const int code = sQ[qi * 8 + kk];  // 0xffff: slot past the last face node
      if (act_i && code != 0xffff && !(DG_TC_X & 1)) {
        const int f = code & 3, i = (code >> 2) & 63;
        float* d = stg0 + si * NC * PST;
        const float* src = uT_i + (code >> 8) * ROWS;
#pragma unroll
        for (int c = 0; c < PH; ++c) cp_async8(d + c * PST, src + 2 * c);
        const int32_t b = cn_i[f];
        const int cd = (codes_i >> (8 * f)) & 0xff;
        if (b >= 0) {  // local neighbour: word offset of its node 0, component 0
          const float* g = p.u_in + b + int(sNP[cd * Nfp + i]) * ROWS;
#pragma unroll
          for (int c = 0; c < PH; ++c) cp_async8(d + (PH + c) * PST, g + 2 * c);
        } else if (b != -1) {  // partition face: the peer's ghost record (b = -2 - record)
          const float* g = p.u_in + p.ghost_base + TileLayout::ghost_rec(b) + sGP[cd * Nfp + i];
#pragma unroll
          for (int c = 0; c < NC; ++c) cp_async4(d + (PH + c / 2) * PST + (c & 1), g + c * Nfp);
        }
      }
      cp_commit();
      if (++si == LT) si = 0;
      if (++qi == NFQ) {
        qi = 0;
        ++ji;
      }
    };
    TC_T(tw);
    for (int G = 0; G < LT - 1; ++G) {  // always LT - 1 groups, so cp_wait<LT - 1> below covers chunk G
      if (G < TOT)
        issue();
      else
        cp_commit();
    }
    int j = 0, q = 0, sc_ = 0, fsl = 0;
    unsigned fph = 0;
    bool act = false;
    const float* gE = nullptr;
    const int32_t* cn = nullptr;
    for (int G = 0; G < TOT; ++G) {
      if (q == 0) {
        act = item && e < count_of(tile_of(j));
        gE = sGeo(j) + e * GEO_W + 9;
        cn = sConn(j) + 4 * e;
      }
      if (G + LT - 1 < TOT)
        issue();
      else
        cp_commit();
#ifdef DG_TC_SYNCFLUX
      cp_wait<0>();
#else
      cp_wait<LT - 1>();  // this thread's copies for chunk G have landed
#endif
      const int code = sQ[q * 8 + kk];
      float fl[6] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
      if (act && code != 0xffff && !(DG_TC_X & 1)) {
        const int f = code & 3;
        const float* gm = gE + 4 * f;
        const float nx = gm[0], ny = gm[1], nz = gm[2], fs = gm[3];
        const bool wall = cn[f] == -1;  // boundary face (ghost records are -2 - record)
        const float* d = stg0 + sc_ * NC * PST;
        float uM[NC], uP[NC];
#pragma unroll
        for (int c = 0; c < PH; ++c) {
          const float2 a2 = *reinterpret_cast<const float2*>(d + c * PST);
          uM[2 * c] = a2.x;
          uM[2 * c + 1] = a2.y;
          const float2 b2 = *reinterpret_cast<const float2*>(d + (PH + c) * PST);
          uP[2 * c] = b2.x;
          uP[2 * c + 1] = b2.y;
        }
        if constexpr (SYS == 0) {
          float dE[3], dH[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {  // PEC wall: E+ = -E-, H+ = H-
            dE[c] = wall ? -2.0f * uM[c] : uP[c] - uM[c];
            dH[c] = wall ? 0.0f : uP[c + 3] - uM[c + 3];
          }
          maxwell_flux<float>(nx, ny, nz, p.alpha, dE, dH, fl);
        } else {  // rigid wall (R17): p+ = p-, v+ = v- - 2 (n.v-) n
          const float ndv = nx * uM[1] + ny * uM[2] + nz * uM[3];
          const float dp = wall ? 0.0f : uP[0] - uM[0];
          float dv[3];
          dv[0] = wall ? -2.0f * ndv * nx : uP[1] - uM[1];
          dv[1] = wall ? -2.0f * ndv * ny : uP[2] - uM[2];
          dv[2] = wall ? -2.0f * ndv * nz : uP[3] - uM[3];
          acoustic_flux<float>(nx, ny, nz, p.alpha, dp, dv, fl);
        }
        const float sc = 0.5f * fs;
#pragma unroll
        for (int c = 0; c < NC; ++c) fl[c] *= sc;
      }
      if (++sc_ == LT) sc_ = 0;
      TC_T(t0);
      tc_wait(f_empty + fsl, fph ^ 1);
      TC_A(5, t0);
      if (item) {
        float* F = sFS + fsl * C::FSC + 8 * NC * e + kk;  // [row NC e + c][kk]
#pragma unroll
        for (int c = 0; c < NC; ++c) F[8 * c] = fl[c];
      }
      if (q == NFQ - 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // meta slot: cross-proxy WAR
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(f_full + fsl);
        if (q == NFQ - 1) mbar_arrive(m_empty + j % RM);  // done with this tile's meta slot
      }
      if (++fsl == LF) {
        fsl = 0;
        fph ^= 1;
      }
      if (++q == NFQ) {
        q = 0;
        ++j;
      }
    }
    TC_A(6, tw);
  }
#ifdef DG_WS_PROFILE
  if (lane == 0)
    for (int i = 0; i < 12; ++i)
      if (tcp[i]) atomicAdd(&g_tc_prof[i], tcp[i]);
#endif
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == C::W_MMA) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

template <int N, int SYS>
void launch_stage_tc_sys(const StageParams<float>& p, const float* ops, int mode, cudaStream_t st) {
  using C = TcCfg<N, SYS>;
  static PerDevice pd;
  const int sms = sms_for_device(pd, [] {
    cudaFuncSetAttribute(dg_stage_tc<N, true, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaFuncSetAttribute(dg_stage_tc<N, false, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaFuncSetAttribute(dg_stage_tc<N, true, SYS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
  });
  if (p.K <= 0) return;
  const int64_t t0 = p.k_begin / C::E;
  const int64_t tc = (p.k_begin + p.K + C::E - 1) / C::E - t0;
  const int cap = sms - p.sm_reserve > 1 ? sms - p.sm_reserve : 1;  // SMs left to concurrent NCCL kernels
  const unsigned grid = unsigned(tc < cap ? tc : cap);
  if (mode == 1 && p.bsig)
    launch_pdl(true, dg_stage_tc<N, true, SYS, true>, grid, C::NT, C::SMEM_BYTES, st, p, ops, t0, tc);
  else if (mode == 1)
    launch_pdl(true, dg_stage_tc<N, true, SYS>, grid, C::NT, C::SMEM_BYTES, st, p, ops, t0, tc);
  else
    launch_pdl(true, dg_stage_tc<N, false, SYS>, grid, C::NT, C::SMEM_BYTES, st, p, ops, t0, tc);
}
template <int N>
void launch_stage_tc(const StageParams<float>& p, const float* ops, int mode, cudaStream_t st) {
  if (p.system == 1)
    launch_stage_tc_sys<N, 1>(p, ops, mode, st);
  else
    launch_stage_tc_sys<N, 0>(p, ops, mode, st);
}

// perm 4: node-major tiles of E elements, (k / E) * TS + n * NC E + NC (k % E) + c
template <int N>
TileLayout tc_layout(int nc) {
  TileLayout L;
  L.nc = nc;
  L.E = nc == 4 ? TcCfg<N, 1>::E : TcCfg<N, 0>::E;
  L.LD = TcCfg<N, 0>::Np;
  L.perm = 4;
  L.TS = nc == 4 ? TcCfg<N, 1>::TS : TcCfg<N, 0>::TS;
  return L;
}

// host: the operator chunks in MMA order, canonical K-major 8-k chunks, split for 3xTF32 with
// hardware truncation (hi = trunc_tf32(float(v)), lo = float(v - hi)): chunk s = [hi | lo].
template <int N>
void tc_ops(const double* Dr, const double* Ds, const double* Dt, const double* LIFT, float* out) {
  using C = TcCfg<N>;
  constexpr int Np = C::Np, NF = C::NF, NP16 = C::NP16;
  auto trunc32 = [](double v) -> float {
    float f = float(v);
    unsigned u;
    std::memcpy(&u, &f, 4);
    u &= 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  const double* D[3] = {Dr, Ds, Dt};
  int v = 0, f = 0;
  for (int s = 0; s < C::NQ; ++s) {
    const bool vol = tc_is_vol(v, f, C::NV, C::NFQ);
    float* hi = out + size_t(s) * C::OPC;
    float* lo = hi + 8 * NP16;
    for (int n = 0; n < NP16; ++n)
      for (int kk = 0; kk < 8; ++kk) {
        double val = 0.0;
        if (n < Np) {
          if (vol) {
            const int m = 8 * (v / 3) + kk;
            if (m < Np) val = D[v % 3][n * Np + m];
          } else {
            const int m = 8 * f + kk;
            if (m < NF) val = LIFT[n * NF + m];
          }
        }
        const float h = trunc32(val);
        hi[tc_cm(n, kk)] = h;
        lo[tc_cm(n, kk)] = float(val - double(h));
      }
    if (vol)
      ++v;
    else
      ++f;
  }
}

}  // namespace dg
