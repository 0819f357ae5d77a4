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

namespace dg {

// the MMA's fixed interleave of the NV volume and NFQ flux chunks of a tile
__host__ __device__ constexpr bool tc_is_vol(int v, int f, int NV, int NFQ) {
  return f >= NFQ || (v < NV && v * NFQ <= f * NV);
}

template <int N>
struct TcCfg {
  static constexpr int Np = Order<N>::Np, Nfp = Order<N>::Nfp, NF = Order<N>::NF;
  static constexpr int E = 21;                      // elements per tile
  static constexpr int ROWS = 6 * E;                // 126 of the 128 MMA rows
  static constexpr int NP16 = (Np + 15) / 16 * 16;  // MMA N
  static constexpr int NO = (Np + 7) / 8;           // node octets
  static constexpr int NV = 3 * NO;                 // volume chunks
  static constexpr int NFQ = (NF + 7) / 8;          // flux chunks
  static constexpr int NQ = NV + NFQ;
  static constexpr int TS = (ROWS * Np + 7) / 8 * 8;  // floats per tile (node-major)
  static constexpr int SLABF = 1024;                // floats per slab slot (8 x 126 used)
  static constexpr int OPC = 2 * 8 * NP16;          // floats per operator chunk (hi | lo)
  static constexpr int ACH = 2 * 128 * 8;           // floats per generated chunk (hi | lo)
  static constexpr bool OP_RES = N <= 4;            // operators resident in shared memory
  static constexpr int RB = OP_RES ? NQ : 4;
  static constexpr int RS = 4;
  static constexpr int RV = 8, RF = 6;
  static constexpr int PW = 6;                      // flux warps (>= 168 items per chunk)
  // 16 warps: 4 per SMSP, so every thread can have 128 registers
  static constexpr int W_LD = 4, W_MMA = 5, W_VG0 = 6, W_FG0 = 10;
  static constexpr int NW = W_FG0 + PW;
  static constexpr int NT = 32 * NW;
  static constexpr int TMEM_COLS = 2 * NP16 <= 32 ? 32 : 2 * NP16 <= 64 ? 64 : 2 * NP16 <= 128 ? 128
                                   : 2 * NP16 <= 256 ? 256 : 512;
  static constexpr int NTAB = NF + 24 * Nfp + 6 * Nfp;  // int16: Fmask | node table | ghost table
  static constexpr int al1k(int b) { return (b + 1023) / 1024 * 1024; }
  static constexpr int OFF_B = 0;
  static constexpr int OFF_AV = OFF_B + al1k(RB * OPC * 4);
  static constexpr int OFF_AF = OFF_AV + RV * ACH * 4;
  static constexpr int OFF_S = OFF_AF + RF * ACH * 4;
  static constexpr int OFF_T = OFF_S + RS * SLABF * 4;
  static constexpr int OFF_BAR = OFF_T + (NTAB * 2 + 15) / 16 * 16;
  static constexpr int NBAR = 2 * RB + 2 * RV + 2 * RF + 2 * RS + 4;
  static constexpr size_t SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(PW * 32 >= 8 * E, "one flux item per thread and chunk");
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
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
// word offset of (row, kk) inside an 8-k chunk of the canonical K-major layout
__host__ __device__ constexpr int tc_cm(int r, int kk) { return ((r >> 3) * 2 + (kk >> 2)) * 32 + (r & 7) * 4 + (kk & 3); }

template <int N, bool UPDATE>
__global__ void __launch_bounds__(TcCfg<N>::NT, 1)
    dg_stage_tc(const StageParams<float> p, const float* __restrict__ ops, int64_t t_begin, int64_t t_count) {
  using C = TcCfg<N>;
  constexpr int Np = C::Np, Nfp = C::Nfp, NF = C::NF, E = C::E, ROWS = C::ROWS, NP16 = C::NP16;
  constexpr int NO = C::NO, NV = C::NV, NFQ = C::NFQ, NQ = C::NQ, TS = C::TS;
  constexpr int RB = C::RB, RS = C::RS, RV = C::RV, RF = C::RF;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  unsigned char* smem = smem_tc;
  pdl_trigger();
  float* sB = reinterpret_cast<float*>(smem + C::OFF_B);
  float* sAV = reinterpret_cast<float*>(smem + C::OFF_AV);
  float* sAF = reinterpret_cast<float*>(smem + C::OFF_AF);
  float* sS = reinterpret_cast<float*>(smem + C::OFF_S);
  int16_t* sFm = reinterpret_cast<int16_t*>(smem + C::OFF_T);
  const int16_t* sNP = sFm + NF;          // [24][Nfp] neighbour node of face node i, by f2*6 + orientation
  const int16_t* sGP = sNP + 24 * Nfp;    // [6][Nfp]  ghost record position, by orientation
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* b_full = bars;
  uint64_t* b_empty = b_full + RB;
  uint64_t* av_full = b_empty + RB;
  uint64_t* av_empty = av_full + RV;
  uint64_t* af_full = av_empty + RV;
  uint64_t* af_empty = af_full + RF;
  uint64_t* s_full = af_empty + RF;
  uint64_t* s_empty = s_full + RS;
  uint64_t* acc_full = s_empty + RS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t J = t_count > blockIdx.x ? (t_count - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t kend = p.k_begin + p.K;
  auto tile_of = [&](int64_t j) { return t_begin + blockIdx.x + j * gridDim.x; };
  auto count_of = [&](int64_t tile) {
    const int64_t k0 = tile * E;
    return int(kend - k0 < E ? kend - k0 : E);
  };

  if (tid == 0) {
    for (int i = 0; i < RB; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    for (int i = 0; i < RV; ++i) {
      mbar_init(av_full + i, 4);
      mbar_init(av_empty + i, 1);
    }
    for (int i = 0; i < RF; ++i) {
      mbar_init(af_full + i, C::PW);
      mbar_init(af_empty + i, 1);
    }
    for (int i = 0; i < RS; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 4);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == C::W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // generated-operand rings start zeroed: rows 126, 127 are never written and must stay finite
  for (int w = tid; w < (RV + RF) * C::ACH; w += C::NT) sAV[w] = 0.0f;
  for (int w = tid; w < C::NTAB; w += C::NT) sFm[w] = p.ftab[w];
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
    const int r = 32 * warp + lane, e = r / 6;
    const bool res_in = UPDATE && !p.first_stage;
    for (int64_t j = 0; j < J; ++j) {
      const int a = int(j & 1);
      const int64_t tile = tile_of(j);
      const bool valid = r < ROWS && e < count_of(tile);
      const int64_t base = tile * TS + r;
      auto ld_grp = [&](int c0, float (&uv)[16], float (&rv)[16]) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = c0 + i;
          const bool ok = UPDATE && valid && n < Np;
          const int64_t o = base + int64_t(ok ? n : 0) * ROWS;
          uv[i] = ok ? __ldg(p.u_in + o) : 0.0f;
          rv[i] = ok && res_in ? p.res[o] : 0.0f;
        }
      };
      auto process = [&](int c0, const float (&uv)[16], const float (&rv)[16]) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + (uint32_t(32 * warp) << 16) + uint32_t(a * NP16 + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (valid) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = c0 + i;
            if (n < Np) {
              const int64_t o = base + int64_t(n) * ROWS;
              const float d = __uint_as_float(v[i]);
              if (UPDATE) {
                const float rr = p.rk_a * rv[i] + p.dt * d;
                p.res[o] = rr;
                p.u_out[o] = uv[i] + p.rk_b * rr;
              } else {
                p.rhs_out[o] = d;
              }
            }
          }
        }
      };
      float ua[16], ra[16], ub[16], rb[16];
      ld_grp(0, ua, ra);
      mbar_wait(acc_full + a, unsigned(j >> 1) & 1);
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
    }
  } else if (warp == C::W_LD) {
    // ===================== slab loader (field tiles) =====================
    if (lane == 0) {
      for (int64_t j = 0; j < J; ++j) {
        const float* src = p.u_in + tile_of(j) * TS;
        for (int o = 0; o < NO; ++o) {
          const int64_t g = j * NO + o;
          const int s = int(g % RS);
          mbar_wait(s_empty + s, (unsigned(g / RS) & 1) ^ 1);
          const int nodes = Np - 8 * o < 8 ? Np - 8 * o : 8;
          unsigned bytes = unsigned(nodes * ROWS * 4);
          bytes = (bytes + 15) & ~15u;  // an odd node count ends 8 B short; the tile padding covers it
          mbar_arrive_tx(s_full + s, bytes);
          bulk_g2s(sS + s * C::SLABF, src + 8 * o * ROWS, bytes, s_full + s);
        }
      }
    } else if (lane == 1) {
      // ====================== operator loader ======================
      if constexpr (C::OP_RES) {
        mbar_arrive_tx(b_full, unsigned(C::OPS_FLOATS * 4));
        bulk_g2s(sB, ops, unsigned(C::OPS_FLOATS * 4), b_full);
      } else {
        for (int64_t j = 0; j < J; ++j) {
          for (int s = 0; s < NQ; ++s) {
            const int64_t g = j * NQ + s;
            const int b = int(g % RB);
            mbar_wait(b_empty + b, (unsigned(g / RB) & 1) ^ 1);
            mbar_arrive_tx(b_full + b, unsigned(C::OPC * 4));
            bulk_g2s(sB + b * C::OPC, ops + int64_t(s) * C::OPC, unsigned(C::OPC * 4), b_full + b);
          }
        }
      }
    }
  } else if (warp == C::W_MMA) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      constexpr uint32_t idesc = tc_idesc(128, NP16);
      if constexpr (C::OP_RES) mbar_wait(b_full, 0);
      int64_t gv = 0, gf = 0;
      for (int64_t j = 0; j < J; ++j) {
        const int a = int(j & 1);
        mbar_wait(acc_empty + a, (unsigned(j >> 1) & 1) ^ 1);
        const uint32_t d = tmem + uint32_t(a * NP16);
        int v = 0, f = 0;
        for (int s = 0; s < NQ; ++s) {
          const float* A;
          uint64_t* rel;
          if (tc_is_vol(v, f, NV, NFQ)) {
            const int slot = int(gv % RV);
            mbar_wait(av_full + slot, unsigned(gv / RV) & 1);
            A = sAV + slot * C::ACH;
            rel = av_empty + slot;
            ++gv;
            ++v;
          } else {
            const int slot = int(gf % RF);
            mbar_wait(af_full + slot, unsigned(gf / RF) & 1);
            A = sAF + slot * C::ACH;
            rel = af_empty + slot;
            ++gf;
            ++f;
          }
          const float* B;
          int b = 0;
          if constexpr (C::OP_RES) {
            B = sB + s * C::OPC;
          } else {
            const int64_t g = j * NQ + s;
            b = int(g % RB);
            mbar_wait(b_full + b, unsigned(g / RB) & 1);
            B = sB + b * C::OPC;
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          tc_mma(d, tc_desc(A), tc_desc(B), idesc, s > 0 ? 1u : 0u);      // G . Op
          tc_mma(d, tc_desc(A + 1024), tc_desc(B), idesc, 1u);            // G_lo . Op
          tc_mma(d, tc_desc(A), tc_desc(B + 8 * NP16), idesc, 1u);        // G . Op_lo
          tc_commit(rel);
          if constexpr (!C::OP_RES) tc_commit(b_empty + b);
        }
        tc_commit(acc_full + a);
      }
    }
  } else if (warp < C::W_FG0) {
    // ================== volume generators (a1 operand) ==================
    const int r = tid - 32 * C::W_VG0, e = r / 6, out = r - 6 * (r / 6);
    // row -> (first field, its derivative direction, second field, its direction, sign):
    // rhsE = curl H, rhsH = -curl E;  out: Ex Ey Ez Hx Hy Hz
    const int f1 = out < 3 ? (out == 0 ? 5 : out == 1 ? 3 : 4) : (out == 3 ? 2 : out == 4 ? 0 : 1);
    const int f2 = out < 3 ? (out == 0 ? 4 : out == 1 ? 5 : 3) : (out == 3 ? 1 : out == 4 ? 2 : 0);
    const int x1 = out % 3 == 0 ? 1 : out % 3 == 1 ? 2 : 0;  // curl_x = d_y(.) - d_z(.), cyclic
    const int x2 = out % 3 == 0 ? 2 : out % 3 == 1 ? 0 : 1;
    const float sg = out < 3 ? 1.0f : -1.0f;
    for (int64_t j = 0; j < J; ++j) {
      const int64_t tile = tile_of(j);
      const bool valid = r < ROWS && e < count_of(tile);
      float al[3], be[3];
      {
        const float* g = p.geo + (tile * E + (valid ? e : 0)) * GEO_W;
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
          al[dd] = valid ? sg * __ldg(g + 3 * dd + x1) : 0.0f;
          be[dd] = valid ? -sg * __ldg(g + 3 * dd + x2) : 0.0f;
        }
      }
      for (int o = 0; o < NO; ++o) {
        const int64_t gs = j * NO + o;
        const int ss = int(gs % RS);
        mbar_wait(s_full + ss, unsigned(gs / RS) & 1);
        const float* sl = sS + ss * C::SLABF + 6 * e;
        float u1[8], u2[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const bool ok = valid && 8 * o + jj < Np;
          u1[jj] = ok ? sl[jj * ROWS + f1] : 0.0f;
          u2[jj] = ok ? sl[jj * ROWS + f2] : 0.0f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + ss);
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
          const int64_t gv = gs * 3 + dd;
          const int slot = int(gv % RV);
          mbar_wait(av_empty + slot, (unsigned(gv / RV) & 1) ^ 1);
          float* A = sAV + slot * C::ACH;
          float vv[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) vv[jj] = al[dd] * u1[jj] + be[dd] * u2[jj];
          float4* h0 = reinterpret_cast<float4*>(A + tc_cm(r, 0));
          float4* h1 = reinterpret_cast<float4*>(A + tc_cm(r, 4));
          float4* l0 = reinterpret_cast<float4*>(A + 1024 + tc_cm(r, 0));
          float4* l1 = reinterpret_cast<float4*>(A + 1024 + tc_cm(r, 4));
          *h0 = make_float4(vv[0], vv[1], vv[2], vv[3]);
          *h1 = make_float4(vv[4], vv[5], vv[6], vv[7]);
          *l0 = make_float4(tf32_lo(vv[0]), tf32_lo(vv[1]), tf32_lo(vv[2]), tf32_lo(vv[3]));
          *l1 = make_float4(tf32_lo(vv[4]), tf32_lo(vv[5]), tf32_lo(vv[6]), tf32_lo(vv[7]));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05.mma operand
          __syncwarp();
          if (lane == 0) mbar_arrive(av_full + slot);
        }
      }
    }
  } else {
    // ============== flux generators (a2 + a3: lift operand) ==============
    const int ft = tid - 32 * C::W_FG0;
    const int kk = ft & 7, e = ft >> 3;
    const bool item = e < E;
    for (int64_t j = 0; j < J; ++j) {
      const int64_t tile = tile_of(j);
      const bool act = item && e < count_of(tile);
      const int64_t k = tile * E + (act ? e : 0);
      float nrm[4][4];
      int32_t fb[4];
      int fcd[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
#pragma unroll
        for (int i = 0; i < 4; ++i) nrm[f][i] = __ldg(p.geo + k * GEO_W + 9 + 4 * f + i);
        fb[f] = act ? __ldg(p.gidx + 4 * k + f) : -1;
        fcd[f] = __ldg(p.fcode + 4 * k + f);
      }
      const float* uT = p.u_in + tile * TS + 6 * e;
      // one face node's traces: u- from the element, u+ from the neighbour / ghost record / PEC mirror
      auto load = [&](int q, float (&uM)[6], float (&uP)[6], int& kind) {
        const int m = 8 * q + kk;
        kind = 0;  // 0: nothing (padding / absent element), 1: PEC wall, 2: interior face
        if (act && m < NF) {
          const int f = m / Nfp, i = m - f * Nfp;
          const float* src = uT + int(sFm[m]) * ROWS;
#pragma unroll
          for (int c = 0; c < 6; ++c) uM[c] = src[c];
          const int32_t b = f == 0 ? fb[0] : f == 1 ? fb[1] : f == 2 ? fb[2] : fb[3];
          const int cd = f == 0 ? fcd[0] : f == 1 ? fcd[1] : f == 2 ? fcd[2] : fcd[3];
          if (b < 0) {
            kind = 1;
          } else if (b & TileLayout::GHOST_FLAG) {
            const float* g = p.u_in + p.ghost_base + (b & ~TileLayout::GHOST_FLAG) + sGP[cd * Nfp + i];
#pragma unroll
            for (int c = 0; c < 6; ++c) uP[c] = g[c * Nfp];
            kind = 2;
          } else {
            const float* g = p.u_in + b + int(sNP[cd * Nfp + i]) * ROWS;
#pragma unroll
            for (int c = 0; c < 6; ++c) uP[c] = g[c];
            kind = 2;
          }
        }
      };
      auto emit = [&](int q, const float (&uM)[6], const float (&uP)[6], int kind) {
        float fl[6] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        if (kind) {
          const int f = (8 * q + kk) / Nfp;
          const float nx = f == 0 ? nrm[0][0] : f == 1 ? nrm[1][0] : f == 2 ? nrm[2][0] : nrm[3][0];
          const float ny = f == 0 ? nrm[0][1] : f == 1 ? nrm[1][1] : f == 2 ? nrm[2][1] : nrm[3][1];
          const float nz = f == 0 ? nrm[0][2] : f == 1 ? nrm[1][2] : f == 2 ? nrm[2][2] : nrm[3][2];
          const float fs = f == 0 ? nrm[0][3] : f == 1 ? nrm[1][3] : f == 2 ? nrm[2][3] : nrm[3][3];
          float dE[3], dH[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {  // PEC wall: E+ = -E-, H+ = H-
            dE[c] = kind == 2 ? uP[c] - uM[c] : -2.0f * uM[c];
            dH[c] = kind == 2 ? uP[c + 3] - uM[c + 3] : 0.0f;
          }
          maxwell_flux<float>(nx, ny, nz, p.alpha, dE, dH, fl);
          const float sc = 0.5f * fs;
#pragma unroll
          for (int c = 0; c < 6; ++c) fl[c] *= sc;
        }
        const int64_t gq = j * NFQ + q;
        const int slot = int(gq % RF);
        mbar_wait(af_empty + slot, (unsigned(gq / RF) & 1) ^ 1);
        float* A = sAF + slot * C::ACH;
        if (item) {
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            const int o = tc_cm(6 * e + c, kk);
            A[o] = fl[c];
            A[1024 + o] = tf32_lo(fl[c]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(af_full + slot);
      };
      float xM[6], xP[6], yM[6], yP[6];
      int xk = 0, yk = 0;
#pragma unroll
      for (int c = 0; c < 6; ++c) xM[c] = xP[c] = yM[c] = yP[c] = 0.0f;
      load(0, xM, xP, xk);
#pragma unroll 1
      for (int q = 0; q < NFQ; q += 2) {
        if (q + 1 < NFQ) load(q + 1, yM, yP, yk);
        emit(q, xM, xP, xk);
        if (q + 1 < NFQ) {
          if (q + 2 < NFQ) load(q + 2, xM, xP, xk);
          emit(q + 1, yM, yP, yk);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == C::W_MMA) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

template <int N>
void launch_stage_tc(const StageParams<float>& p, const float* ops, int mode, cudaStream_t st) {
  using C = TcCfg<N>;
  static PerDevice pd;
  const int sms = sms_for_device(pd, [] {
    cudaFuncSetAttribute(dg_stage_tc<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
    cudaFuncSetAttribute(dg_stage_tc<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM_BYTES));
  });
  if (p.K <= 0) return;
  const int64_t t0 = p.k_begin / C::E;
  const int64_t tc = (p.k_begin + p.K + C::E - 1) / C::E - t0;
  const unsigned grid = unsigned(tc < sms ? tc : sms);
  if (mode == 1)
    launch_pdl(true, dg_stage_tc<N, true>, grid, C::NT, C::SMEM_BYTES, st, p, ops, t0, tc);
  else
    launch_pdl(true, dg_stage_tc<N, false>, grid, C::NT, C::SMEM_BYTES, st, p, ops, t0, tc);
}

// perm 4: node-major tiles of E elements, (k / E) * TS + n * 6E + 6 (k % E) + c
template <int N>
TileLayout tc_layout() {
  using C = TcCfg<N>;
  TileLayout L;
  L.E = C::E;
  L.LD = C::Np;
  L.perm = 4;
  L.TS = C::TS;
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
