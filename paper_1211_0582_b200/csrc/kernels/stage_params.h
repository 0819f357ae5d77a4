// Parameters shared by the host launcher and the stage kernels.
//
// Device data layout:
//   u, res      [Kl + ghosts][ES] words; element k's component c, node n at
//               k*ES + c*Np + n (ES = 6*Np, rounded up to 4 words for FP32 so every
//               element tile is 16-B aligned: the microblock idea of PAPER.md:745-765)
//   ghost traces (multi-GPU) follow the local tiles: ghost face g, component c,
//               face node i at ghost_base + g*6*Nfp + c*Nfp + i
//   gidx        int32 [Kl][4*Nfp]: offset of the exterior trace u+ of face node m
//               (component 0); component stride Np for element nodes, Nfp for ghost
//               traces (offset >= ghost_base); -1 on a PEC boundary face
//               TC kernel (perm 4): compressed per face instead, per tile [TC_CONNT] int32:
//               [E][4] word offset of the neighbour's (node 0, component 0), or -2 - (ghost
//               record offset), or -1 (PEC); then [E] x 4 packed u8 codes f2*6 + orientation
//               (ghost: orientation); the face-node tables ftab rebuild the node (SURVEY §7
//               hard part 5).  geo is per tile [E][GEO_W] padded to tc_geot(E).
//   geo         [Kl][GEO_W]: rx ry rz sx sy sz tx ty tz, then 4 x (nx ny nz Fscale)
//   ops         Dr | Ds | Dt ([Np][Np] each, row-major) | LIFT ([Np][4Nfp])
//   fmask       int16 [4*Nfp]
//   ops_pad     (MMA variant) Dr|Ds|Dt zero-padded to [3][M8][KV], LIFT to [M8][4Nfp]
//               (M8 = Np rounded up to 8, KV = Np rounded up to 4)
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define DG_HD __host__ __device__ __forceinline__
#else
#define DG_HD inline
#endif

namespace dg {

constexpr int GEO_W = 26;  // 25 used (rx..tz, 4 x (n, Fscale)); padded to 16 B for bulk copies
// TC kernel: geometry words per tile of E elements (E x 26, padded to 16 B; 548 Maxwell, 624 acoustics)
constexpr int tc_geot(int E) { return (E * GEO_W + 3) / 4 * 4; }
constexpr int TC_CONNT = 128;  // TC kernel: connectivity words per tile

// Field layout in device memory: element k, component c, node n lives at
//   (k / E) * TS + col(k % E, c) * LD + n.
// BASIC/MMA kernels: E = 1, LD = Np, TS = ES, col = c        -> k*ES + c*Np + n
// WS kernels:        perm = 1: E = tile, LD = padded K extent, TS = 6*E*LD,
//                    col = the MMA column permutation (the tile is the smem image
//                    of the mma.sync B operand, so one bulk copy moves it).
// TC kernel:         perm = 2: the tile is the tcgen05 K-major SWIZZLE_NONE
//                    canonical image of the B operand: column col = 6e + c, node n
//                    in core matrix (col/8, n/4) of 8 rows x 4 words:
//                    ((col/8)*(LD/4) + n/4)*32 + (col%8)*4 + n%4.
// FFMA kernel:       perm = 3: elements fastest, (c*LD + n)*E + e (col = c*E + e), so a
//                    warp's lanes (consecutive elements) read and write consecutive words.
// TC kernel:         perm = 4: node-major tiles, n*(nc*E) + nc*e + c (col = nc*e + c): one
//                    row of the tcgen05 accumulator per (element, component), so the
//                    epilogue's lanes (consecutive rows) touch consecutive words, and a
//                    node octet of a tile is one contiguous bulk copy.
// Padding (rows n >= Np, absent elements) is zero in every layout.
struct TileLayout {
  int nc = 6;  // fields per element (6 Maxwell; 4 acoustics, perm 0 only)
  int E = 1;
  int LD = 0;
  int perm = 0;
  int64_t TS = 0;
  DG_HD int col(int e, int c) const {
    return perm == 1 ? 4 * nc * (e >> 2) + 8 * (c >> 1) + 2 * (e & 3) + (c & 1) : perm == 3 ? c * E + e : nc * e + c;
  }
  DG_HD int coff(int c) const { return perm == 1 ? 8 * (c >> 1) + (c & 1) : c; }  // perm 0/1: col(e,c) - col(e,0)
  // perm 0/1/3: word offset of component c relative to component 0 of the same (element, node)
  DG_HD int64_t cofs(int c) const {
    return perm == 3 ? int64_t(c) * LD * E : perm == 4 ? int64_t(c) : int64_t(coff(c)) * LD;
  }
  DG_HD int64_t inner(int cl, int n) const {  // word offset of (column, node) inside a tile
    return perm == 2   ? int64_t(((cl >> 3) * (LD >> 2) + (n >> 2)) * 32 + (cl & 7) * 4 + (n & 3))
           : perm == 3 ? (int64_t(cl / E) * LD + n) * E + cl % E
           : perm == 4 ? int64_t(n) * (nc * E) + cl
                       : int64_t(cl) * LD + n;
  }
  DG_HD int64_t off(int64_t k, int c, int n) const { return (k / E) * TS + inner(col(int(k % E), c), n); }
  DG_HD int64_t ntiles(int64_t K) const { return (K + E - 1) / E; }
  // gather-index encoding: perm 0/1/3 store off(k2, 0, n2) (+ cofs(c) per component);
  // perm 2 stores (k2 << 8) | n2 and the kernel evaluates off() per component.
  // Ghost records are ghost_base + rec (perm 0/1/3) or GHOST_FLAG | rec (perm 2).
  // -1 is a PEC wall.  Word offsets therefore reach 2^31 - 1 (17 GB of FP64 state per rank).
  static constexpr int32_t GHOST_FLAG = int32_t(1) << 30;
  // TC kernel (perm 4) per-face connectivity: a ghost record rec is stored as -2 - rec (-1 is a PEC
  // wall), so the word offsets of local neighbours keep the full int32 range (a flag bit would cut
  // it to 2^30 words: C4 at N = 9 FP32 holds 1.39e9 words per state copy)
  static DG_HD int32_t ghost_code(int64_t rec) { return int32_t(-2 - rec); }
  static DG_HD int32_t ghost_rec(int32_t code) { return -2 - code; }
  // tiled layouts (perm >= 1): a face whose neighbour sits in the SAME tile is encoded as the
  // negative code intra(e2, n2) = -2 - ((e2 << 8) | n2) — the kernel reads u+ from the tile
  // already in shared memory instead of gathering it (the paper's flux-gather granularity,
  // PAPER.md:720-743).
  static DG_HD int32_t intra(int e2, int n2) { return -2 - ((e2 << 8) | n2); }
  static DG_HD bool is_intra(int32_t gi) { return gi < -1; }
  static DG_HD int intra_e(int32_t gi) { return (-2 - gi) >> 8; }
  static DG_HD int intra_n(int32_t gi) { return (-2 - gi) & 255; }
};

template <typename T>
struct StageParams {
  const T* u_in;       // current stage fields
  T* u_out;            // LSERK: next stage fields (ping-pong); RHS mode: unused
  T* res;              // LSERK residual (in place)
  T* rhs_out;          // RHS mode: d_t u in device layout
  const T* geo;
  const int32_t* gidx;  // TC kernel (perm 4): per-tile face connectivity [tile][TC_CONNT] instead (above)
  const int16_t* ftab;  // TC kernel: Fmask [4Nfp] | neighbour node [24][Nfp] | ghost position [6][Nfp]
  const T* ops;
  const T* ops_pad;    // MMA variant: Dr|Ds|Dt as [3][M8][KV] + LIFT [M8][4Nfp], zero-padded
  const int16_t* fmask;
  int64_t K;           // number of elements processed by this launch
  int64_t k_begin;     // first element (launches may cover a sub-range)
  int64_t ES;          // element stride (words)
  int64_t ghost_base;  // offset of the ghost-trace region
  T rk_a, rk_b, dt, alpha;
  int first_stage;     // 1: a_s == 0, do not read res
  int sm_reserve;      // persistent kernels leave this many SMs free (for the concurrent trace exchange)
  // multi-rank stages: the launch's tiles [0, bsig_tiles) hold the partition-boundary
  // elements; the store warps add the number of those tiles to *bsig once they are written (nullptr: off)
  unsigned* bsig;
  int64_t bsig_tiles;
  int system;          // dg_system: 0 Maxwell, 1 acoustics (BASIC kernel)
};

// Launchers, one per (order, precision), defined in stage_N*.cu.
// mode 0: RHS only (writes rhs_out); mode 1: fused lift + LSERK update.
template <typename T>
using StageLauncher = void (*)(const StageParams<T>&, int mode, int variant, void* stream);

StageLauncher<double> stage_launcher_f64(int N);
TileLayout ws_layout_f64(int N);   // tiled layout of the FP64 WS kernel for order N
TileLayout ws32_layout_f32(int N); // tiled layout of the FP32 (3xTF32) WS kernel
size_t ws32_ops_count(int N);      // floats in its split hi/lo operator buffer
void ws32_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* LIFT, float* out);
TileLayout tc_layout_f32(int N, int nc);  // tcgen05 (TC) kernel layout (nc = 6 Maxwell, 4 acoustics)
TileLayout ffma_layout_f32(int N); // FFMA kernel layout (perm 3)
size_t ffma_ops_count(int N);      // floats in its transposed operator buffer
void ffma_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* LIFT, float* out);
TileLayout ffma_layout_f64(int N); // FP64 (DFMA) instance of the FFMA kernel
size_t ffma64_ops_count(int N);
void ffma64_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* LIFT, double* out);
size_t tc_ops_count(int N);
void tc_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* LIFT, float* out);
StageLauncher<float> stage_launcher_f32(int N);

}  // namespace dg
