// C-ABI implementation of libdg (see include/dg.h for the contract).
#include <cuda.h>  // CUstream / CUdeviceptr of the stream memory operations (entry points resolved at run time)
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dg.h"
#include "host/mesh.h"
#include "host/partition.h"
#include "host/refelem.h"
#include "kernels/stage_params.h"

namespace dg {
template <typename S, typename T>
void cm_to_tiles(const S* src, T* dst, int64_t K, int Np, const TileLayout& L, void* st);
template <typename T, typename D>
void tiles_to_cm(const T* src, D* dst, int64_t K, int Np, const TileLayout& L, void* st);
template <typename T>
void pack_traces(const T* u, T* buf, const int32_t* sidx, int64_t nfaces, int Nfp, const TileLayout& L, void* st);
template <typename T>
void poison_padding(T* buf, int64_t K, int Np, const TileLayout& L, void* st);
template <typename T>
void check_padding(const T* buf, int64_t K, int Np, const TileLayout& L, unsigned long long* counts, void* st);
}  // namespace dg

namespace {

thread_local std::string g_err;

dg_status fail(dg_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

// ---------------------------------------------------------------- NCCL (dlopen)
// NCCL is loaded lazily and only for nranks > 1; its types are re-declared
// here (ABI-stable across 2.x) so the library has no link-time NCCL dependency.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat32_ = 7, ncclFloat64_ = 8 };
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { a.err = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return a; }
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.Send = (decltype(a.Send))dlsym(h, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(h, "ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart && a.GroupEnd;
    if (!a.ok) a.err = "libnccl is missing required symbols";
    return a;
  }();
  return api;
}

// SMs a multi-rank stage launch leaves to the concurrent pack + NCCL send/recv kernels of the
// trace exchange (one channel per peer direction on a slab partition; RCB has up to 3 peers per
// cut level).  Nothing waits for them inside a kernel: without free SMs they would only start later.
constexpr int kNcclSmReserve = 4;

// Stream memory operations (driver API, resolved through the runtime so libdg needs no -lcuda):
// the comm stream waits for the stage kernel's boundary-tile counter (kernels/stage_ws.cuh
// signal_boundary) and resets it.  A front-end wait: no SM is held, no kernel spins.
struct MemOps {
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  bool ok = false;
};
MemOps& memops() {
  static MemOps m = [] {
    MemOps a;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      a.wait32 = reinterpret_cast<decltype(a.wait32)>(f);
    f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      a.write32 = reinterpret_cast<decltype(a.write32)>(f);
    a.ok = a.wait32 && a.write32;
    return a;
  }();
  return m;
}

// LSERK4 coefficients: Carpenter & Kennedy (5,4), as tabulated in HW (reading R5)
const double kRkA[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                        -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kRkB[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                        1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                        2277821191437.0 / 14882151754819.0};

}  // namespace

struct dg_solver {
  dg_config cfg{};
  int N = 0, Np = 0, Nfp = 0;
  int nc = 6;  // fields per element (dg_system)
  bool host_only = false;
  bool fp64 = true;
  size_t wsize = 8;
  dg::RefElem ref;
  dg::MeshData mesh;
  dg::Partition part;
  bool has_mesh = false, has_fields = false;
  // device
  int64_t ES = 0, ghost_base = 0, ghost_words = 0, Kl = 0, ntiles = 0;
  dg::TileLayout lay;          // device field layout (depends on precision/variant)
  void* d_u[2] = {nullptr, nullptr};
  void* d_res = nullptr;
  void* d_scratch = nullptr;   // [Kl][ES] (solver precision)
  double* d_stage64 = nullptr; // [nc][Kl][Np] FP64 host-layout staging
  void* d_geo = nullptr;
  int32_t* d_gidx = nullptr;
  int16_t* d_ftab = nullptr;   // TC kernel: Fmask + orientation tables (d_gidx holds the per-face connectivity)
  void* d_ops = nullptr;
  void* d_ops_pad = nullptr;   // FP64 MMA variant operators, zero-padded
  int16_t* d_fmask = nullptr;
  void* d_send = nullptr;      // [n_ghost][nc][Nfp]
  int32_t* d_sidx = nullptr;   // [n_ghost][Nfp] element-node offsets for packing
  cudaStream_t stream = nullptr, comm = nullptr;
  // pipelined host I/O (dg_fields_upload_async / dg_fields_download_async): copy streams,
  // double-buffered FP64 staging, and the events that order them with the compute stream
  cudaStream_t h2d = nullptr, d2h = nullptr;
  double* d_in[2] = {nullptr, nullptr};
  double* d_out[2] = {nullptr, nullptr};
  cudaEvent_t ev_in_ready[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_free[2] = {};
  int in_idx = 0, out_idx = 0;
  bool own_stream = false;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_copied = nullptr;  // loopback transport
  cudaEvent_t ev_done = nullptr;  // stage kernel complete (variants without the boundary signal)
  // boundary-first multi-rank stages: boundary tiles [0, nbt) of the local order;
  // d_bsig counts the boundary tiles a stage has written; ghosts_valid: the ghost region of
  // d_u[cur] holds the current partition-face traces (false after a field upload)
  unsigned* d_bsig = nullptr;
  int64_t nbt = 0;
  bool ghosts_valid = false;
  bool loopback = false;  // nranks > 1 without NCCL: stepped only by dg_group_lserk_step
  ncclComm_t ncomm = nullptr;
  int cur = 0;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  double graph_dt[2] = {0, 0};
  int variant = DG_VARIANT_AUTO;
};

namespace {

dg_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) return fail(DG_ERR_OOM, std::string(what) + ": out of device memory");
  return fail(DG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

void free_dev(void*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

void release_device(dg_solver* s) {
  for (int i = 0; i < 2; ++i) {
    if (s->graph[i]) cudaGraphExecDestroy(s->graph[i]);
    s->graph[i] = nullptr;
    free_dev(s->d_u[i]);
  }
  free_dev(s->d_res);
  free_dev(s->d_scratch);
  void* p = s->d_stage64; free_dev(p); s->d_stage64 = nullptr;
  free_dev(s->d_geo);
  p = s->d_gidx; free_dev(p); s->d_gidx = nullptr;
  p = s->d_ftab; free_dev(p); s->d_ftab = nullptr;
  free_dev(s->d_ops);
  free_dev(s->d_ops_pad);
  p = s->d_fmask; free_dev(p); s->d_fmask = nullptr;
  free_dev(s->d_send);
  p = s->d_bsig; free_dev(p); s->d_bsig = nullptr;
  s->nbt = 0;
  s->ghosts_valid = false;
  p = s->d_sidx; free_dev(p); s->d_sidx = nullptr;
  for (int i = 0; i < 2; ++i) {
    p = s->d_in[i]; free_dev(p); s->d_in[i] = nullptr;
    p = s->d_out[i]; free_dev(p); s->d_out[i] = nullptr;
  }
}



// DG_VARIANT_AUTO: the measured-best kernel per (precision, order) on the bench
// config (NEXT-4 sweep, tools/variant_sweep.py, profiles/r2_final/variant_sweep.jsonl): FP64 ->
// FFMA (register-tiled DFMA) at N = 1, MMA_WS (DMMA) otherwise; FP32 -> FFMA (register-tiled
// SIMT) at N = 1, 2, 3, TC (tcgen05 kind::tf32 3xTF32, TMEM operands) at N >= 4.  N = 3 is a tie on
// C2 (TC 0.137-0.142 / FFMA 0.138 ms) and FFMA on the HBM-resident C4 mesh (4.96 vs 5.61 ms).
int auto_variant(bool fp64, int N) {
  if (fp64) return N == 1 ? DG_VARIANT_FFMA : DG_VARIANT_MMA_WS;
  return N <= 3 ? DG_VARIANT_FFMA : DG_VARIANT_TC;
}

// acoustics (measured on C2, profiles/r2_acoustics_sweep.jsonl): FP64 -> DFMA (FFMA kernel) at N = 1,
// DMMA (MMA_WS) above; FP32 -> FFMA below N = 4, tcgen05 (TC) above
int auto_variant_acoustics(bool fp64, int N) {
  if (fp64) return N == 1 ? DG_VARIANT_FFMA : DG_VARIANT_MMA_WS;
  return N <= 3 ? DG_VARIANT_FFMA : DG_VARIANT_TC;
}

dg_status need_device(dg_solver* s) {
  if (!s) return fail(DG_ERR_ARG, "null solver");
  if (s->host_only) return fail(DG_ERR_STATE, "compute call on a host-only solver (device = -1)");
  cudaError_t e = cudaSetDevice(s->cfg.device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  return DG_OK;
}

template <typename T>
dg::StageParams<T> base_params(dg_solver* s) {
  dg::StageParams<T> p{};
  p.geo = static_cast<const T*>(s->d_geo);
  p.gidx = s->d_gidx;
  p.ftab = s->d_ftab;
  p.ops = static_cast<const T*>(s->d_ops);
  p.ops_pad = static_cast<const T*>(s->d_ops_pad);
  p.fmask = s->d_fmask;
  p.ES = s->ES;
  p.ghost_base = s->ghost_base;
  p.alpha = T(s->cfg.alpha);
  p.system = s->cfg.system;
  p.K = s->Kl;
  p.k_begin = 0;
  return p;
}

template <typename T>
void launch_stage(dg_solver* s, dg::StageParams<T> p, int mode, int64_t k0, int64_t k1, cudaStream_t st) {
  dg::StageLauncher<T> L;
  if constexpr (sizeof(T) == 8)
    L = dg::stage_launcher_f64(s->N);
  else
    L = dg::stage_launcher_f32(s->N);
  p.k_begin = k0;
  p.K = k1 - k0;
  L(p, mode, s->variant, st);
}

// Send/receive the packed partition-face traces (multi-rank NCCL path): grouped
// ncclSend/ncclRecv per peer on the comm stream, received straight into u's ghost region.
template <typename T>
dg_status nccl_exchange(dg_solver* s, T* u) {
  const auto& P = s->part;
  NcclApi& n = nccl();
  const size_t rec = size_t(s->nc) * s->Nfp;
  const int dtype = sizeof(T) == 8 ? ncclFloat64_ : ncclFloat32_;
  if (n.GroupStart() != 0) return fail(DG_ERR_NCCL, "ncclGroupStart failed");
  for (const auto& pp : P.peers) {
    T* sb = static_cast<T*>(s->d_send) + pp.send_off * rec;
    T* rb = u + s->ghost_base + pp.recv_off * rec;
    ncclResult_t r1 = n.Send(sb, pp.nfaces * rec, dtype, pp.rank, s->ncomm, s->comm);
    ncclResult_t r2 = n.Recv(rb, pp.nfaces * rec, dtype, pp.rank, s->ncomm, s->comm);
    if (r1 != 0 || r2 != 0) { n.GroupEnd(); return fail(DG_ERR_NCCL, "ncclSend/ncclRecv failed"); }
  }
  if (n.GroupEnd() != 0) return fail(DG_ERR_NCCL, "ncclGroupEnd failed");
  return DG_OK;
}

// Whether the solver's stage kernel signals its boundary tiles (kernels/stage_ws.cuh
// signal_boundary): the warp-specialized kernels do; BASIC and MMA do not, and for them the
// exchange starts after the whole stage kernel.
bool signals_boundary(const dg_solver* s) {
  return memops().ok && (s->variant == DG_VARIANT_MMA_WS || s->variant == DG_VARIANT_TC || s->variant == DG_VARIANT_FFMA);
}

// Blocking-order exchange of u's traces before the next launch (priming after a field upload,
// and the RHS path): fork -> pack + send/recv on the comm stream -> join.
template <typename T>
dg_status exchange_now(dg_solver* s, T* u) {
  CK(cudaEventRecord(s->ev_fork, s->stream));
  CK(cudaStreamWaitEvent(s->comm, s->ev_fork, 0));
  dg::pack_traces<T>(u, static_cast<T*>(s->d_send), s->d_sidx, s->part.n_ghost_faces, s->Nfp, s->lay, s->comm);
  dg_status st = nccl_exchange<T>(s, u);
  if (st != DG_OK) return st;
  CK(cudaEventRecord(s->ev_join, s->comm));
  CK(cudaStreamWaitEvent(s->stream, s->ev_join, 0));
  return DG_OK;
}

// The comm-stream side of a boundary-first stage, up to the pack of u_out: wait until the
// stage kernel has written its boundary tiles (counter = nbt; the counter is then reset for
// the next stage), or — for kernels without the signal — until it completed.
dg_status await_boundary(dg_solver* s) {
  if (signals_boundary(s)) {
    MemOps& mo = memops();
    const CUdeviceptr sig = CUdeviceptr(reinterpret_cast<uintptr_t>(s->d_bsig));
    if (mo.wait32(CUstream(s->comm), sig, cuuint32_t(s->nbt), CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS ||
        mo.write32(CUstream(s->comm), sig, 0u, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(DG_ERR_CUDA, "cuStreamWaitValue32 / cuStreamWriteValue32 failed");
  } else {
    CK(cudaStreamWaitEvent(s->comm, s->ev_done, 0));
  }
  return DG_OK;
}

// One LSERK stage: u[cur] -> u[cur^1], as ONE launch over all local tiles (boundary tiles
// first).  Multi-rank: the ghost region of u[cur] is already valid (previous stage's
// exchange, or exchange_now); while the interior tiles run, the comm stream packs the
// boundary elements' u_out and exchanges them into u[cur^1]'s ghost region for the next
// stage, which waits for it (ev_join).  DESIGN.md §10.
template <typename T>
dg_status enqueue_stage(dg_solver* s, int stage, double dt, int cur) {
  dg::StageParams<T> p = base_params<T>(s);
  T* uin = static_cast<T*>(s->d_u[cur]);
  T* uout = static_cast<T*>(s->d_u[cur ^ 1]);
  p.u_in = uin;
  p.u_out = uout;
  p.res = static_cast<T*>(s->d_res);
  p.rk_a = T(kRkA[stage]);
  p.rk_b = T(kRkB[stage]);
  p.dt = T(dt);
  p.first_stage = stage == 0 ? 1 : 0;
  if (s->part.n_ghost_faces == 0) {
    launch_stage<T>(s, p, 1, 0, s->Kl, s->stream);
    CK(cudaGetLastError());
    return DG_OK;
  }
  CK(cudaEventRecord(s->ev_fork, s->stream));  // before the launch: the comm branch runs beside it
  p.sm_reserve = kNcclSmReserve;
  if (signals_boundary(s)) {
    p.bsig = s->d_bsig;
    p.bsig_tiles = s->nbt;
  }
  launch_stage<T>(s, p, 1, 0, s->Kl, s->stream);
  CK(cudaGetLastError());
  if (!signals_boundary(s)) CK(cudaEventRecord(s->ev_done, s->stream));
  CK(cudaStreamWaitEvent(s->comm, s->ev_fork, 0));
  dg_status st = await_boundary(s);
  if (st != DG_OK) return st;
  dg::pack_traces<T>(uout, static_cast<T*>(s->d_send), s->d_sidx, s->part.n_ghost_faces, s->Nfp, s->lay, s->comm);
  st = nccl_exchange<T>(s, uout);
  if (st != DG_OK) return st;
  CK(cudaEventRecord(s->ev_join, s->comm));
  CK(cudaStreamWaitEvent(s->stream, s->ev_join, 0));
  return DG_OK;
}

template <typename T>
dg::StageParams<T> stage_params(dg_solver* s, int stage, double dt, int cur) {
  dg::StageParams<T> p = base_params<T>(s);
  p.u_in = static_cast<T*>(s->d_u[cur]);
  p.u_out = static_cast<T*>(s->d_u[cur ^ 1]);
  p.res = static_cast<T*>(s->d_res);
  p.rk_a = T(kRkA[stage]);
  p.rk_b = T(kRkB[stage]);
  p.dt = T(dt);
  p.first_stage = stage == 0 ? 1 : 0;
  return p;
}

// Loopback transport: the exchange of a group of same-process solvers that partition one mesh.
// Identical to the NCCL path except that each partition's ghost records are copied
// device-to-device from its peers' send buffers.  The packs read u[src] (after `ready`: the
// previous stage kernel's boundary signal, or — priming — nothing further) and the copies
// write the ghost regions of u[src].
template <typename T>
dg_status group_exchange(dg_solver* const* g, int n, int src, bool after_stage) {
  const size_t rec = size_t(g[0]->nc) * g[0]->Nfp;
  for (int i = 0; i < n; ++i) {  // pack (after my boundary tiles, after peers finished reading my send buffer)
    dg_solver* s = g[i];
    if (s->part.n_ghost_faces == 0) continue;
    if (!after_stage) {
      CK(cudaEventRecord(s->ev_fork, s->stream));
      CK(cudaStreamWaitEvent(s->comm, s->ev_fork, 0));
    } else {
      dg_status st = await_boundary(s);
      if (st != DG_OK) return st;
    }
    for (const auto& pp : s->part.peers) CK(cudaStreamWaitEvent(s->comm, g[pp.rank]->ev_copied, 0));
    dg::pack_traces<T>(static_cast<T*>(s->d_u[src]), static_cast<T*>(s->d_send), s->d_sidx, s->part.n_ghost_faces,
                       s->Nfp, s->lay, s->comm);
    CK(cudaEventRecord(s->ev_packed, s->comm));
  }
  for (int q = 0; q < n; ++q) {  // receive: copy peers' records into my ghost region
    dg_solver* s = g[q];
    if (s->part.n_ghost_faces == 0) continue;
    for (const auto& pp : s->part.peers) {
      dg_solver* r = g[pp.rank];
      const dg::PeerPlan* back = nullptr;
      for (const auto& rp : r->part.peers)
        if (rp.rank == q) back = &rp;
      if (!back || back->nfaces != pp.nfaces) return fail(DG_ERR_STATE, "inconsistent partition plans in group");
      CK(cudaStreamWaitEvent(s->comm, r->ev_packed, 0));
      T* dst = static_cast<T*>(s->d_u[src]) + s->ghost_base + pp.recv_off * rec;
      const T* srcp = static_cast<const T*>(r->d_send) + back->send_off * rec;
      CK(cudaMemcpyAsync(dst, srcp, pp.nfaces * rec * sizeof(T), cudaMemcpyDeviceToDevice, s->comm));
    }
    CK(cudaEventRecord(s->ev_copied, s->comm));
    CK(cudaEventRecord(s->ev_join, s->comm));
  }
  if (!after_stage)
    for (int q = 0; q < n; ++q)
      if (g[q]->part.n_ghost_faces > 0) CK(cudaStreamWaitEvent(g[q]->stream, g[q]->ev_join, 0));
  return DG_OK;
}

// One LSERK stage of a loopback group: every partition's stage kernel (one launch, boundary
// tiles first), then the exchange of the boundary traces of u[cur^1] beside the interior tiles.
template <typename T>
dg_status group_stage(dg_solver* const* g, int n, int stage, double dt, int cur) {
  for (int i = 0; i < n; ++i) {
    dg_solver* s = g[i];
    dg::StageParams<T> p = stage_params<T>(s, stage, dt, cur);
    if (s->part.n_ghost_faces > 0) {
      CK(cudaEventRecord(s->ev_fork, s->stream));
      p.sm_reserve = kNcclSmReserve;  // the pack kernel runs beside the interior tiles
      if (signals_boundary(s)) {
        p.bsig = s->d_bsig;
        p.bsig_tiles = s->nbt;
      }
    }
    launch_stage<T>(s, p, 1, 0, s->Kl, s->stream);
    CK(cudaGetLastError());
    if (s->part.n_ghost_faces > 0) {
      if (!signals_boundary(s)) CK(cudaEventRecord(s->ev_done, s->stream));
      CK(cudaStreamWaitEvent(s->comm, s->ev_fork, 0));
    }
  }
  dg_status st = group_exchange<T>(g, n, cur ^ 1, true);
  if (st != DG_OK) return st;
  for (int q = 0; q < n; ++q)
    if (g[q]->part.n_ghost_faces > 0) CK(cudaStreamWaitEvent(g[q]->stream, g[q]->ev_join, 0));
  return DG_OK;
}

template <typename T>
dg_status enqueue_rhs(dg_solver* s, T* out_tiles) {
  dg::StageParams<T> p = base_params<T>(s);
  T* uin = static_cast<T*>(s->d_u[s->cur]);
  p.u_in = uin;
  p.rhs_out = out_tiles;
  if (s->part.n_ghost_faces > 0 && !s->ghosts_valid) {
    dg_status st = exchange_now<T>(s, uin);
    if (st != DG_OK) return st;
    s->ghosts_valid = true;
  }
  launch_stage<T>(s, p, 0, 0, s->Kl, s->stream);
  CK(cudaGetLastError());
  return DG_OK;
}

template <typename T>
dg_status upload_setup(dg_solver* s) {
  const auto& m = s->mesh;
  const auto& P = s->part;
  const int Np = s->Np, Nfp = s->Nfp, NF = 4 * Nfp;
  const int64_t Kl = P.K_local;
  s->Kl = Kl;
  const bool ws = s->variant == DG_VARIANT_AUTO || s->variant == DG_VARIANT_MMA_WS;
  const bool tc = sizeof(T) == 4 && s->variant == DG_VARIANT_TC;
  const bool ff = s->variant == DG_VARIANT_FFMA;  // (AUTO resolved at create)
  if (ff) {
    s->lay = sizeof(T) == 8 ? dg::ffma_layout_f64(s->N) : dg::ffma_layout_f32(s->N);
    s->lay.nc = s->nc;  // acoustics: 4 fields per element (FfCfg<T, N, NC>::TS)
    s->lay.TS = int64_t(s->nc) * s->lay.LD * s->lay.E;
  } else if (sizeof(T) == 8 && ws) {
    s->lay = dg::ws_layout_f64(s->N);
    s->lay.nc = s->nc;  // acoustics: 4-element column groups of 4 x 4 columns (WsCfg<N, 4>::TS)
    s->lay.TS = int64_t(s->nc) * s->lay.E * s->lay.LD;
  } else if (sizeof(T) == 4 && ws) {
    s->lay = dg::ws32_layout_f32(s->N);
  } else if (tc) {
    s->lay = dg::tc_layout_f32(s->N, s->nc);
  } else {
    s->lay = dg::TileLayout();
    s->lay.nc = s->nc;
    s->lay.E = 1;
    s->lay.LD = Np;
    s->lay.perm = 0;
    s->lay.TS = sizeof(T) == 8 ? s->nc * Np : ((s->nc * Np + 3) / 4) * 4;
  }
  s->ES = s->lay.TS;
  s->ntiles = s->lay.ntiles(Kl);
  const int64_t twords = s->ntiles * s->lay.TS;
  s->ghost_base = twords;
  s->ghost_words = P.n_ghost_faces * s->nc * Nfp;
  const int64_t uwords = s->ghost_base + s->ghost_words;
  if (uwords >= (int64_t(1) << 31))
    return fail(DG_ERR_ARG, "local problem too large for 32-bit gather indices on one rank (partition further)");
  const size_t wb = sizeof(T);
  for (int i = 0; i < 2; ++i) {
    CK(cudaMalloc(&s->d_u[i], std::max<int64_t>(uwords, 1) * wb));
    CK(cudaMemsetAsync(s->d_u[i], 0, std::max<int64_t>(uwords, 1) * wb, s->stream));
  }
  CK(cudaMalloc(&s->d_res, std::max<int64_t>(twords, 1) * wb));
  CK(cudaMemsetAsync(s->d_res, 0, std::max<int64_t>(twords, 1) * wb, s->stream));
  CK(cudaMalloc(&s->d_scratch, std::max<int64_t>(twords, 1) * wb));
  CK(cudaMemsetAsync(s->d_scratch, 0, std::max<int64_t>(twords, 1) * wb, s->stream));
  CK(cudaMalloc((void**)&s->d_stage64, std::max<int64_t>(s->nc * Kl * Np, 1) * sizeof(double)));
  // geometry [Kpad][GEO_W] (padding elements zero); TC kernel (perm 4): per tile [E][GEO_W]
  // padded to tc_geot(E) words, so one tile's record is one 16-B aligned bulk copy
  const bool tcl = s->lay.perm == 4;
  const int64_t gstride = tcl ? dg::tc_geot(s->lay.E) : s->lay.E * dg::GEO_W;
  std::vector<T> geo(size_t(std::max<int64_t>(s->ntiles * gstride, 1)), T(0));
  for (int64_t l = 0; l < Kl; ++l) {
    const int64_t k = P.local_ids[l];
    const int64_t g0 = (l / s->lay.E) * gstride + (l % s->lay.E) * dg::GEO_W;
    for (int i = 0; i < 9; ++i) geo[g0 + i] = T(m.rst_x[9 * k + i]);
    for (int i = 0; i < 16; ++i) geo[g0 + 9 + i] = T(m.nrm[16 * k + i]);
  }
  CK(cudaMalloc(&s->d_geo, geo.size() * wb));
  CK(cudaMemcpy(s->d_geo, geo.data(), geo.size() * wb, cudaMemcpyHostToDevice));
  std::vector<int32_t> gidx;
  if (tcl) {
    // TC kernel: per-face (neighbour base, f2*6 + orientation) + smem tables, 20 B per element,
    // packed per tile as [E][4] bases | [E] x 4 codes (u8) | pad to TC_CONNT words
    std::vector<int32_t> fbase;
    std::vector<uint8_t> fcode;
    std::vector<int16_t> ftab;
    dg::build_face_connectivity(s->ref, m, P, s->lay, fbase, fcode, ftab);
    const int E = s->lay.E;
    gidx.assign(size_t(s->ntiles) * dg::TC_CONNT, 0);
    for (int64_t t = 0; t < s->ntiles; ++t)
      for (int e = 0; e < E; ++e) {
        uint32_t codes = 0;
        for (int f = 0; f < 4; ++f) {
          gidx[t * dg::TC_CONNT + 4 * e + f] = fbase[(t * E + e) * 4 + f];
          codes |= uint32_t(fcode[(t * E + e) * 4 + f]) << (8 * f);
        }
        gidx[t * dg::TC_CONNT + 4 * E + e] = int32_t(codes);
      }
    CK(cudaMalloc((void**)&s->d_ftab, ftab.size() * sizeof(int16_t)));
    CK(cudaMemcpy(s->d_ftab, ftab.data(), ftab.size() * sizeof(int16_t), cudaMemcpyHostToDevice));
  } else {
    dg::build_gather_index(s->ref, m, P, s->lay, s->ghost_base, gidx);
  }
  if (gidx.empty()) gidx.push_back(-1);
  CK(cudaMalloc((void**)&s->d_gidx, gidx.size() * sizeof(int32_t)));
  CK(cudaMemcpy(s->d_gidx, gidx.data(), gidx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  // operators Dr|Ds|Dt|LIFT
  std::vector<T> ops(size_t(3) * Np * Np + size_t(Np) * NF);
  for (int i = 0; i < Np; ++i)
    for (int j = 0; j < Np; ++j) {
      ops[size_t(i) * Np + j] = T(s->ref.Dr(i, j));
      ops[size_t(Np) * Np + size_t(i) * Np + j] = T(s->ref.Ds(i, j));
      ops[size_t(2) * Np * Np + size_t(i) * Np + j] = T(s->ref.Dt(i, j));
    }
  for (int i = 0; i < Np; ++i)
    for (int j = 0; j < NF; ++j) ops[size_t(3) * Np * Np + size_t(i) * NF + j] = T(s->ref.LIFT(i, j));
  CK(cudaMalloc(&s->d_ops, ops.size() * wb));
  CK(cudaMemcpy(s->d_ops, ops.data(), ops.size() * wb, cudaMemcpyHostToDevice));
  if (sizeof(T) == 8 && s->lay.perm == 3) {
    // FFMA (DFMA) kernel: transposed, row-padded operators (stage_ffma.cuh)
    std::vector<double> pad(dg::ffma64_ops_count(s->N));
    dg::ffma64_ops_build(s->N, s->ref.Dr.a.data(), s->ref.Ds.a.data(), s->ref.Dt.a.data(), s->ref.LIFT.a.data(),
                         pad.data());
    CK(cudaMalloc(&s->d_ops_pad, pad.size() * sizeof(double)));
    CK(cudaMemcpy(s->d_ops_pad, pad.data(), pad.size() * sizeof(double), cudaMemcpyHostToDevice));
  } else if (sizeof(T) == 8) {
    // [3][M8][KV] + [M8][NF], zero padding (stage_mma.cuh)
    const int M8 = (Np + 7) / 8 * 8, KV = (Np + 3) / 4 * 4;
    std::vector<T> pad(size_t(3) * M8 * KV + size_t(M8) * NF, T(0));
    const dg::Mat* D[3] = {&s->ref.Dr, &s->ref.Ds, &s->ref.Dt};
    for (int b = 0; b < 3; ++b)
      for (int i = 0; i < Np; ++i)
        for (int j = 0; j < Np; ++j) pad[(size_t(b) * M8 + i) * KV + j] = T((*D[b])(i, j));
    for (int i = 0; i < Np; ++i)
      for (int j = 0; j < NF; ++j) pad[size_t(3) * M8 * KV + size_t(i) * NF + j] = T(s->ref.LIFT(i, j));
    CK(cudaMalloc(&s->d_ops_pad, pad.size() * wb));
    CK(cudaMemcpy(s->d_ops_pad, pad.data(), pad.size() * wb, cudaMemcpyHostToDevice));
  } else {
    // FP32 3xTF32: hi/lo split operators, zero-padded (stage_ws32.cuh / stage_tc.cuh);
    // FFMA: transposed, row-padded operators (stage_ffma.cuh)
    const bool tcv = s->lay.perm == 4, ffv = s->lay.perm == 3;
    std::vector<float> pad(tcv ? dg::tc_ops_count(s->N) : ffv ? dg::ffma_ops_count(s->N) : dg::ws32_ops_count(s->N));
    if (ffv)
      dg::ffma_ops_build(s->N, s->ref.Dr.a.data(), s->ref.Ds.a.data(), s->ref.Dt.a.data(), s->ref.LIFT.a.data(),
                         pad.data());
    else if (tcv)
      dg::tc_ops_build(s->N, s->ref.Dr.a.data(), s->ref.Ds.a.data(), s->ref.Dt.a.data(), s->ref.LIFT.a.data(),
                       pad.data());
    else
      dg::ws32_ops_build(s->N, s->ref.Dr.a.data(), s->ref.Ds.a.data(), s->ref.Dt.a.data(), s->ref.LIFT.a.data(),
                         pad.data());
    CK(cudaMalloc(&s->d_ops_pad, pad.size() * sizeof(float)));
    CK(cudaMemcpy(s->d_ops_pad, pad.data(), pad.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  std::vector<int16_t> fm(NF);
  for (int i = 0; i < NF; ++i) fm[i] = int16_t(s->ref.Fmask[i]);
  CK(cudaMalloc((void**)&s->d_fmask, NF * sizeof(int16_t)));
  CK(cudaMemcpy(s->d_fmask, fm.data(), NF * sizeof(int16_t), cudaMemcpyHostToDevice));
  if (P.n_ghost_faces > 0) {
    CK(cudaMalloc(&s->d_send, P.n_ghost_faces * s->nc * Nfp * wb));
    CK(cudaMalloc((void**)&s->d_bsig, sizeof(unsigned)));
    CK(cudaMemset(s->d_bsig, 0, sizeof(unsigned)));
    s->nbt = (P.K_boundary + s->lay.E - 1) / s->lay.E;  // tiles holding the boundary elements (local order)
    std::vector<int32_t> sidx(size_t(P.n_ghost_faces) * Nfp);
    for (int64_t g = 0; g < P.n_ghost_faces; ++g)
      for (int j = 0; j < Nfp; ++j)
        sidx[g * Nfp + j] = s->lay.perm == 2
                                ? int32_t((P.send_elem[g] << 8) | s->ref.Fmask[P.send_face[g] * Nfp + j])
                                : int32_t(s->lay.off(P.send_elem[g], 0, s->ref.Fmask[P.send_face[g] * Nfp + j]));
    CK(cudaMalloc((void**)&s->d_sidx, sidx.size() * sizeof(int32_t)));
    CK(cudaMemcpy(s->d_sidx, sidx.data(), sidx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  CK(cudaStreamSynchronize(s->stream));
  return DG_OK;
}

template <typename T>
dg_status capture_step(dg_solver* s, int parity, double dt) {
  if (s->graph[parity]) {
    cudaGraphExecDestroy(s->graph[parity]);
    s->graph[parity] = nullptr;
  }
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  dg_status st = DG_OK;
  int cur = parity;
  for (int stage = 0; stage < 5 && st == DG_OK; ++stage) {
    st = enqueue_stage<T>(s, stage, dt, cur);
    cur ^= 1;
  }
  cudaError_t e = cudaStreamEndCapture(s->stream, &g);
  if (st != DG_OK) { if (g) cudaGraphDestroy(g); return st; }
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&s->graph[parity], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  s->graph_dt[parity] = dt;
  return DG_OK;
}

// DG_GRAPH=0 (environment): enqueue the five stage launches of each step directly instead of
// launching the captured graph (A/B measurement of the step boundary, profiles/r1_graph_ab.jsonl).
static bool graphs_enabled() {
  static const int v = [] {
    const char* e = std::getenv("DG_GRAPH");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

template <typename T>
dg_status lserk_steps(dg_solver* s, double dt, int nsteps) {
  if (nsteps > 0 && s->part.n_ghost_faces > 0 && !s->ghosts_valid) {  // prime: traces of the uploaded fields
    dg_status st = exchange_now<T>(s, static_cast<T*>(s->d_u[s->cur]));
    if (st != DG_OK) return st;
    s->ghosts_valid = true;  // every stage's exchange keeps them valid from here on
  }
  if (!graphs_enabled()) {
    for (int n = 0; n < nsteps; ++n) {
      for (int stage = 0; stage < 5; ++stage) {
        dg_status st = enqueue_stage<T>(s, stage, dt, s->cur);
        if (st != DG_OK) return st;
        s->cur ^= 1;
      }
    }
    return DG_OK;
  }
  for (int n = 0; n < nsteps; ++n) {
    const int par = s->cur;
    if (!s->graph[par] || s->graph_dt[par] != dt) {
      dg_status st = capture_step<T>(s, par, dt);
      if (st != DG_OK) return st;
    }
    CK(cudaGraphLaunch(s->graph[par], s->stream));
    s->cur ^= 1;  // five stages: odd number of ping-pong swaps
  }
  return DG_OK;
}

template <typename T>
dg_status time_stage(dg_solver* s, int reps, double* ms) {
  for (int i = 0; i < reps + 1; ++i) {
    if (i == 1) CK(cudaEventRecord(s->ev_t0, s->stream));
    dg::StageParams<T> p = base_params<T>(s);
    p.u_in = static_cast<T*>(s->d_u[s->cur]);
    p.u_out = static_cast<T*>(s->d_u[s->cur ^ 1]);
    p.res = static_cast<T*>(s->d_res);
    p.rk_a = T(kRkA[1]);
    p.rk_b = T(kRkB[1]);
    p.dt = T(1e-6);
    p.first_stage = 0;
    launch_stage<T>(s, p, 1, 0, s->Kl, s->stream);
  }
  CK(cudaEventRecord(s->ev_t1, s->stream));
  CK(cudaEventSynchronize(s->ev_t1));
  CK(cudaGetLastError());
  float f = 0;
  CK(cudaEventElapsedTime(&f, s->ev_t0, s->ev_t1));
  *ms = double(f) / reps;
  return DG_OK;
}

}  // namespace

#ifdef DG_WS_PROFILE
namespace dg {
#define DG_PDECL(n) void ws_prof_N##n(unsigned long long*, int); void tc_dbg_N##n(float*);
DG_PDECL(1) DG_PDECL(2) DG_PDECL(3) DG_PDECL(4) DG_PDECL(5) DG_PDECL(6) DG_PDECL(7) DG_PDECL(8) DG_PDECL(9)
}  // namespace dg
// profiling builds only (libdg_prof.so): read/reset the WS kernel's cycle counters
extern "C" __attribute__((visibility("default"))) void dg_debug_tc_dump(int N, float* dev) {
  static void (*const t[9])(float*) = {dg::tc_dbg_N1, dg::tc_dbg_N2, dg::tc_dbg_N3, dg::tc_dbg_N4, dg::tc_dbg_N5,
                                       dg::tc_dbg_N6, dg::tc_dbg_N7, dg::tc_dbg_N8, dg::tc_dbg_N9};
  if (N >= 1 && N <= 9) t[N - 1](dev);
}
extern "C" __attribute__((visibility("default"))) void dg_debug_ws_profile(int N, unsigned long long* out, int reset) {
  static void (*const t[9])(unsigned long long*, int) = {dg::ws_prof_N1, dg::ws_prof_N2, dg::ws_prof_N3,
                                                         dg::ws_prof_N4, dg::ws_prof_N5, dg::ws_prof_N6,
                                                         dg::ws_prof_N7, dg::ws_prof_N8, dg::ws_prof_N9};
  if (N >= 1 && N <= 9) t[N - 1](out, reset);
}
#endif

extern "C" {

void dg_config_default(dg_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->order = 3;
  c->precision = 8;
  c->alpha = 1.0;
  c->device = 0;
  c->stream = nullptr;
  c->rank = 0;
  c->nranks = 1;
  c->nccl_id = nullptr;
  c->variant = DG_VARIANT_AUTO;
  c->reorder = 0;
  c->partition = DG_PARTITION_RANGES;
  c->system = DG_SYSTEM_MAXWELL;
}

const char* dg_last_error(void) { return g_err.c_str(); }

const char* dg_version(void) {
  return "dg-b200 abi " "1" " sm_100a (" __DATE__ " " __TIME__ ")";
}

dg_status dg_create(const dg_config* cfg, dg_solver** out) {
  g_err.clear();
  if (!cfg || !out) return fail(DG_ERR_ARG, "null argument");
  *out = nullptr;
  if (cfg->order < 1 || cfg->order > 9) return fail(DG_ERR_ORDER, "order N must be in 1..9");
  if (cfg->precision != 4 && cfg->precision != 8) return fail(DG_ERR_ARG, "precision must be 4 or 8");
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks) return fail(DG_ERR_ARG, "bad rank/nranks");
  if (cfg->variant < 0 || cfg->variant > 6) return fail(DG_ERR_ARG, "bad variant");
  if (cfg->variant == DG_VARIANT_FUSED)
    return fail(DG_ERR_ARG, "DG_VARIANT_FUSED was withdrawn (slower than the per-stage WS launches; DESIGN.md §8)");
  if (cfg->variant == DG_VARIANT_TC && cfg->precision != 4)
    return fail(DG_ERR_ARG, "DG_VARIANT_TC is the FP32 tcgen05 kernel");
  if (cfg->system != DG_SYSTEM_MAXWELL && cfg->system != DG_SYSTEM_ACOUSTICS) return fail(DG_ERR_ARG, "bad system");
  if (cfg->partition != DG_PARTITION_RANGES && cfg->partition != DG_PARTITION_RCB)
    return fail(DG_ERR_ARG, "bad partition method");
  if (cfg->system == DG_SYSTEM_ACOUSTICS && (cfg->variant == DG_VARIANT_MMA ||
                                             (cfg->variant == DG_VARIANT_MMA_WS && cfg->precision != 8)))
    return fail(DG_ERR_ARG, "DG_SYSTEM_ACOUSTICS runs on the BASIC, FFMA, FP64 MMA_WS (DMMA) and FP32 TC kernels");
  std::unique_ptr<dg_solver> s(new dg_solver());
  s->cfg = *cfg;
  s->N = cfg->order;
  s->fp64 = cfg->precision == 8;
  s->wsize = s->fp64 ? 8 : 4;
  s->nc = cfg->system == DG_SYSTEM_ACOUSTICS ? 4 : 6;
  // acoustics (NEXT-3): AUTO -> the measured-best kernel of the SYS = 1 instances
  s->variant = cfg->variant != DG_VARIANT_AUTO        ? cfg->variant
               : cfg->system == DG_SYSTEM_ACOUSTICS ? auto_variant_acoustics(cfg->precision == 8, cfg->order)
                                                    : auto_variant(cfg->precision == 8, cfg->order);
  s->host_only = cfg->device < 0;
  try {
    s->ref = dg::build_ref_elem(s->N);
  } catch (const std::exception& e) {
    return fail(DG_ERR_ORDER, std::string("reference element: ") + e.what());
  }
  s->Np = s->ref.Np;
  s->Nfp = s->ref.Nfp;
  if (!s->host_only) {
    s->loopback = cfg->nranks > 1 && !cfg->nccl_id;  // in-process partitions (dg_group_lserk_step)
    CK(cudaSetDevice(cfg->device));
    if (cfg->stream) {
      s->stream = static_cast<cudaStream_t>(cfg->stream);
    } else {
      CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
      s->own_stream = true;
    }
    CK(cudaStreamCreateWithFlags(&s->comm, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreate(&s->ev_t0));
    CK(cudaEventCreate(&s->ev_t1));
    CK(cudaEventCreateWithFlags(&s->ev_packed, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_copied, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_done, cudaEventDisableTiming));
    if (cfg->nranks > 1 && !s->loopback) {
      NcclApi& n = nccl();
      if (!n.ok) return fail(DG_ERR_NCCL, n.err);
      ncclUniqueId id;
      std::memcpy(&id, cfg->nccl_id, sizeof(id));
      ncclResult_t r = n.CommInitRank(&s->ncomm, cfg->nranks, id, cfg->rank);
      if (r != 0)
        return fail(DG_ERR_NCCL, std::string("ncclCommInitRank: ") + (n.GetErrorString ? n.GetErrorString(r) : "?"));
    }
  }
  *out = s.release();
  return DG_OK;
}

dg_status dg_mesh_upload(dg_solver* s, int64_t nv, const double* VX, int64_t K, const int64_t* EToV,
                         const int32_t* part) {
  g_err.clear();
  if (!s || !VX || !EToV || nv <= 0 || K <= 0) return fail(DG_ERR_ARG, "bad mesh arguments");
  std::string err;
  try {
    err = dg::build_mesh(s->ref, nv, VX, K, EToV, s->mesh);
    if (err.empty())
    if (err.empty() && !part && s->cfg.partition == DG_PARTITION_RCB && s->cfg.nranks > 1) {
      std::vector<int32_t> own;
      dg::rcb_owners(s->mesh, s->cfg.nranks, own);
      err = dg::build_partition(s->mesh, s->cfg.rank, s->cfg.nranks, own.data(), s->part, s->cfg.reorder != 0);
    } else if (err.empty()) {
      err = dg::build_partition(s->mesh, s->cfg.rank, s->cfg.nranks, part, s->part, s->cfg.reorder != 0);
    }
  } catch (const std::exception& e) {
    err = e.what();
  }
  if (!err.empty()) {
    s->has_mesh = false;
    return fail(DG_ERR_MESH, err);
  }
  s->has_mesh = true;
  s->has_fields = false;
  s->Kl = s->part.K_local;
  if (s->host_only) return DG_OK;
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  CK(cudaStreamSynchronize(s->stream));
  if (s->h2d) CK(cudaStreamSynchronize(s->h2d));  // staging buffers may still be in use
  if (s->d2h) CK(cudaStreamSynchronize(s->d2h));
  release_device(s);
  s->cur = 0;
  return s->fp64 ? upload_setup<double>(s) : upload_setup<float>(s);
}

dg_status dg_local_elements(dg_solver* s, int64_t* K_local, int64_t* ids) {
  if (!s) return fail(DG_ERR_ARG, "null solver");
  if (!s->has_mesh) return fail(DG_ERR_STATE, "no mesh uploaded");
  if (K_local) *K_local = s->part.K_local;
  if (ids) std::memcpy(ids, s->part.local_ids.data(), s->part.K_local * sizeof(int64_t));
  return DG_OK;
}

dg_status dg_get_sizes(dg_solver* s, int32_t* Np, int32_t* Nfp, int64_t* K_local, int64_t* K_global) {
  if (!s) return fail(DG_ERR_ARG, "null solver");
  if (Np) *Np = s->Np;
  if (Nfp) *Nfp = s->Nfp;
  if (K_local) *K_local = s->has_mesh ? s->part.K_local : 0;
  if (K_global) *K_global = s->has_mesh ? s->mesh.K : 0;
  return DG_OK;
}

static dg_status upload_common(dg_solver* s, const void* src, bool from_host) {
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!s->has_mesh) return fail(DG_ERR_STATE, "no mesh uploaded");
  if (!src) return fail(DG_ERR_ARG, "null field pointer");
  const int64_t n = s->nc * s->Kl * s->Np;
  s->cur = 0;
  if (from_host) {
    CK(cudaMemcpyAsync(s->d_stage64, src, n * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    if (s->fp64)
      dg::cm_to_tiles<double, double>(s->d_stage64, static_cast<double*>(s->d_u[0]), s->Kl, s->Np, s->lay, s->stream);
    else
      dg::cm_to_tiles<double, float>(s->d_stage64, static_cast<float*>(s->d_u[0]), s->Kl, s->Np, s->lay, s->stream);
  } else {
    if (s->fp64)
      dg::cm_to_tiles<double, double>(static_cast<const double*>(src), static_cast<double*>(s->d_u[0]), s->Kl,
                                      s->Np, s->lay, s->stream);
    else
      dg::cm_to_tiles<float, float>(static_cast<const float*>(src), static_cast<float*>(s->d_u[0]), s->Kl, s->Np,
                                    s->lay, s->stream);
  }
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(s->d_res, 0, std::max<int64_t>(s->ntiles * s->lay.TS, 1) * s->wsize, s->stream));
  s->ghosts_valid = false;
  if (from_host) CK(cudaStreamSynchronize(s->stream));
  s->has_fields = true;
  return DG_OK;
}

dg_status dg_fields_upload(dg_solver* s, const double* f) { g_err.clear(); return upload_common(s, f, true); }
dg_status dg_fields_upload_device(dg_solver* s, const void* f) { g_err.clear(); return upload_common(s, f, false); }

static dg_status download_common(dg_solver* s, void* dst, bool to_host, bool rhs) {
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (rhs && s->loopback) return fail(DG_ERR_STATE, "loopback partition solver: rhs needs its peers (use one solver)");
  if (!s->has_fields) return fail(DG_ERR_STATE, "no fields uploaded");
  if (!dst) return fail(DG_ERR_ARG, "null output pointer");
  const int64_t n = s->nc * s->Kl * s->Np;
  const void* tiles = s->d_u[s->cur];
  if (rhs) {
    st = s->fp64 ? enqueue_rhs<double>(s, static_cast<double*>(s->d_scratch))
                 : enqueue_rhs<float>(s, static_cast<float*>(s->d_scratch));
    if (st != DG_OK) return st;
    tiles = s->d_scratch;
  }
  if (to_host) {
    if (s->fp64)
      dg::tiles_to_cm<double, double>(static_cast<const double*>(tiles), s->d_stage64, s->Kl, s->Np, s->lay, s->stream);
    else
      dg::tiles_to_cm<float, double>(static_cast<const float*>(tiles), s->d_stage64, s->Kl, s->Np, s->lay, s->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst, s->d_stage64, n * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  } else {
    if (s->fp64)
      dg::tiles_to_cm<double, double>(static_cast<const double*>(tiles), static_cast<double*>(dst), s->Kl, s->Np,
                                      s->lay, s->stream);
    else
      dg::tiles_to_cm<float, float>(static_cast<const float*>(tiles), static_cast<float*>(dst), s->Kl, s->Np, s->lay,
                                    s->stream);
    CK(cudaGetLastError());
  }
  return DG_OK;
}

// lazily create the copy streams / events and the staging buffers of the pipelined I/O
static dg_status io_setup(dg_solver* s) {
  if (!s->h2d) {
    CK(cudaStreamCreateWithFlags(&s->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&s->ev_in_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_in_free[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_out_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_out_free[i], cudaEventDisableTiming));
    }
  }
  const size_t bytes = size_t(std::max<int64_t>(s->nc * s->Kl * s->Np, 1)) * sizeof(double);
  for (int i = 0; i < 2; ++i) {
    if (!s->d_in[i]) CK(cudaMalloc((void**)&s->d_in[i], bytes));
    if (!s->d_out[i]) CK(cudaMalloc((void**)&s->d_out[i], bytes));
  }
  return DG_OK;
}

dg_status dg_fields_upload_async(dg_solver* s, const double* f) {
  g_err.clear();
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!s->has_mesh) return fail(DG_ERR_STATE, "no mesh uploaded");
  if (!f) return fail(DG_ERR_ARG, "null field pointer");
  st = io_setup(s);
  if (st != DG_OK) return st;
  const int i = s->in_idx;
  s->in_idx ^= 1;
  const size_t bytes = size_t(s->nc * s->Kl * s->Np) * sizeof(double);
  CK(cudaStreamWaitEvent(s->h2d, s->ev_in_free[i], 0));  // the conversion that last read d_in[i]
  CK(cudaMemcpyAsync(s->d_in[i], f, bytes, cudaMemcpyHostToDevice, s->h2d));
  CK(cudaEventRecord(s->ev_in_ready[i], s->h2d));
  CK(cudaStreamWaitEvent(s->stream, s->ev_in_ready[i], 0));
  s->cur = 0;
  if (s->fp64)
    dg::cm_to_tiles<double, double>(s->d_in[i], static_cast<double*>(s->d_u[0]), s->Kl, s->Np, s->lay, s->stream);
  else
    dg::cm_to_tiles<double, float>(s->d_in[i], static_cast<float*>(s->d_u[0]), s->Kl, s->Np, s->lay, s->stream);
  CK(cudaGetLastError());
  CK(cudaEventRecord(s->ev_in_free[i], s->stream));
  CK(cudaMemsetAsync(s->d_res, 0, std::max<int64_t>(s->ntiles * s->lay.TS, 1) * s->wsize, s->stream));
  s->ghosts_valid = false;
  s->has_fields = true;
  return DG_OK;
}

dg_status dg_fields_download_async(dg_solver* s, double* f) {
  g_err.clear();
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!s->has_fields) return fail(DG_ERR_STATE, "no fields uploaded");
  if (!f) return fail(DG_ERR_ARG, "null output pointer");
  st = io_setup(s);
  if (st != DG_OK) return st;
  const int o = s->out_idx;
  s->out_idx ^= 1;
  const size_t bytes = size_t(s->nc * s->Kl * s->Np) * sizeof(double);
  CK(cudaStreamWaitEvent(s->stream, s->ev_out_free[o], 0));  // the copy that last read d_out[o]
  if (s->fp64)
    dg::tiles_to_cm<double, double>(static_cast<const double*>(s->d_u[s->cur]), s->d_out[o], s->Kl, s->Np, s->lay,
                                    s->stream);
  else
    dg::tiles_to_cm<float, double>(static_cast<const float*>(s->d_u[s->cur]), s->d_out[o], s->Kl, s->Np, s->lay,
                                   s->stream);
  CK(cudaGetLastError());
  CK(cudaEventRecord(s->ev_out_ready[o], s->stream));
  CK(cudaStreamWaitEvent(s->d2h, s->ev_out_ready[o], 0));
  CK(cudaMemcpyAsync(f, s->d_out[o], bytes, cudaMemcpyDeviceToHost, s->d2h));
  CK(cudaEventRecord(s->ev_out_free[o], s->d2h));
  return DG_OK;
}

dg_status dg_fields_download(dg_solver* s, double* f) { g_err.clear(); return download_common(s, f, true, false); }
dg_status dg_fields_download_device(dg_solver* s, void* f) { g_err.clear(); return download_common(s, f, false, false); }
dg_status dg_rhs(dg_solver* s, double* r) { g_err.clear(); return download_common(s, r, true, true); }
dg_status dg_rhs_device(dg_solver* s, void* r) { g_err.clear(); return download_common(s, r, false, true); }

dg_status dg_lserk_step(dg_solver* s, double dt, int32_t nsteps) {
  g_err.clear();
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!s->has_fields) return fail(DG_ERR_STATE, "no fields uploaded");
  if (nsteps < 0) return fail(DG_ERR_ARG, "nsteps < 0");
  if (s->loopback) return fail(DG_ERR_STATE, "loopback partition solver: step it with dg_group_lserk_step");
  return s->fp64 ? lserk_steps<double>(s, dt, nsteps) : lserk_steps<float>(s, dt, nsteps);
}

dg_status dg_group_lserk_step(dg_solver* const* group, int32_t n, double dt, int32_t nsteps) {
  g_err.clear();
  if (!group || n < 1 || nsteps < 0) return fail(DG_ERR_ARG, "bad group arguments");
  std::vector<dg_solver*> g(n, nullptr);
  for (int i = 0; i < n; ++i) {
    dg_solver* s = group[i];
    dg_status st = need_device(s);
    if (st != DG_OK) return st;
    if (!s->has_fields) return fail(DG_ERR_STATE, "group member without fields");
    if (s->cfg.nranks != n || s->cfg.rank < 0 || s->cfg.rank >= n || g[s->cfg.rank])
      return fail(DG_ERR_ARG, "group must hold ranks 0..n-1 of one partition, once each");
    if (n > 1 && !s->loopback) return fail(DG_ERR_ARG, "group members must be loopback solvers (nccl_id NULL)");
    g[s->cfg.rank] = s;
  }
  for (int i = 1; i < n; ++i)
    if (g[i]->N != g[0]->N || g[i]->fp64 != g[0]->fp64 || g[i]->cur != g[0]->cur || g[i]->mesh.K != g[0]->mesh.K ||
        g[i]->lay.E != g[0]->lay.E || g[i]->lay.perm != g[0]->lay.perm || g[i]->nc != g[0]->nc)
      return fail(DG_ERR_ARG, "group members differ in order, precision, variant, mesh or step parity");
  bool prime = false;
  for (int i = 0; i < n; ++i) prime = prime || (g[i]->part.n_ghost_faces > 0 && !g[i]->ghosts_valid);
  if (nsteps > 0 && prime) {
    const int cur = g[0]->cur;
    dg_status st = g[0]->fp64 ? group_exchange<double>(g.data(), n, cur, false)
                              : group_exchange<float>(g.data(), n, cur, false);
    if (st != DG_OK) return st;
    for (int i = 0; i < n; ++i) g[i]->ghosts_valid = true;
  }
  for (int step = 0; step < nsteps; ++step) {
    for (int stage = 0; stage < 5; ++stage) {
      const int cur = g[0]->cur;
      dg_status st = g[0]->fp64 ? group_stage<double>(g.data(), n, stage, dt, cur)
                                : group_stage<float>(g.data(), n, stage, dt, cur);
      if (st != DG_OK) return st;
      for (int i = 0; i < n; ++i) g[i]->cur ^= 1;
    }
  }
  return DG_OK;
}

dg_status dg_synchronize(dg_solver* s) {
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaStreamSynchronize(s->comm));
  if (s->h2d) CK(cudaStreamSynchronize(s->h2d));
  if (s->d2h) CK(cudaStreamSynchronize(s->d2h));
  CK(cudaGetLastError());
  return DG_OK;
}

dg_status dg_get_maps(dg_solver* s, int64_t* EToE, int8_t* EToF, int64_t* vmapM, int64_t* vmapP) {
  if (!s) return fail(DG_ERR_ARG, "null solver");
  if (!s->has_mesh) return fail(DG_ERR_STATE, "no mesh uploaded");
  const auto& m = s->mesh;
  if (EToE) std::memcpy(EToE, m.EToE.data(), m.EToE.size() * sizeof(int64_t));
  if (EToF) std::memcpy(EToF, m.EToF.data(), m.EToF.size());
  if (vmapM || vmapP) dg::build_maps(s->ref, s->mesh);
  if (vmapM) std::memcpy(vmapM, m.vmapM.data(), m.vmapM.size() * sizeof(int64_t));
  if (vmapP) std::memcpy(vmapP, m.vmapP.data(), m.vmapP.size() * sizeof(int64_t));
  return DG_OK;
}

dg_status dg_get_nodes(dg_solver* s, double* x, double* y, double* z) {
  if (!s || !x || !y || !z) return fail(DG_ERR_ARG, "null argument");
  if (!s->has_mesh) return fail(DG_ERR_STATE, "no mesh uploaded");
  const int64_t K = s->mesh.K, Np = s->Np;
  std::vector<double> X(K * Np), Y(K * Np), Z(K * Np);
  dg::node_coords(s->ref, s->mesh, X.data(), Y.data(), Z.data());
  for (int64_t l = 0; l < s->part.K_local; ++l) {
    const int64_t k = s->part.local_ids[l];
    std::memcpy(x + l * Np, &X[k * Np], Np * sizeof(double));
    std::memcpy(y + l * Np, &Y[k * Np], Np * sizeof(double));
    std::memcpy(z + l * Np, &Z[k * Np], Np * sizeof(double));
  }
  return DG_OK;
}

dg_status dg_get_reference(dg_solver* s, double* r, double* st_, double* t, double* Dr, double* Ds, double* Dt,
                           double* M, double* LIFT, int32_t* Fmask) {
  if (!s) return fail(DG_ERR_ARG, "null solver");
  const auto& R = s->ref;
  const size_t Np = R.Np;
  if (r) std::memcpy(r, R.r.data(), Np * sizeof(double));
  if (st_) std::memcpy(st_, R.s.data(), Np * sizeof(double));
  if (t) std::memcpy(t, R.t.data(), Np * sizeof(double));
  if (Dr) std::memcpy(Dr, R.Dr.a.data(), Np * Np * sizeof(double));
  if (Ds) std::memcpy(Ds, R.Ds.a.data(), Np * Np * sizeof(double));
  if (Dt) std::memcpy(Dt, R.Dt.a.data(), Np * Np * sizeof(double));
  if (M) std::memcpy(M, R.M.a.data(), Np * Np * sizeof(double));
  if (LIFT) std::memcpy(LIFT, R.LIFT.a.data(), R.LIFT.a.size() * sizeof(double));
  if (Fmask)
    for (size_t i = 0; i < R.Fmask.size(); ++i) Fmask[i] = R.Fmask[i];
  return DG_OK;
}

dg_status dg_get_geometry(dg_solver* s, double* J, double* rst_x, double* nrm) {
  if (!s) return fail(DG_ERR_ARG, "null solver");
  if (!s->has_mesh) return fail(DG_ERR_STATE, "no mesh uploaded");
  const auto& m = s->mesh;
  if (J) std::memcpy(J, m.J.data(), m.J.size() * sizeof(double));
  if (rst_x) std::memcpy(rst_x, m.rst_x.data(), m.rst_x.size() * sizeof(double));
  if (nrm) std::memcpy(nrm, m.nrm.data(), m.nrm.size() * sizeof(double));
  return DG_OK;
}

dg_status dg_poison_padding(dg_solver* s) {
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!s->has_fields) return fail(DG_ERR_STATE, "dg_poison_padding before dg_fields_upload");
  void* bufs[4] = {s->d_u[0], s->d_u[1], s->d_res, s->d_scratch};
  for (void* b : bufs) {
    if (s->fp64)
      dg::poison_padding<double>(static_cast<double*>(b), s->Kl, s->Np, s->lay, s->stream);
    else
      dg::poison_padding<float>(static_cast<float*>(b), s->Kl, s->Np, s->lay, s->stream);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s->stream));
  return DG_OK;
}

dg_status dg_check_padding(dg_solver* s, int64_t* counts) {
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!counts) return fail(DG_ERR_ARG, "null counts");
  if (!s->has_fields) return fail(DG_ERR_STATE, "dg_check_padding before dg_fields_upload");
  unsigned long long* d = nullptr;
  CK(cudaMalloc((void**)&d, 8 * sizeof(unsigned long long)));
  CK(cudaMemsetAsync(d, 0, 8 * sizeof(unsigned long long), s->stream));
  void* bufs[4] = {s->d_u[0], s->d_u[1], s->d_res, s->d_scratch};
  for (int i = 0; i < 4; ++i) {
    if (s->fp64)
      dg::check_padding<double>(static_cast<const double*>(bufs[i]), s->Kl, s->Np, s->lay, d + 2 * i, s->stream);
    else
      dg::check_padding<float>(static_cast<const float*>(bufs[i]), s->Kl, s->Np, s->lay, d + 2 * i, s->stream);
  }
  unsigned long long h[8];
  cudaError_t e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "dg_check_padding");
  for (int i = 0; i < 8; ++i) counts[i] = int64_t(h[i]);
  return DG_OK;
}

dg_status dg_time_stage_kernel(dg_solver* s, int32_t reps, double* ms) {
  g_err.clear();
  dg_status st = need_device(s);
  if (st != DG_OK) return st;
  if (!s->has_fields) return fail(DG_ERR_STATE, "no fields uploaded");
  if (reps < 1 || !ms) return fail(DG_ERR_ARG, "reps < 1 or null output");
  return s->fp64 ? time_stage<double>(s, reps, ms) : time_stage<float>(s, reps, ms);
}

dg_status dg_launches_per_step(dg_solver* s, int32_t* n) {
  if (!s || !n) return fail(DG_ERR_ARG, "null argument");
  const bool halo = s->has_mesh && s->part.n_ghost_faces > 0;
  // per stage: the stage kernel (+ the pack kernel of the trace exchange)
  *n = 5 * (halo ? 2 : 1);
  return DG_OK;
}

dg_status dg_kernel_variant(dg_solver* s, int32_t* variant) {
  if (!s || !variant) return fail(DG_ERR_ARG, "null argument");
  *variant = int32_t(s->variant);
  return DG_OK;
}

void dg_destroy(dg_solver* s) {
  if (!s) return;
  if (!s->host_only) {
    cudaSetDevice(s->cfg.device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->comm) cudaStreamSynchronize(s->comm);
    if (s->h2d) cudaStreamSynchronize(s->h2d);
    if (s->d2h) cudaStreamSynchronize(s->d2h);
    release_device(s);
    for (int i = 0; i < 2; ++i) {
      if (s->ev_in_ready[i]) cudaEventDestroy(s->ev_in_ready[i]);
      if (s->ev_in_free[i]) cudaEventDestroy(s->ev_in_free[i]);
      if (s->ev_out_ready[i]) cudaEventDestroy(s->ev_out_ready[i]);
      if (s->ev_out_free[i]) cudaEventDestroy(s->ev_out_free[i]);
    }
    if (s->h2d) cudaStreamDestroy(s->h2d);
    if (s->d2h) cudaStreamDestroy(s->d2h);
    if (s->ncomm && nccl().ok) nccl().CommDestroy(s->ncomm);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->ev_t0) cudaEventDestroy(s->ev_t0);
    if (s->ev_t1) cudaEventDestroy(s->ev_t1);
    if (s->ev_packed) cudaEventDestroy(s->ev_packed);
    if (s->ev_copied) cudaEventDestroy(s->ev_copied);
    if (s->ev_done) cudaEventDestroy(s->ev_done);
    if (s->comm) cudaStreamDestroy(s->comm);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  }
  delete s;
}

}  // extern "C"
