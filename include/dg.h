/*
 * dg.h — C ABI of the B200 nodal-DG Maxwell library (libdg.so).
 *
 * What it computes: the semi-discrete DG operator of PAPER.md eq. (4)
 *
 *
 *     d_t u^k = - sum_nu D^{k,d nu} F(u^k) + L^k [ n.F - (n.F)^* ]
 *
 * for 3-D Maxwell in vacuum (d_t E = curl H, d_t H = -curl E, eps = mu = 1) on
 * straight-sided, face-conforming tetrahedra, with
 * nodal trace picking, the upwind flux of fig:flux-code a
 * with jump [[u]] = u+ - u- (reading R1), PEC
 * walls E+ = -E-, H+ = H- (reading R4), the lifting matrix of fig:lifting-matrix
 * (PAPER.md:170-216), advanced by 5-stage 2N-storage LSERK4 ("RK4 time stepping",
 * PAPER.md:1179-1181; reading R5).  Every step of the hot path runs in the
 * library's own sm_100a CUDA kernels; there is no CPU fallback.
 *
 * Conventions (all entry points)
 *   - Every call returns dg_status; nothing throws or aborts across the ABI.
 *     On failure dg_last_error() returns a thread-local description.
 *   - Host arrays are borrowed for the duration of the call and copied.
 *     Device buffers the solver allocates are owned by it and freed by
 *     dg_destroy.  Caller device pointers (the *_device variants) are borrowed
 *     and must stay valid until the enqueued work completes.
 *   - One host thread per solver; separate solvers are independent.
 *   - Call order: dg_create -> dg_mesh_upload -> dg_fields_upload[_device] ->
 *     { dg_rhs[_device] | dg_lserk_step }* -> dg_fields_download[_device].
 *     A call out of order returns DG_ERR_STATE.
 *   - Fields on the host are FP64, component-major [6][K_local][Np] in the
 *     order (Ex, Ey, Ez, Hx, Hy, Hz), node index fastest (HW's Np x K per
 *     component).  With dg_config.system = DG_SYSTEM_ACOUSTICS every "[6]" below
 *     reads "[4]", components (p, vx, vy, vz).  Node n of element k is the n-th warp&blend node mapped
 *     affinely (dg_get_nodes).  FP32 solvers round on upload and widen exactly
 *     on download.
 *   - Work is enqueued on the solver's stream (dg_config.stream, or a
 *     solver-owned stream).  Calls that return host data synchronise it;
 *     asynchronous CUDA errors surface at the next synchronising call.
 *   - dt is always explicit: the library never chooses a time step.
 */
#ifndef DG_H_
#define DG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_ABI_VERSION 1

#if defined(__GNUC__)
#define DG_API __attribute__((visibility("default")))
#else
#define DG_API
#endif

typedef struct dg_solver dg_solver; /* opaque */

typedef enum {
  DG_OK = 0,
  DG_ERR_ARG = 1,   /* null pointer, bad size or bad enum value */
  DG_ERR_ORDER = 2, /* order N outside 1..9 */
  DG_ERR_MESH = 3,  /* J <= 0, face shared by > 2 tets, unmatched face nodes, bad ids */
  DG_ERR_STATE = 4, /* call out of order, or a compute call on a host-only solver */
  DG_ERR_CUDA = 5,  /* CUDA runtime error (message has the CUDA error string) */
  DG_ERR_NCCL = 6,  /* NCCL error or NCCL not loadable */
  DG_ERR_OOM = 7    /* device allocation failed */
} dg_status;

typedef enum {
  DG_VARIANT_AUTO = 0,   /* measured best per (precision, N): FP64 MMA_WS (N >= 2) / FFMA (N = 1);
                            FP32 TC (N >= 4) / FFMA (N <= 3) (tools/variant_sweep.py) */
  DG_VARIANT_BASIC = 1,  /* one fused element-tile kernel per stage, FMA contractions */
  DG_VARIANT_MMA = 2,    /* FP64: DMMA contractions, cp.async-pipelined persistent kernel
                            (FP32: same as BASIC) */
  DG_VARIANT_MMA_WS = 3, /* warp-specialized TMA/mbarrier pipeline; contractions on tensor
                            cores: FP64 DMMA, FP32 3xTF32 HMMA */
  DG_VARIANT_TC = 4,     /* FP32, N = 1..9: the whole RHS of a 21-element (acoustics: 24) tile as one K-chunked
                            tcgen05.mma kind::tf32 GEMM (3xTF32): chain rule + curl folded into
                            the generated operand (written to tensor memory), upwind flux as
                            the lift operand, TMEM accumulators, LSERK update in the epilogue
                            (5th-generation tensor cores; stage_tc.cuh) */
  DG_VARIANT_FUSED = 5,  /* withdrawn in round 2 (dg_create returns DG_ERR_ARG): the stage-fused
                            WS launch was slower than per-stage launches */
  DG_VARIANT_FFMA = 6    /* the warp-specialized TMA pipeline with both contractions as
                            register-tiled FFMA (FP32) / DFMA (FP64), no tensor cores: the
                            SIMT side of the TF32-or-FFMA and DMMA-or-DFMA comparisons
                             */
} dg_variant;

/* The linear hyperbolic system u_t + div F(u) = 0 the operator is
 * built for.  Both go through the same four stages (volume, flux gather, lift, update). */
typedef enum {
  DG_SYSTEM_MAXWELL = 0,   /* 6 fields (E, H): the north_star path; every variant */
  DG_SYSTEM_ACOUSTICS = 1  /* 4 fields (p, v), rho0 = c = 1: p_t + div v = 0, v_t + grad p = 0;
                              upwind flux (-A_n + alpha |A_n|)[[u]]; rigid walls v.n = 0
                              (mirror p+ = p-, v+ = v- - 2 (n.v-) n); R16/R17.
                              FFMA, MMA_WS (FP64 DMMA), TC (FP32 tcgen05) and BASIC kernels; AUTO:
                              FP64 FFMA at N = 1, MMA_WS above; FP32 FFMA for N <= 3, TC above
                              (MMA, FP32 MMA_WS -> DG_ERR_ARG) */
} dg_system;

typedef struct {
  int32_t order;        /* polynomial order N, 1..9 */
  int32_t precision;    /* 8 = FP64, 4 = FP32 arithmetic and storage on the device */
  double alpha;         /* flux upwinding: 1.0 upwind (default), 0.0 central (fig:flux-code a) */
  int32_t device;       /* CUDA device ordinal; -1 = host-only solver (setup/maps/nodes only) */
  void* stream;         /* cudaStream_t to enqueue on; NULL = solver-owned stream */
  int32_t rank;         /* this process's rank, 0..nranks-1 */
  int32_t nranks;       /* number of ranks (one GPU each); 1 = single GPU */
  const void* nccl_id;  /* 128-byte ncclUniqueId from rank 0 (nranks > 1).  NULL with nranks > 1
                           makes a loopback partition solver: no NCCL; the ranks live in this
                           process and are stepped together by dg_group_lserk_step */
  int32_t variant;      /* dg_variant */
  int32_t reorder;      /* 1: renumber this rank's elements along a Morton curve of their
                           centroids (within the partition-boundary and interior groups) for
                           gather locality and intra-tile faces; dg_local_elements reports the
                           storage order.  0 (default): ascending global id within each group */
  int32_t system;       /* dg_system (default DG_SYSTEM_MAXWELL) */
  int32_t partition;    /* element owner when dg_mesh_upload gets part = NULL:
                           DG_PARTITION_RANGES (default): contiguous element-index ranges
                           (z-slabs on the cell-ordered Kuhn box); DG_PARTITION_RCB: recursive
                           coordinate bisection of the element centroids (longest extent,
                           rank-weighted median, ties by element id) */
} dg_config;

typedef enum { DG_PARTITION_RANGES = 0, DG_PARTITION_RCB = 1 } dg_partition;

/* Fill *cfg with defaults: N=3, FP64, alpha=1, device 0, own stream, 1 rank, AUTO,
 * no reorder, Maxwell, range partition. */
DG_API void dg_config_default(dg_config* cfg);

/* Create a solver.  Builds the reference element of order N on the host (FP64).
 * Errors: DG_ERR_ARG (null, precision not 4/8, nranks < 1, rank out of range, bad
 * variant or variant/system/precision/rank combination), DG_ERR_ORDER, DG_ERR_CUDA
 * (device unusable), DG_ERR_NCCL. */
DG_API dg_status dg_create(const dg_config* cfg, dg_solver** out);

/* Upload the (global) mesh: nv vertices VX[nv][3] (FP64), K tets EToV[K][4]
 * (0-based, positively oriented; not re-oriented).  part[K] gives the owner
 * rank of every element, or NULL for the built-in partition (contiguous element
 * ranges, i.e. z-slabs on the Kuhn box).  Builds connectivity, maps, geometry
 * and moves them to the device.  Errors:
 * DG_ERR_ARG, DG_ERR_MESH, DG_ERR_OOM, DG_ERR_CUDA, DG_ERR_NCCL.
 * May be called again to replace the mesh (fields must be re-uploaded). */
DG_API dg_status dg_mesh_upload(dg_solver* s, int64_t nv, const double* VX, int64_t K,
                         const int64_t* EToV, const int32_t* part);

/* Number of elements this rank owns and (optional) their global ids in storage order: the
 * partition-boundary elements (a face on another rank) first, then the interior ones, each
 * group ascending (or Morton-ordered with reorder = 1). */
DG_API dg_status dg_local_elements(dg_solver* s, int64_t* K_local, int64_t* global_ids);

/* Sizes: Np, Nfp, local and global element counts (any may be NULL). */
DG_API dg_status dg_get_sizes(dg_solver* s, int32_t* Np, int32_t* Nfp, int64_t* K_local, int64_t* K_global);

/* Upload fields f[6][K_local][Np] (host FP64).  Resets the LSERK residual to 0. */
DG_API dg_status dg_fields_upload(dg_solver* s, const double* f);
/* Same from device memory in the solver precision, layout [6][K_local][Np]. */
DG_API dg_status dg_fields_upload_device(dg_solver* s, const void* f_dev);

/* rhs[6][K_local][Np] (host FP64) = d_t u of the current fields (eq. 4).  Synchronises. */
DG_API dg_status dg_rhs(dg_solver* s, double* rhs);
/* Same into device memory in the solver precision, layout [6][K_local][Np]; asynchronous. */
DG_API dg_status dg_rhs_device(dg_solver* s, void* rhs_dev);

/* Advance nsteps >= 0 LSERK4 steps of size dt (5 stages each; asynchronous,
 * graph-launched).  With nranks > 1 every stage is ONE launch over the local tiles,
 * partition-boundary tiles first; once those are written (a counter the comm stream
 * waits for with cuStreamWaitValue32 — no kernel waits on anything) the comm stream
 * packs their face traces and exchanges them through NCCL send/recv into the ghost
 * region the NEXT stage reads, beside the interior tiles (DESIGN.md
 * §10).  The first step after a field upload primes the ghosts with one exchange.
 * Loopback solvers return DG_ERR_STATE (use dg_group_lserk_step). */
DG_API dg_status dg_lserk_step(dg_solver* s, double dt, int32_t nsteps);

/* Advance a group of loopback partition solvers (same mesh, order, precision and
 * variant; group[i] may be given in any order but must cover ranks 0..n-1 once)
 * by nsteps LSERK4 steps in lockstep.  The NCCL path's stage structure (one launch,
 * boundary tiles first, boundary signal, pack beside the interior tiles) with the
 * records copied device-to-device into the peers' ghost regions instead of
 * ncclSend/Recv.  Results are bitwise identical to one solver
 * on the whole mesh (reading R15).  Asynchronous.  Errors: DG_ERR_ARG,
 * DG_ERR_STATE (missing fields), DG_ERR_CUDA. */
DG_API dg_status dg_group_lserk_step(dg_solver* const* group, int32_t n, double dt, int32_t nsteps);

/* Copy the current fields out: host FP64 [6][K_local][Np] (synchronises) or
 * device memory in the solver precision (asynchronous). */
DG_API dg_status dg_fields_download(dg_solver* s, double* f);
DG_API dg_status dg_fields_download_device(dg_solver* s, void* f_dev);

/* Pipelined host I/O (FP64 host layout as dg_fields_upload / dg_fields_download).
 * Both calls only ENQUEUE work and return: the host->device copy runs on a solver-owned
 * copy-in stream into one of two staging buffers, the device->host copy on a copy-out
 * stream from one of two staging buffers, and the layout conversions on the compute
 * stream, ordered with dg_lserk_step / dg_rhs by events.  Consecutive
 * upload_async / lserk_step / download_async cycles therefore overlap the copies of one
 * cycle with the computation of its neighbours (PCIe is full duplex).  The host arrays
 * are borrowed until dg_synchronize returns (use page-locked memory for asynchronous
 * copies; pageable memory works but the driver then stages synchronously).  The fields
 * are ready for stepping when upload_async returns (ordering is on the device); a
 * download's data is valid after dg_synchronize.  upload_async resets the residual like
 * dg_fields_upload.  Errors: DG_ERR_ARG, DG_ERR_STATE (no mesh / no fields), DG_ERR_CUDA. */
DG_API dg_status dg_fields_upload_async(dg_solver* s, const double* f);
DG_API dg_status dg_fields_download_async(dg_solver* s, double* f);

/* Wait for all work enqueued by this solver (compute and copy streams); surfaces
 * asynchronous CUDA errors. */
DG_API dg_status dg_synchronize(dg_solver* s);

/* Parity exports of the host setup (work on host-only solvers too).
 * dg_get_maps: global mesh, EToE[K][4], EToF[K][4] (boundary face -> itself),
 *   vmapM/vmapP[K][4][Nfp] global node ids k*Np+n (boundary: vmapP = vmapM).
 * dg_get_nodes: physical node coordinates of the LOCAL elements, [K_local][Np].
 * dg_get_reference: r,s,t[Np], Dr,Ds,Dt,M[Np][Np], LIFT[Np][4Nfp], Fmask[4][Nfp]
 *   (row-major FP64; any pointer may be NULL). */
DG_API dg_status dg_get_maps(dg_solver* s, int64_t* EToE, int8_t* EToF, int64_t* vmapM, int64_t* vmapP);
DG_API dg_status dg_get_nodes(dg_solver* s, double* x, double* y, double* z);
DG_API dg_status dg_get_reference(dg_solver* s, double* r, double* st, double* t, double* Dr, double* Ds,
                           double* Dt, double* M, double* LIFT, int32_t* Fmask);
/* Geometry of the global mesh: J[K], rst_x[K][9] (rx ry rz sx sy sz tx ty tz),
 * nrm[K][4][4] (nx ny nz Fscale). */
DG_API dg_status dg_get_geometry(dg_solver* s, double* J, double* rst_x, double* nrm);

/* Measurement helper: time `reps` back-to-back launches of the LSERK stage
 * kernel (stage-1 coefficients, reading the current fields, writing the
 * ping-pong buffer and the residual) with CUDA events on the solver stream;
 * *ms_per_launch = mean device time per launch.  The current fields are
 * unchanged; the residual is clobbered, which is harmless because the next
 * step's first stage ignores it (a_0 = 0). */
DG_API dg_status dg_time_stage_kernel(dg_solver* s, int32_t reps, double* ms_per_launch);

/* Padding hygiene, for tests.  dg_poison_padding writes NaN
 * into every padding word (layout padding, absent elements of the last tile) of both field
 * buffers, the residual and the RHS scratch buffer; dg_check_padding fills counts[8] with,
 * for each of those four buffers in that order, (padding words that are no longer NaN, real
 * DOFs that are not finite).  A kernel that reads padding into its arithmetic, or writes
 * outside the real DOFs, shows up as non-zero counts.  Both synchronise.  Errors: DG_ERR_ARG,
 * DG_ERR_STATE (host-only solver, no fields), DG_ERR_CUDA. */
DG_API dg_status dg_poison_padding(dg_solver* s);
DG_API dg_status dg_check_padding(dg_solver* s, int64_t* counts);

/* Number of kernel launches one LSERK4 step enqueues on this rank (5 stage kernels, plus 5
 * pack kernels with partition faces). */
DG_API dg_status dg_launches_per_step(dg_solver* s, int32_t* n);

/* The stage kernel this solver runs (dg_variant; DG_VARIANT_AUTO resolved at dg_create to the
 * measured-best kernel for its precision, order and system).  Valid for host-only solvers too.  DG_ERR_ARG on null pointers. */
DG_API dg_status dg_kernel_variant(dg_solver* s, int32_t* variant);

/* Thread-local description of the last error ("" if none). */
DG_API const char* dg_last_error(void);
/* Library version string (build id, ABI version, compiled arch). */
DG_API const char* dg_version(void);

/* Free every device and host resource of the solver (NULL is a no-op). */
DG_API void dg_destroy(dg_solver* s);

#ifdef __cplusplus
}
#endif
#endif /* DG_H_ */
