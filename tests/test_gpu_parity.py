"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on identical seeded inputs.

Tolerances (DESIGN.md §"Tolerances"):
  * FP64: max|gpu - oracle| / max|oracle| <= 1e-12 (north_star), for a single RHS
    and after a fixed number of LSERK4 steps;
  * FP32: <= 1e-4 after the steps (north_star); a single FP32 RHS <= 2e-5
    (single-precision rounding of Np-term dot products, ~Np * 6e-8, plus the
    rounded geometry/operators);
  * maps and connectivity: bit-exact (tests/test_abi.py).
"""
import numpy as np
import pytest

import dg_inputs as di
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1211_0582_b200.dg import Solver, group_lserk_step  # noqa: E402

TOL_RHS = {8: 1e-12, 4: 2e-5}
TOL_STEP = {8: 1e-12, 4: 1e-4}


def relerr(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def mesh(n, sh=None, rot=None, jit=None):
    VX, E = di.kuhn_box(n)
    if sh is not None:
        E, _ = di.shuffle_elements(E, sh)
    if rot is not None:
        E = di.rotate_local_vertices(E, rot)
    if jit is not None:
        VX = di.jitter_interior(VX, n, jit)
    return VX, E


_SETUPS = {}


def setup(key, VX, E, N):
    k = (key, N)
    if k not in _SETUPS:
        _SETUPS[k] = oracle.Setup(VX, E, N)
    return _SETUPS[k]


# FP64 BASIC, MMA, MMA_WS (DMMA), FFMA (register-tiled DFMA); FP32 BASIC, MMA_WS (3xTF32 HMMA),
# TC (tcgen05), FFMA (register-tiled FFMA)
VARIANTS = [(8, 1), (8, 2), (8, 3), (8, 6), (4, 1), (4, 3), (4, 4), (4, 6)]
VIDS = ["f64-basic", "f64-mma", "f64-ws", "f64-ffma", "f32-basic", "f32-ws", "f32-tc", "f32-ffma"]


def supported(N, prec, variant):
    pass  # every variant covers N = 1..9


@pytest.mark.parametrize("prec,variant", VARIANTS, ids=VIDS)
@pytest.mark.parametrize("N", range(1, 10))
def test_rhs_random_fields_shuffled_jittered(N, prec, variant):
    supported(N, prec, variant)
    VX, E = mesh(3, 1, 2, 3)                      # K = 162: ragged tail for every tile size
    st = setup("m3", VX, E, N)
    U = di.random_fields(st.K, N, seed=0)
    s = Solver(N, precision=prec, variant=variant)
    s.mesh_upload(VX, E)
    s.fields_upload(U)
    R = s.rhs()
    Ro = oracle.rhs(st, U)
    assert relerr(R, Ro) < TOL_RHS[prec]
    # fields round-trip (FP32: exact widening of the rounded upload)
    back = s.fields_download()
    if prec == 8:
        assert np.array_equal(back, U)
    else:
        assert np.array_equal(back, U.astype(np.float32).astype(np.float64))
    s.close()


@pytest.mark.parametrize("prec", [8, 4])
def test_c1_cavity_100_steps(prec):
    # config C1: unit cube, 2x2x2 cubes x 6 tets, N=3, 100 LSERK4 steps
    N = 3
    VX, E = di.kuhn_box(2)
    st = setup("c1", VX, E, N)
    U0 = di.cavity_mode_101(st.x, st.y, st.z)
    dt = di.dt_rule(VX, E, N)
    s = Solver(N, precision=prec)
    s.mesh_upload(VX, E)
    x, y, z = s.get_nodes()
    s.fields_upload(di.cavity_mode_101(x, y, z))
    s.lserk_step(dt, 100)
    U = s.fields_download()
    Uo = oracle.lserk4(st, U0, dt, 100)
    assert relerr(U, Uo) < TOL_STEP[prec]
    s.close()


@pytest.mark.parametrize("prec,variant", VARIANTS, ids=VIDS)
@pytest.mark.parametrize("N", range(1, 10))
def test_lserk_steps_all_orders(N, prec, variant):
    supported(N, prec, variant)
    VX, E = mesh(2, 5, 6, 7)
    st = setup("m2", VX, E, N)
    U0 = di.random_fields(st.K, N, seed=1)
    dt = di.dt_rule(VX, E, N)
    s = Solver(N, precision=prec, variant=variant)
    s.mesh_upload(VX, E)
    s.fields_upload(U0)
    # split the steps across calls: exercises both graph parities and re-use
    s.lserk_step(dt, 3)
    s.lserk_step(dt, 4)
    U = s.fields_download()
    Uo = oracle.lserk4(st, U0, dt, 7)
    assert relerr(U, Uo) < TOL_STEP[prec]
    s.close()


def test_single_element_all_pec():
    VX = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    E = np.array([[0, 1, 2, 3]])
    for N in (1, 5, 9):
        st = oracle.Setup(VX, E, N)
        U = di.random_fields(1, N, seed=4)
        s = Solver(N)
        s.mesh_upload(VX, E)
        s.fields_upload(U)
        assert relerr(s.rhs(), oracle.rhs(st, U)) < 1e-12
        s.close()


def test_zero_fields_zero_rhs_and_dt_zero_identity():
    VX, E = di.kuhn_box(2)
    s = Solver(4)
    s.mesh_upload(VX, E)
    s.fields_upload(np.zeros((6, s.K_local, s.Np)))
    assert np.all(s.rhs() == 0)
    U = di.random_fields(s.K_local, 4, seed=2)
    s.fields_upload(U)
    s.lserk_step(0.0, 3)
    assert np.array_equal(s.fields_download(), U)
    s.close()


def test_central_flux_alpha0():
    N = 3
    VX, E = mesh(2, 3, 4, 5)
    st = oracle.Setup(VX, E, N)
    U = di.random_fields(st.K, N, seed=3)
    s = Solver(N, alpha=0.0)
    s.mesh_upload(VX, E)
    s.fields_upload(U)
    assert relerr(s.rhs(), oracle.rhs(st, U, alpha=0.0)) < 1e-12
    s.close()


@pytest.mark.parametrize("prec", [8, 4])
def test_central_flux_energy_conserved_on_gpu(prec):
    # NEXT-2: alpha = 0 with PEC walls is a skew operator in the M_g inner
    # product, so the discrete energy is conserved up to the O(dt^6) LSERK4 defect
    # (oracle pin: tests/test_oracle_operator.py::test_central_flux_energy_drift_small);
    # the upwind flux (alpha = 1) must dissipate.
    N = 4
    VX, E = mesh(2, 7, 8, None)
    st = oracle.Setup(VX, E, N)
    U0 = di.random_fields(st.K, N, seed=11)
    dt = di.dt_rule(VX, E, N)
    e0 = oracle.energy(st, U0)
    out = {}
    for alpha in (0.0, 1.0):
        s = Solver(N, precision=prec, alpha=alpha)
        s.mesh_upload(VX, E)
        s.fields_upload(U0)
        s.lserk_step(dt, 50)
        out[alpha] = s.fields_download()
        s.close()
    # random fields load the top of the spectrum, where the LSERK4 defect |R(iy)| - 1
    # ~ -y^6/72 gives an oracle drift of -2.25e-6 over 50 steps (upwind: -39%)
    assert abs(oracle.energy(st, out[0.0]) - e0) / e0 < (1e-5 if prec == 8 else 1e-4)
    assert oracle.energy(st, out[1.0]) < 0.7 * e0
    if prec == 8:
        ref = oracle.lserk4(st, U0, dt, 50, alpha=0.0)
        assert relerr(out[0.0], ref) < 1e-11
        assert abs(oracle.energy(st, out[0.0]) - oracle.energy(st, ref)) < 1e-12 * e0


@pytest.mark.parametrize("prec,variant", VARIANTS, ids=VIDS)
@pytest.mark.parametrize("N", [1, 3, 4, 7])
def test_morton_reorder(N, prec, variant):
    # reorder=1: the library renumbers elements along a Morton curve; fields are in the
    # storage order dg_local_elements reports, results must equal the oracle's permuted
    supported(N, prec, variant)
    VX, E = mesh(6, 31, 32, 33)
    st = setup("m6", VX, E, N)
    U0 = di.random_fields(st.K, N, seed=9)
    s = Solver(N, precision=prec, variant=variant, reorder=True)
    s.mesh_upload(VX, E)
    ids = s.local_elements()
    assert np.array_equal(np.sort(ids), np.arange(st.K)) and not np.array_equal(ids, np.arange(st.K))
    s.fields_upload(np.ascontiguousarray(U0[:, ids]))
    assert relerr(s.rhs(), oracle.rhs(st, U0)[:, ids]) < TOL_RHS[prec]
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 2)
    assert relerr(s.fields_download(), oracle.lserk4(st, U0, dt, 2)[:, ids]) < TOL_STEP[prec]
    s.close()


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("N", [1, 4, 9])
def test_bench_mesh_full_size(N, prec):
    # the bench workload (config C2: Kuhn n=15, K=20250), full-size comparison
    # of one RHS and one graph-launched LSERK4 step
    VX, E = di.kuhn_box(15)
    st = setup("c2", VX, E, N)
    U0 = di.random_fields(st.K, N, seed=0)
    s = Solver(N, precision=prec)
    s.mesh_upload(VX, E)
    s.fields_upload(U0)
    assert relerr(s.rhs(), oracle.rhs(st, U0)) < TOL_RHS[prec]
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 1)
    assert relerr(s.fields_download(), oracle.lserk4(st, U0, dt, 1)) < TOL_STEP[prec]
    s.close()


@pytest.mark.parametrize("prec,variant", VARIANTS, ids=VIDS)
@pytest.mark.parametrize("N", range(1, 10))
def test_many_tiles_per_cta_shuffled(N, prec, variant):
    supported(N, prec, variant)
    # K = 10368 on a shuffled/rotated/jittered mesh: the persistent MMA kernel runs
    # several element tiles per CTA (exercises its cp.async double buffering)
    VX, E = mesh(12, 21, 22, 23)
    st = setup("m12", VX, E, N)
    U0 = di.random_fields(st.K, N, seed=5)
    s = Solver(N, precision=prec, variant=variant)
    s.mesh_upload(VX, E)
    s.fields_upload(U0)
    assert relerr(s.rhs(), oracle.rhs(st, U0)) < TOL_RHS[prec]
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 2)
    assert relerr(s.fields_download(), oracle.lserk4(st, U0, dt, 2)) < TOL_STEP[prec]
    s.close()


def _submesh(VX, E, EToE, seeds, layers):
    keep = set(int(k) for k in seeds)
    front = set(keep)
    for _ in range(layers):
        nxt = set()
        for k in front:
            nxt.update(int(v) for v in EToE[k])
        front = nxt - keep
        keep |= nxt
    keep = np.array(sorted(keep))
    verts = np.unique(E[keep])
    remap = -np.ones(VX.shape[0], dtype=np.int64)
    remap[verts] = np.arange(len(verts))
    return keep, VX[verts], remap[E[keep]]


def test_sampled_oracle_at_c4_size():
    # config C4's mesh (Kuhn n=56, K=1,053,696, N=4, FP64) in the bench launch
    # configuration.  The oracle cannot run the whole mesh; it recomputes sampled
    # elements exactly on a sub-mesh of their face neighbourhood: 1 layer for one
    # RHS, 6 layers for one LSERK4 step (5 stages; the artificial boundary of the
    # sub-mesh cannot reach the centre).
    N, n = 4, 56
    VX, E = di.kuhn_box(n)
    K = E.shape[0]
    s = Solver(N)
    s.mesh_upload(VX, E)
    EToE, _, _, _ = s.get_maps()
    U0 = di.random_fields(K, N, seed=9)
    s.fields_upload(U0)
    R = s.rhs()
    rng = np.random.default_rng(0)
    samples = np.concatenate([[0, K - 1], rng.integers(0, K, 6)])
    keep, sVX, sE = _submesh(VX, E, EToE, samples, 1)
    st = oracle.Setup(sVX, sE, N)
    Rs = oracle.rhs(st, U0[:, keep])
    pos = np.searchsorted(keep, samples)
    assert relerr(R[:, samples], Rs[:, pos]) < 1e-12
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 1)
    U1 = s.fields_download()
    for k in samples[:3]:
        keep, sVX, sE = _submesh(VX, E, EToE, [k], 6)
        st = oracle.Setup(sVX, sE, N)
        Us = oracle.lserk4(st, U0[:, keep], dt, 1)
        p = np.searchsorted(keep, k)
        assert relerr(U1[:, k], Us[:, p]) < 1e-12
    s.close()


def test_sampled_oracle_beyond_2pow30_words():
    # maximum-size edge case: one rank whose state exceeds 2^30 words (FP32 N=9 -> the tcgen05
    # kernel, Kuhn n=52, K=843,648: 1.11e9 words per copy), so the last elements' neighbour
    # offsets need bit 30 of the int32 connectivity (ghost records and intra-tile faces are
    # negative codes; a flag bit here once cut the reach to 2^30 and faulted on C4 at N = 9).
    # Sampled elements, including the last one, against the oracle on their face-neighbourhood
    # sub-mesh.
    psutil = pytest.importorskip("psutil")
    if psutil.virtual_memory().available < 70e9:
        pytest.skip("needs ~70 GB of host memory for the FP64 host arrays")
    N, n, prec = 9, 52, 4
    VX, E = di.kuhn_box(n)
    K = E.shape[0]
    assert 6 * di.np_of(N) * K > 2 ** 30
    s = Solver(N, precision=prec)
    s.mesh_upload(VX, E)
    EToE, _, _, _ = s.get_maps()
    U0 = di.random_fields(K, N, seed=11)
    s.fields_upload(U0)
    R = s.rhs()
    rng = np.random.default_rng(1)
    samples = np.concatenate([[0, K - 1, K - 2], rng.integers(0, K, 3)])
    keep, sVX, sE = _submesh(VX, E, EToE, samples, 1)
    st = oracle.Setup(sVX, sE, N)
    Rs = oracle.rhs(st, U0[:, keep])
    pos = np.searchsorted(keep, samples)
    assert relerr(R[:, samples], Rs[:, pos]) < TOL_RHS[prec]
    del R
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 1)
    U1 = s.fields_download()
    for k in (K - 1, samples[-1]):
        keep, sVX, sE = _submesh(VX, E, EToE, [k], 6)
        st = oracle.Setup(sVX, sE, N)
        Us = oracle.lserk4(st, U0[:, keep], dt, 1)
        p = np.searchsorted(keep, k)
        assert relerr(U1[:, k], Us[:, p]) < TOL_STEP[prec]
    s.close()


@pytest.mark.parametrize("prec,variant", VARIANTS, ids=VIDS)
@pytest.mark.parametrize("P,how", [(2, "slabs"), (3, "random"), (4, "random")])
def test_partitioned_loopback_bitwise_equal_to_one_gpu(P, how, prec, variant):
    # a6 / §8(e): P partitions of one mesh stepped together; partition-face traces
    # travel through the pack kernel + ghost records exactly as on the NCCL path.
    # Per-element arithmetic is partition-independent (reading R15): bitwise equal.
    N = 3
    VX, E = mesh(6, 31, 32)
    K = E.shape[0]
    U0 = di.random_fields(K, N, seed=6)
    dt = di.dt_rule(VX, E, N)
    ref = Solver(N, precision=prec, variant=variant)
    ref.mesh_upload(VX, E)
    ref.fields_upload(U0)
    ref.lserk_step(dt, 3)
    Uref = ref.fields_download()
    ref.close()
    part = None if how == "slabs" else np.random.default_rng(P).integers(0, P, K).astype(np.int32)
    solvers, ids = [], []
    for r in range(P):
        sv = Solver(N, precision=prec, variant=variant, rank=r, nranks=P)
        sv.mesh_upload(VX, E, part)
        ids.append(sv.local_elements())
        sv.fields_upload(U0[:, ids[-1]])
        solvers.append(sv)
    assert sorted(np.concatenate(ids).tolist()) == list(range(K))
    group_lserk_step(solvers[::-1], dt, 3)          # any order of the group
    U = np.empty_like(U0)
    for sv, ix in zip(solvers, ids):
        U[:, ix] = sv.fields_download()
        sv.close()
    assert np.array_equal(U, Uref)
    if prec == 8:
        st = setup("m6p", VX, E, N)
        assert relerr(U, oracle.lserk4(st, U0, dt, 3)) < 1e-12


@pytest.mark.parametrize("prec", [8, 4])
def test_partitioned_loopback_p8_c4_per_rank_size(prec):
    # C4 (Kuhn n=56, K = 1 053 696, N = 4) as 8 z-slab partitions of 131 712 elements each
    # (the per-rank size of the 8-GPU C4 run), AUTO kernels (FP64 DMMA WS, FP32 tcgen05):
    # boundary-first single-launch stages with the trace exchange beside the interior tiles;
    # two steps bitwise equal to one solver over the whole mesh (reading R15).
    N, n, P = 4, 56, 8
    VX, E = di.kuhn_box(n)
    K = E.shape[0]
    U0 = di.random_fields(K, N, seed=8)
    dt = di.dt_rule(VX, E, N)
    ref = Solver(N, precision=prec)
    ref.mesh_upload(VX, E)
    ref.fields_upload(U0)
    ref.lserk_step(dt, 2)
    Uref = ref.fields_download()
    ref.close()
    solvers, ids = [], []
    for r in range(P):
        sv = Solver(N, precision=prec, rank=r, nranks=P)
        sv.mesh_upload(VX, E)
        ids.append(sv.local_elements())
        assert len(ids[-1]) == K // P
        sv.fields_upload(U0[:, ids[-1]])
        solvers.append(sv)
    group_lserk_step(solvers, dt, 1)
    group_lserk_step(solvers, dt, 1)                # ghosts stay valid across calls
    for sv, ix in zip(solvers, ids):
        assert np.array_equal(sv.fields_download(), Uref[:, ix])
        sv.close()


@pytest.mark.parametrize("N,ns", [(2, (2, 4, 8, 16)), (4, (2, 4, 8)), (6, (1, 2, 4))])
def test_convergence_study_c3(N, ns):
    # BASELINE.json configs[2] (C3): exact PEC cavity eigenmode (1,1,1) on h-refined
    # Kuhn meshes, T = 0.25 with the dt rule.  FP64: L2 error ~ h^(N+1) on the GPU
    # path (rate >= N + 0.5 on the finest pair) and GPU == oracle (<= 1e-12) on the
    # meshes the oracle finishes quickly.  FP32: tracks the FP64 discretisation
    # error down to its rounding floor (|e32 - e64| <= max(3e-6, 1e-3 e64)).
    import math
    T = 0.25
    errs = {8: [], 4: []}
    for n in ns:
        VX, E = di.kuhn_box(n)
        st = setup(f"cavity{n}", VX, E, N)
        U0 = di.cavity_mode_111(st.x, st.y, st.z)
        dt0 = di.dt_rule(VX, E, N)
        steps = int(math.ceil(T / dt0))
        ex = di.cavity_mode_111(st.x, st.y, st.z, t=T)
        for prec in (8, 4):
            s = Solver(N, precision=prec)
            s.mesh_upload(VX, E)
            x, y, z = s.get_nodes()
            s.fields_upload(di.cavity_mode_111(x, y, z))
            s.lserk_step(T / steps, steps)
            U = s.fields_download()
            s.close()
            errs[prec].append(math.sqrt(2 * oracle.energy(st, U - ex)))
            if prec == 8 and st.K <= 400:
                Uo = oracle.lserk4(st, U0, T / steps, steps)
                assert relerr(U, Uo) < 1e-12
    e64, e32 = errs[8], errs[4]
    rates = [math.log2(e64[i] / e64[i + 1]) for i in range(len(e64) - 1)]
    assert rates[-1] >= N + 0.5, (e64, rates)
    for a, b in zip(e32, e64):
        assert abs(a - b) <= max(3e-6, 1e-3 * b), (e32, e64)


# ------------------------------------------------------------------ NEXT-3: acoustics
from oracle import acoustics as oac  # noqa: E402
from paper_1211_0582_b200.dg import DG_SYSTEM_ACOUSTICS  # noqa: E402


@pytest.mark.parametrize("prec,variant", [(8, 1), (8, 6), (8, 3), (4, 1), (4, 6), (4, 4)],
                         ids=["f64-basic", "f64-ffma", "f64-ws", "f32-basic", "f32-ffma", "f32-tc"])
@pytest.mark.parametrize("N", range(1, 10))
def test_acoustics_rhs_and_steps(N, prec, variant):
    # the second linear system through the BASIC, FFMA, FP64 DMMA WS and tcgen05 TC stage kernels:
    # RHS and 2 LSERK4 steps vs the acoustics oracle on a shuffled/rotated/jittered mesh
    VX, E = mesh(3, 1, 2, 3)
    st = setup("m3", VX, E, N)
    U = di.random_fields(st.K, N, seed=2, nfields=4)
    s = Solver(N, precision=prec, system=DG_SYSTEM_ACOUSTICS, variant=variant)
    s.mesh_upload(VX, E)
    s.fields_upload(U)
    assert relerr(s.rhs(), oac.rhs(st, U)) < TOL_RHS[prec]
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 2)
    assert relerr(s.fields_download(), oac.lserk4(st, U, dt, 2)) < TOL_STEP[prec]
    s.close()


def test_acoustics_alpha0_energy_and_partitions():
    N = 3
    VX, E = mesh(4, 41, 42, 43)
    st = setup("m4", VX, E, N)
    K = st.K
    U0 = di.random_fields(K, N, seed=8, nfields=4)
    dt = di.dt_rule(VX, E, N)
    s = Solver(N, alpha=0.0, system=DG_SYSTEM_ACOUSTICS)
    s.mesh_upload(VX, E)
    s.fields_upload(U0)
    assert relerr(s.rhs(), oac.rhs(st, U0, alpha=0.0)) < 1e-12
    s.lserk_step(dt, 20)
    U = s.fields_download()
    s.close()
    e0 = oac.energy(st, U0)
    assert abs(oac.energy(st, U) - e0) / e0 < 1e-5
    assert relerr(U, oac.lserk4(st, U0, dt, 20, alpha=0.0)) < 1e-11
    # 3 loopback partitions (4-field ghost records): bitwise equal to one solver
    ref = Solver(N, system=DG_SYSTEM_ACOUSTICS)
    ref.mesh_upload(VX, E)
    ref.fields_upload(U0)
    ref.lserk_step(dt, 3)
    Uref = ref.fields_download()
    ref.close()
    part = np.random.default_rng(3).integers(0, 3, K).astype(np.int32)
    solvers, ids = [], []
    for r in range(3):
        sv = Solver(N, rank=r, nranks=3, system=DG_SYSTEM_ACOUSTICS)
        sv.mesh_upload(VX, E, part)
        ids.append(sv.local_elements())
        sv.fields_upload(U0[:, ids[-1]])
        solvers.append(sv)
    group_lserk_step(solvers, dt, 3)
    Up = np.empty_like(U0)
    for sv, ix in zip(solvers, ids):
        Up[:, ix] = sv.fields_download()
        sv.close()
    assert np.array_equal(Up, Uref)


@pytest.mark.parametrize("N,prec,variant", [(4, 4, 4), (7, 4, 4), (4, 8, 3), (7, 8, 3)],
                         ids=["tc-N4", "tc-N7", "ws-N4", "ws-N7"])
def test_acoustics_tensor_kernels_partitions_and_many_tiles(N, prec, variant):
    # acoustics through the tensor-core kernels (FP32 tcgen05: 24-element tiles; FP64 DMMA WS: 4 x 4-column
    # element groups), 4-field ghost records, rigid walls, on a mesh with many tiles per CTA: RHS vs the
    # oracle on sampled elements, and 3 loopback partitions bitwise equal to one solver after 2 steps
    VX, E = mesh(9, 5, 6, 7)
    K = E.shape[0]
    U0 = di.random_fields(K, N, seed=9, nfields=4)
    dt = di.dt_rule(VX, E, N)
    ref = Solver(N, precision=prec, system=DG_SYSTEM_ACOUSTICS, variant=variant)
    ref.mesh_upload(VX, E)
    EToE, _, _, _ = ref.get_maps()
    ref.fields_upload(U0)
    R = ref.rhs()
    samples = np.array([0, K // 3, K - 1])
    keep, sVX, sE = _submesh(VX, E, EToE, samples, 1)
    st = oracle.Setup(sVX, sE, N)
    Rs = oac.rhs(st, U0[:, keep])
    assert relerr(R[:, samples], Rs[:, np.searchsorted(keep, samples)]) < TOL_RHS[prec]
    ref.lserk_step(dt, 2)
    Uref = ref.fields_download()
    ref.close()
    part = np.random.default_rng(N).integers(0, 3, K).astype(np.int32)
    solvers, ids = [], []
    for r in range(3):
        sv = Solver(N, precision=prec, rank=r, nranks=3, system=DG_SYSTEM_ACOUSTICS, variant=variant)
        sv.mesh_upload(VX, E, part)
        ids.append(sv.local_elements())
        sv.fields_upload(U0[:, ids[-1]])
        solvers.append(sv)
    group_lserk_step(solvers, dt, 2)
    Up = np.empty_like(U0)
    for sv, ix in zip(solvers, ids):
        Up[:, ix] = sv.fields_download()
        sv.close()
    assert np.array_equal(Up, Uref)


@pytest.mark.parametrize("N", [2, 4])
def test_acoustics_convergence_rigid_wall_mode(N):
    import math
    T = 0.25
    errs = []
    for n in (2, 4, 8):
        VX, E = di.kuhn_box(n)
        s = Solver(N, system=DG_SYSTEM_ACOUSTICS)
        s.mesh_upload(VX, E)
        x, y, z = s.get_nodes()
        dt0 = di.dt_rule(VX, E, N)
        steps = int(math.ceil(T / dt0))
        s.fields_upload(di.acoustic_mode(x, y, z))
        s.lserk_step(T / steps, steps)
        D = s.fields_download() - di.acoustic_mode(x, y, z, t=T)
        s.close()
        st = setup(f"cavity{n}", VX, E, N)
        errs.append(math.sqrt(2 * oac.energy(st, D)))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] >= N + 0.5, (errs, rates)




# ------------------------------------------------------------------ pipelined host I/O
@pytest.mark.parametrize("prec", [8, 4])
def test_pipelined_async_io_equals_synchronous(prec):
    # upload_async / lserk_step / download_async cycles (copy streams, double-buffered
    # staging) give exactly the fields of the synchronous calls, for every cycle
    N = 4
    VX, E = mesh(5, 61, 62, 63)
    K = E.shape[0]
    dt = di.dt_rule(VX, E, N)
    ins = [torch.from_numpy(di.random_fields(K, N, seed=20 + k)).pin_memory().numpy() for k in range(4)]
    outs = [torch.empty((6, K, di.np_of(N)), dtype=torch.float64).pin_memory().numpy() for _ in range(4)]
    a = Solver(N, precision=prec)
    a.mesh_upload(VX, E)
    for k in range(4):
        a.fields_upload_async(ins[k])
        a.lserk_step(dt, 1 + k % 2)
        a.fields_download_async(outs[k])
    a.synchronize()
    ref = Solver(N, precision=prec)
    ref.mesh_upload(VX, E)
    for k in range(4):
        ref.fields_upload(ins[k])
        ref.lserk_step(dt, 1 + k % 2)
        assert np.array_equal(outs[k], ref.fields_download())
    a.close()
    ref.close()


@pytest.mark.parametrize("prec,variant", VARIANTS, ids=VIDS)
@pytest.mark.parametrize("N", [1, 3, 4, 8])
def test_nan_poisoned_padding(N, prec, variant):
    # SPEC.md:230 / SURVEY §4 item 4: every padding word of the field buffers (tile / LD padding,
    # absent elements of the ragged last tile) is NaN; the RHS and two steps must leave the
    # real DOFs finite and equal to the oracle, and must neither read nor overwrite the padding
    VX, E = mesh(3, 1, 2, 3)                      # K = 162: ragged last tile for every tile size
    st = setup("m3", VX, E, N)
    U = di.random_fields(st.K, N, seed=0)
    s = Solver(N, precision=prec, variant=variant)
    s.mesh_upload(VX, E)
    s.fields_upload(U)
    s.poison_padding()
    R = s.rhs()
    assert np.isfinite(R).all()
    assert relerr(R, oracle.rhs(st, U)) < TOL_RHS[prec]
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 2)
    Un = s.fields_download()
    assert np.isfinite(Un).all()
    assert relerr(Un, oracle.lserk4(st, U, dt, 2)) < TOL_STEP[prec]
    for name, (pad_not_nan, bad_dofs) in zip(("u0", "u1", "res", "scratch"), s.check_padding()):
        assert bad_dofs == 0, (name, bad_dofs)
        assert pad_not_nan == 0, (name, pad_not_nan)
    s.close()


@pytest.mark.parametrize("prec,variant", [(8, 3), (4, 4), (4, 6)], ids=["f64-ws", "f32-tc", "f32-ffma"])
def test_rcb_loopback_p8_bitwise(prec, variant):
    # 8 partitions by recursive coordinate bisection (several peers per rank, ghost faces on every
    # side) through the boundary-first single-launch stages: bitwise equal to one solver (R15)
    from paper_1211_0582_b200.dg import DG_PARTITION_RCB
    N = 3
    VX, E = mesh(6, 51, 52, 53)
    K = E.shape[0]
    U0 = di.random_fields(K, N, seed=12)
    dt = di.dt_rule(VX, E, N)
    ref = Solver(N, precision=prec, variant=variant)
    ref.mesh_upload(VX, E)
    ref.fields_upload(U0)
    ref.lserk_step(dt, 2)
    Uref = ref.fields_download()
    ref.close()
    solvers, ids = [], []
    for r in range(8):
        sv = Solver(N, precision=prec, variant=variant, rank=r, nranks=8, partition=DG_PARTITION_RCB)
        sv.mesh_upload(VX, E)
        ids.append(sv.local_elements())
        sv.fields_upload(U0[:, ids[-1]])
        solvers.append(sv)
    assert sorted(np.concatenate(ids).tolist()) == list(range(K))
    group_lserk_step(solvers, dt, 2)
    U = np.empty_like(U0)
    for sv, ix in zip(solvers, ids):
        U[:, ix] = sv.fields_download()
        sv.close()
    assert np.array_equal(U, Uref)


@pytest.mark.parametrize("prec,variant", [(4, 4), (8, 3)], ids=["f32-tc", "f64-ws"])
def test_acoustics_alpha0_tensor_kernels(prec, variant):
    # central acoustic flux (alpha = 0) through the tensor-core kernels: RHS vs the oracle, and the
    # discrete acoustic energy conserved over 20 steps to the time-integration error
    N = 4
    VX, E = mesh(3, 61, 62, 63)
    st = setup("m3b", VX, E, N)
    U0 = di.random_fields(st.K, N, seed=13, nfields=4)
    s = Solver(N, precision=prec, alpha=0.0, system=DG_SYSTEM_ACOUSTICS, variant=variant)
    s.mesh_upload(VX, E)
    s.fields_upload(U0)
    assert relerr(s.rhs(), oac.rhs(st, U0, alpha=0.0)) < TOL_RHS[prec]
    dt = di.dt_rule(VX, E, N)
    s.lserk_step(dt, 20)
    U = s.fields_download()
    s.close()
    e0 = oac.energy(st, U0)
    assert abs(oac.energy(st, U) - e0) / e0 < (1e-5 if prec == 8 else 1e-4)
