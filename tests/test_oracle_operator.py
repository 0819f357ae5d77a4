"""Pins of the oracle's Maxwell operator and LSERK4 against closed forms,
brute-force operator properties, exact solutions and golden values."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import dg_inputs as di
from oracle import Setup, build_reference, energy, lserk4, lserk4_coefficients, rhs
from oracle.maxwell import lserk_integrate, upwind_flux

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ------------------------------------------------------------------ flux
def test_flux_worked_examples():
    for row in _golden("flux_examples.txt"):
        bar = row.index("|")
        vals = [float(v) for v in row[:bar]]
        want = np.array([float(v) for v in row[bar + 1:]])
        alpha, n, dE, dH = vals[0], vals[1:4], vals[4:7], vals[7:10]
        fl = upwind_flux(tuple(np.array([v]) for v in n), tuple(np.array([v]) for v in dE),
                         tuple(np.array([v]) for v in dH), alpha)
        got = np.array([fl[0][0], fl[1][0], fl[2][0]]) / 2.0
        assert np.allclose(got, want, atol=1e-15)


def test_flux_vector_identities():
    # fluxE = n x (dH - alpha n x dE), fluxH = -n x (dE + alpha n x dH): checked
    # with numpy's cross product on random unit normals; zero jump -> zero flux
    rng = np.random.default_rng(0)
    n = rng.normal(size=(50, 3)); n /= np.linalg.norm(n, axis=1)[:, None]
    dE = rng.normal(size=(50, 3)); dH = rng.normal(size=(50, 3))
    for alpha in (0.0, 1.0, 0.3):
        fl = upwind_flux(tuple(n.T), tuple(dE.T), tuple(dH.T), alpha)
        fE = np.stack(fl[:3], 1); fH = np.stack(fl[3:], 1)
        assert np.allclose(fE, np.cross(n, dH - alpha * np.cross(n, dE)), atol=1e-14)
        assert np.allclose(fH, -np.cross(n, dE + alpha * np.cross(n, dH)), atol=1e-14)
        z = upwind_flux(tuple(n.T), tuple(0 * dE.T), tuple(0 * dH.T), alpha)
        assert all(np.all(v == 0) for v in z)


# ------------------------------------------------------------------ operator
def _dense_operator(st, alpha):
    K, Np = st.K, st.Np
    n = 6 * K * Np
    A = np.zeros((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        A[:, j] = rhs(st, e.reshape(6, K, Np), alpha).ravel()
        e[j] = 0.0
    Mg = np.kron(np.eye(6), np.kron(np.diag(st.J), st.ref.M))
    return A, Mg


@pytest.mark.parametrize("N", [1, 2, 3])
def test_operator_skew_central_and_dissipative_upwind(N):
    # alpha = 0 + PEC: M_g A is skew (discrete energy conserved);
    # alpha = 1: M_g A + (M_g A)^T <= 0 (energy non-increasing) -- derived in SURVEY §8c
    VX, E = di.kuhn_box(1)
    E = di.rotate_local_vertices(E, 11)
    VX = VX.copy()
    st = Setup(VX, E, N)
    A0, Mg = _dense_operator(st, 0.0)
    S = Mg @ A0
    assert np.abs(S + S.T).max() < 1e-13 * np.abs(S).max()
    A1, _ = _dense_operator(st, 1.0)
    S1 = Mg @ A1
    ev = np.linalg.eigvalsh(0.5 * (S1 + S1.T))
    assert ev.max() < 1e-13 * np.abs(S1).max()
    assert ev.min() < -1e-3          # the upwind term really dissipates
    lam = np.linalg.eigvals(A1)
    assert lam.real.max() < 1e-11 * np.abs(lam).max()


def test_operator_skew_on_jittered_shuffled_mesh():
    VX, E = di.kuhn_box(2)
    E, _ = di.shuffle_elements(E, 3)
    E = di.rotate_local_vertices(E, 4)
    VX = di.jitter_interior(VX, 2, 5)
    st = Setup(VX, E, 1)
    A0, Mg = _dense_operator(st, 0.0)
    S = Mg @ A0
    assert np.abs(S + S.T).max() < 1e-13 * np.abs(S).max()


def test_zero_and_linearity():
    VX, E = di.kuhn_box(2)
    st = Setup(VX, E, 3)
    assert np.all(rhs(st, np.zeros((6, st.K, st.Np))) == 0)
    u = di.random_fields(st.K, 3, seed=0)
    v = di.random_fields(st.K, 3, seed=1)
    lhs = rhs(st, 2.5 * u - 0.75 * v)
    r = 2.5 * rhs(st, u) - 0.75 * rhs(st, v)
    assert np.abs(lhs - r).max() < 1e-13 * np.abs(r).max()


def test_rhs_exact_for_continuous_polynomial_fields():
    # H = (0, 0, x): continuous, degree 1, tangential-jump free; E = 0.
    # Then all jumps vanish (dH = 0 on PEC walls, dE = -2E = 0), so
    # d_t E = curl H = (0, -1, 0) and d_t H = -curl E = 0 exactly.
    VX, E = di.kuhn_box(2)
    E = di.rotate_local_vertices(E, 1)
    VX = di.jitter_interior(VX, 2, 7)
    st = Setup(VX, E, 2)
    U = np.zeros((6, st.K, st.Np))
    U[5] = st.x
    R = rhs(st, U)
    want = np.zeros_like(R)
    want[1] = -1.0
    assert np.abs(R - want).max() < 1e-11
    # E = (0, 0, x(1-x) y(1-y)) (degree 4, vanishes on x,y walls, normal on z walls):
    # PEC brackets vanish, so d_t H = -curl E = -(dEz/dy, -dEz/dx, 0), d_t E = 0.
    st4 = Setup(VX, E, 4)
    x, y = st4.x, st4.y
    U = np.zeros((6, st4.K, st4.Np))
    U[2] = x * (1 - x) * y * (1 - y)
    R = rhs(st4, U)
    want = np.zeros_like(R)
    want[3] = -(x * (1 - x) * (1 - 2 * y))
    want[4] = (1 - 2 * x) * y * (1 - y)
    assert np.abs(R - want).max() < 1e-11


# ------------------------------------------------------------------ LSERK4
def test_lserk4_coefficients_golden():
    a, b, _ = lserk4_coefficients()
    for name, s, num, den in _golden("lserk4_coefficients.txt"):
        v = int(num) / int(den)
        got = (a if name == "a" else b)[int(s)]
        assert got == v


def _stability_poly_coeffs():
    # R(z) of the 2N-storage scheme computed with exact rational arithmetic from
    # the golden coefficients (independent of the oracle's float loop)
    A = {}
    B = {}
    for name, s, num, den in _golden("lserk4_coefficients.txt"):
        (A if name == "a" else B)[int(s)] = Fraction(int(num), int(den))
    # polynomials in z as coefficient lists
    def add(p, q):
        n = max(len(p), len(q))
        return [(p[i] if i < len(p) else 0) + (q[i] if i < len(q) else 0) for i in range(n)]

    def scal(c, p):
        return [c * v for v in p]

    def shift(p):  # multiply by z
        return [Fraction(0)] + p

    u = [Fraction(1)]
    res = [Fraction(0)]
    for s in range(5):
        res = add(scal(A[s], res), shift(u))      # res = a res + dt*lambda*u  (z = dt*lambda)
        u = add(u, scal(B[s], res))
    return u


def test_lserk4_order_conditions_and_stability_polynomial():
    c = _stability_poly_coeffs()
    for k, want in enumerate([1, 1, Fraction(1, 2), Fraction(1, 6), Fraction(1, 24)]):
        assert abs(float(c[k] - want)) < 1e-13, k        # 4th order (closed form)
    assert abs(float(c[5]) - 0.005) < 1e-6                # z^5/200
    # the oracle's float loop reproduces R(z) on u' = lambda u
    for z in (-0.3, -1.0 + 0.5j, 2.0j):
        got = lserk_integrate(lambda u: z * u, np.array([1.0 + 0j]), 1.0, 1)[0]
        want = sum(float(ck) * z ** k for k, ck in enumerate(c))
        assert abs(got - want) < 1e-13


def test_lserk4_global_order_four():
    errs = []
    for nsteps in (10, 20, 40):
        dt = 1.0 / nsteps
        u = lserk_integrate(lambda u: -u, np.array([1.0]), dt, nsteps)[0]
        errs.append(abs(u - math.exp(-1.0)))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 15.0 < r1 < 17.5 and 15.0 < r2 < 17.5


# ------------------------------------------------------------------ end to end
@pytest.fixture(scope="module")
def c1():
    VX, E = di.kuhn_box(2)
    st = Setup(VX, E, 3)
    U0 = di.cavity_mode_101(st.x, st.y, st.z)
    dt = di.dt_rule(VX, E, 3)
    return st, U0, dt


def test_c1_survey_fingerprints(c1):
    st, U0, dt = c1
    fp = {row[0]: float(row[2]) for row in _golden("survey_fingerprints.txt") if row[0].startswith("c1")}
    R = rhs(st, U0)
    assert abs(np.abs(R).sum() - fp["c1_rhs_abs_sum"]) < 1e-10 * fp["c1_rhs_abs_sum"]
    assert abs(np.abs(R).max() - fp["c1_rhs_abs_max"]) < 1e-10 * fp["c1_rhs_abs_max"]
    energies = []
    U = lserk4(st, U0, dt, 100, callback=lambda s, V: energies.append(energy(st, V)))
    assert abs(U.sum() - fp["c1_100_sum"]) < 1e-10 * abs(fp["c1_100_sum"])
    assert abs(np.abs(U).sum() - fp["c1_100_abs_sum"]) < 1e-10 * fp["c1_100_abs_sum"]
    assert abs(energies[-1] - fp["c1_100_energy"]) < 1e-10
    # upwind energy non-increasing every step
    e = [energy(st, U0)] + energies
    assert all(e[i + 1] <= e[i] * (1 + 1e-12) for i in range(len(e) - 1))
    # and close to the exact mode (PEC cavity eigenmode)
    ex = di.cavity_mode_101(st.x, st.y, st.z, t=100 * dt)
    l2 = math.sqrt(2 * energy(st, U - ex))
    assert l2 < 0.01 and abs(l2 - 5.592e-3) < 1e-6      # 5.592e-3


def test_central_flux_energy_drift_small(c1):
    st, U0, dt = c1
    e0 = energy(st, U0)
    U = lserk4(st, U0, dt, 50, alpha=0.0)
    assert abs(energy(st, U) - e0) / e0 < 1e-6


@pytest.mark.parametrize("N", [2, 3, 4])
def test_h_convergence_to_exact_cavity_mode(N):
    # exact PEC eigenmode (1,1,1) of the unit cube; L2 error ~ h^(N+1)
    T = 0.25
    errs = []
    for n in (1, 2, 4):
        VX, E = di.kuhn_box(n)
        st = Setup(VX, E, N)
        U0 = di.cavity_mode_111(st.x, st.y, st.z)
        dt0 = di.dt_rule(VX, E, N)
        ns = int(math.ceil(T / dt0))
        U = lserk4(st, U0, T / ns, ns)
        ex = di.cavity_mode_111(st.x, st.y, st.z, t=T)
        errs.append(math.sqrt(2 * energy(st, U - ex)))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] >= N + 0.5, (errs, rates)
