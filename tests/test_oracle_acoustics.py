"""Pins of the oracle's acoustics operator (oracle/acoustics.py)
against closed forms, brute-force operator properties and an exact solution."""
import math

import numpy as np
import pytest

import dg_inputs as di
from oracle import Setup
from oracle import acoustics as ac


def test_flux_closed_form_and_upwinding():
    # 2 n.(F - F*) = (-A_n + alpha |A_n|) [[u]], A_n = [[0, n^T], [n, 0]], |A_n| = diag(1, n n^T);
    # checked against the explicit 4x4 matrices, and alpha = 1 is the exact Riemann
    # (characteristic) upwinding: the incoming characteristic p - n.v carries u+, the
    # outgoing p + n.v carries u-
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = rng.normal(size=3); n /= np.linalg.norm(n)
        d = rng.normal(size=4)
        An = np.zeros((4, 4)); An[0, 1:] = n; An[1:, 0] = n
        absA = np.zeros((4, 4)); absA[0, 0] = 1.0; absA[1:, 1:] = np.outer(n, n)
        w, V = np.linalg.eigh(An)
        assert np.allclose(V @ np.diag(np.abs(w)) @ V.T, absA, atol=1e-14)
        for alpha in (0.0, 0.5, 1.0):
            got = ac.upwind_flux(tuple(n), d[0], tuple(d[1:]), alpha)
            assert np.allclose(np.array(got), (-An + alpha * absA) @ d, atol=1e-14)
        uM = rng.normal(size=4); uP = rng.normal(size=4)
        # Godunov state: characteristic w+ = p + n.v from the inside, w- = p - n.v from outside
        wp = uM[0] + n @ uM[1:]
        wm = uP[0] - n @ uP[1:]
        ps = 0.5 * (wp + wm)
        vs_n = 0.5 * (wp - wm)
        vt = 0.5 * ((uM[1:] - (n @ uM[1:]) * n) + (uP[1:] - (n @ uP[1:]) * n))  # tangential: no flux anyway
        Fs = np.concatenate([[vs_n], ps * n])      # n.F(u*) = (n.v*, p* n)
        FM = An @ uM
        got = np.array(ac.upwind_flux(tuple(n), uP[0] - uM[0], tuple(uP[1:] - uM[1:]), 1.0))
        assert np.allclose(got, 2.0 * (FM - Fs), atol=1e-13), vt


@pytest.mark.parametrize("N", [2, 3])
def test_exact_rhs_of_polynomial_fields(N):
    # continuous polynomial fields with v.n = 0 on the walls: no jumps, so the DG RHS is
    # the exact -div v, -grad p (degree <= N, represented exactly)
    VX, E = di.kuhn_box(2)
    E, _ = di.shuffle_elements(E, 2)
    E = di.rotate_local_vertices(E, 3)
    VX = di.jitter_interior(VX, 2, 4)
    st = Setup(VX, E, N)
    x, y, z = st.x, st.y, st.z
    p = x * x * y + z if N >= 3 else x * y + z
    U = np.stack([p, x * (1 - x), y * (1 - y), z * (1 - z)])
    R = ac.rhs(st, U)
    want_p = -(3.0 - 2 * x - 2 * y - 2 * z)
    if N >= 3:
        want_v = [-2 * x * y, -x * x, -np.ones_like(x)]
    else:
        want_v = [-y, -x, -np.ones_like(x)]
    assert np.abs(R[0] - want_p).max() < 1e-11
    for c in range(3):
        assert np.abs(R[1 + c] - want_v[c]).max() < 1e-11
    # constant pressure at rest is steady (wall mirror keeps [[u]] = 0)
    C = np.stack([np.full_like(x, 2.5), 0 * x, 0 * x, 0 * x])
    assert np.abs(ac.rhs(st, C)).max() < 1e-12


def _dense(st, alpha):
    K, Np = st.K, st.Np
    n = 4 * K * Np
    A = np.zeros((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        A[:, j] = ac.rhs(st, e.reshape(4, K, Np), alpha).ravel()
        e[j] = 0.0
    Mg = np.kron(np.eye(4), np.kron(np.diag(st.J), st.ref.M))
    return A, Mg


@pytest.mark.parametrize("N", [1, 2])
def test_operator_skew_central_dissipative_upwind(N):
    VX, E = di.kuhn_box(1)
    E = di.rotate_local_vertices(E, 5)
    st = Setup(VX, E, N)
    A0, Mg = _dense(st, 0.0)
    S = Mg @ A0
    assert np.abs(S + S.T).max() < 1e-13 * np.abs(S).max()
    A1, _ = _dense(st, 1.0)
    S1 = Mg @ A1
    ev = np.linalg.eigvalsh(0.5 * (S1 + S1.T))
    assert ev.max() < 1e-13 * np.abs(S1).max() and ev.min() < -1e-3


@pytest.mark.parametrize("N", [2, 3])
def test_h_convergence_to_exact_rigid_wall_mode(N):
    T = 0.25
    errs = []
    for n in (1, 2, 4):
        VX, E = di.kuhn_box(n)
        st = Setup(VX, E, N)
        U0 = di.acoustic_mode(st.x, st.y, st.z, lmn=(1, 1, 1))
        dt0 = di.dt_rule(VX, E, N)
        ns = int(math.ceil(T / dt0))
        U = ac.lserk4(st, U0, T / ns, ns)
        ex = di.acoustic_mode(st.x, st.y, st.z, t=T, lmn=(1, 1, 1))
        errs.append(math.sqrt(2 * ac.energy(st, U - ex)))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] >= N + 0.5, (errs, rates)


def test_energy_central_conserved_upwind_dissipates():
    VX, E = di.kuhn_box(2)
    E, _ = di.shuffle_elements(E, 6)
    st = Setup(VX, E, 3)
    U0 = di.random_fields(st.K, 3, seed=4, nfields=4)
    dt = di.dt_rule(VX, E, 3)
    e0 = ac.energy(st, U0)
    assert abs(ac.energy(st, ac.lserk4(st, U0, dt, 30, alpha=0.0)) - e0) / e0 < 1e-5
    es = []
    ac.lserk4(st, U0, dt, 30, alpha=1.0, callback=lambda s, V: es.append(ac.energy(st, V)))
    assert all(b <= a * (1 + 1e-14) for a, b in zip([e0] + es, es)) and es[-1] < 0.8 * e0
