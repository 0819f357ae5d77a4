"""Pins of the oracle's reference element against closed forms, invariants and
golden values (not against itself).  CPU only."""
import itertools
import math
import os

import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

from oracle import refelem
from oracle.refelem import build_reference

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ORDERS = list(range(1, 10))


@pytest.fixture(scope="module")
def refs():
    return {N: build_reference(N) for N in ORDERS}


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def test_dims_closed_form(refs):
    # Np = dim P_N(tet) = C(N+3,3), Nfp = C(N+2,2)
    for N, R in refs.items():
        assert R.Np == math.comb(N + 3, 3) and R.Nfp == math.comb(N + 2, 2)
        assert R.r.shape == (R.Np,) and R.LIFT.shape == (R.Np, 4 * R.Nfp)
        assert R.Dr.shape == (R.Np, R.Np)


def test_order_range():
    with pytest.raises(ValueError):
        build_reference(0)
    with pytest.raises(ValueError):
        build_reference(10)


VERTS = np.array([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float)


def test_n1_vertices_n2_midpoints(refs):
    P1 = np.stack([refs[1].r, refs[1].s, refs[1].t], 1)
    assert np.allclose(np.sort(P1, axis=0), np.sort(VERTS, axis=0), atol=1e-14)
    for v in VERTS:
        assert np.min(np.linalg.norm(P1 - v, axis=1)) < 1e-14
    P2 = np.stack([refs[2].r, refs[2].s, refs[2].t], 1)
    want = list(VERTS) + [(VERTS[a] + VERTS[b]) / 2 for a, b in itertools.combinations(range(4), 2)]
    assert P2.shape[0] == 10
    for w in want:
        assert np.min(np.linalg.norm(P2 - w, axis=1)) < 1e-14


def test_edge_nodes_are_gll_closed_form(refs):
    # edge v0-v1 (s = t = -1): the r-coordinates are the GLL points, i.e. the
    # roots of (1-x^2) P_N'(x) -- computed here with numpy's Legendre series and
    # compared with the closed forms stored in golden/gll_points.txt
    gold = {int(r[0]): np.array([float(v) for v in r[1:]]) for r in _golden("gll_points.txt")}
    for N, R in refs.items():
        on = (np.abs(R.s + 1) < 1e-10) & (np.abs(R.t + 1) < 1e-10)
        x = np.sort(R.r[on])
        roots = npleg.Legendre.basis(N).deriv().roots() if N > 1 else np.array([])
        ref = np.sort(np.concatenate([[-1.0, 1.0], np.real(roots)]))
        assert np.allclose(x, ref, atol=1e-13), N
        if N in gold:
            assert np.allclose(x, gold[N], atol=1e-15), N


def _bary(R):
    return np.stack([-(1 + R.r + R.s + R.t) / 2, (1 + R.r) / 2, (1 + R.s) / 2, (1 + R.t) / 2], 1)


def test_node_set_symmetric_under_all_24_vertex_permutations(refs):
    for N, R in refs.items():
        B = _bary(R)
        for p in itertools.permutations(range(4)):
            Bp = B[:, p]
            # every permuted node coincides with some node
            d = np.abs(Bp[:, None, :] - B[None, :, :]).max(axis=2).min(axis=1)
            assert d.max() < 5e-15, (N, p)


def test_edge_node_counts_and_face_counts(refs):
    for N, R in refs.items():
        B = _bary(R)
        nz = (B > 1e-10).sum(axis=1)
        assert (nz == 1).sum() == 4                       # vertices
        assert (nz == 2).sum() == 6 * (N - 1)             # edge interiors
        assert (nz == 3).sum() == 4 * (N - 1) * (N - 2) // 2   # face interiors
        assert R.Fmask.shape == (4, R.Nfp)
        for f, (col, val) in enumerate([(3, 0.0), (2, 0.0), (0, 0.0), (1, 0.0)]):
            assert np.all(np.abs(B[R.Fmask[f], col] - val) < 1e-10)
            assert np.all(np.diff(R.Fmask[f]) > 0)


def test_interpolation_conditioning(refs):
    conds = [np.linalg.cond(refs[N].V) for N in ORDERS]
    assert max(conds) < 100.0


def _monomials(N):
    for a in range(N + 1):
        for b in range(N + 1 - a):
            for c in range(N + 1 - a - b):
                yield a, b, c


def test_D_exact_on_all_monomials(refs):
    for N, R in refs.items():
        r, s, t = R.r, R.s, R.t
        err = 0.0
        for a, b, c in _monomials(N):
            f = r ** a * s ** b * t ** c
            fr = a * r ** max(a - 1, 0) * s ** b * t ** c if a else 0 * r
            fs = b * r ** a * s ** max(b - 1, 0) * t ** c if b else 0 * r
            ft = c * r ** a * s ** b * t ** max(c - 1, 0) if c else 0 * r
            err = max(err, np.abs(R.Dr @ f - fr).max(), np.abs(R.Ds @ f - fs).max(),
                      np.abs(R.Dt @ f - ft).max())
        assert err < 1e-12, (N, err)


def test_D_row_sums_zero_and_corner_entry(refs):
    for N, R in refs.items():
        for D in (R.Dr, R.Ds, R.Dt):
            assert np.abs(D.sum(axis=1)).max() < 1e-12
        # l_0 restricted to edge v0-v1 is the 1-D GLL Lagrange polynomial; its
        # endpoint derivative is -N(N+1)/4 (closed form for GLL)
        assert abs(R.Dr[0, 0] + N * (N + 1) / 4) < 1e-11


def test_mass_volume_and_face_areas(refs):
    for N, R in refs.items():
        one = np.ones(R.Np)
        assert abs(one @ R.M @ one - 4.0 / 3.0) < 1e-12          # |bi-unit tet| = 4/3
        assert np.allclose(R.M, R.M.T, atol=1e-14)
        assert np.linalg.eigvalsh(R.M).min() > 0
        for Mf in R.face_mass:
            o = np.ones(R.Nfp)
            assert abs(o @ Mf @ o - 2.0) < 1e-12                 # reference triangle area 2


def test_mass_integrates_polynomials_exactly(refs):
    # int_tet r^2 dV over the bi-unit tet: with barycentric l1 = (1+r)/2, r = 2 l1 - 1,
    # int l1^a = 6 V a! / (a+3)! with V = 4/3; so int r^2 = 4/3*(4*(2/20) - 4*(1/4) + 1)
    for N, R in refs.items():
        if N < 2:
            continue
        one = np.ones(R.Np)
        val = one @ R.M @ (R.r ** 2)
        V = 4.0 / 3.0
        i1 = 6 * V * 1 / math.factorial(4)        # int l1
        i2 = 6 * V * 2 / math.factorial(5)        # int l1^2
        exact = 4 * i2 - 4 * i1 + V
        assert abs(val - exact) < 1e-12, N


def test_lift_identity_M_L_equals_Emat(refs):
    # fig:lifting-matrix: L = M^-1 [M^{A1} .. M^{A4}] embedded at face rows
    for N, R in refs.items():
        E = np.zeros((R.Np, 4 * R.Nfp))
        for f in range(4):
            E[np.ix_(R.Fmask[f], range(f * R.Nfp, (f + 1) * R.Nfp))] = R.face_mass[f]
        assert np.abs(R.M @ R.LIFT - E).max() < 1e-11 * max(1.0, np.abs(E).max()), N


def test_integration_by_parts_identities(refs):
    # M D + D^T M = sum_faces n_mu dS face mass (closed form per reference normal):
    # r: +face2 - face3;  s: +face2 - face1;  t: +face2 - face0
    for N, R in refs.items():
        def EME(f):
            E = np.zeros((R.Np, R.Np))
            E[np.ix_(R.Fmask[f], R.Fmask[f])] = R.face_mass[f]
            return E
        for D, neg in ((R.Dr, 3), (R.Ds, 1), (R.Dt, 0)):
            lhs = R.M @ D + D.T @ R.M
            rhs = EME(2) - EME(neg)
            assert np.abs(lhs - rhs).max() < 1e-11, (N, neg)


def test_lift_first_entry_pattern(refs):
    # SURVEY.md Appendix B (independent prototype): LIFT[0,0] = 1.5 (N+1)
    for N, R in refs.items():
        assert abs(R.LIFT[0, 0] - 1.5 * (N + 1)) < 1e-10


def test_survey_node_fingerprints(refs):
    for row in _golden("survey_fingerprints.txt"):
        name, N, val = row[0], int(row[1]), float(row[2])
        if name == "sum_r2":
            assert abs((refs[N].r ** 2).sum() - val) < 1e-10 * max(1, abs(val))
        elif name == "sum_rst":
            R = refs[N]
            assert abs((R.r * R.s * R.t).sum() - val) < 1e-10 * max(1, abs(val))


def test_jacobi_orthonormality_by_quadrature():
    # orthonormality of P_n^{(a,b)} w.r.t. (1-x)^a (1+x)^b, checked with numpy's
    # Gauss-Legendre rule (independent of jacobi_gq)
    x, w = npleg.leggauss(40)
    for a, b in ((0, 0), (1, 0), (3, 0), (1, 1)):
        wt = w * (1 - x) ** a * (1 + x) ** b
        P = np.array([refelem.jacobi_p(x, a, b, n) for n in range(7)])
        G = (P * wt) @ P.T
        assert np.abs(G - np.eye(7)).max() < 1e-12


def test_jacobi_gq_integrates_polynomials():
    # Gauss-Jacobi with N+1 points is exact to degree 2N+1 for the Jacobi weight
    x, w = refelem.jacobi_gq(0.0, 0.0, 4)
    for d in range(10):
        exact = (1 - (-1) ** (d + 1)) / (d + 1)
        assert abs((w * x ** d).sum() - exact) < 1e-13
