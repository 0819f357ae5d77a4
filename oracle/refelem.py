"""Oracle reference element (test infrastructure only; see oracle/__init__.py).

Follows, step by step and in HW's notation, the construction the paper cites
but does not reproduce:

* nodes: "a set of interpolation nodes [warburton_explicit_2006]"
  -> HW Nodes3D (warp & blend) with HW's alpha_opt table (reading R6);
* V, Vr, Vs, Vt: generalized Vandermonde of the orthonormal Dubiner basis (HW
  Vandermonde3D / GradVandermonde3D);
* M = (V V^T)^-1, S = M Dr, D^{d mu} = M^-1 S^{d mu}  (eq. 3a-3c);
* face mass M^A (eq. 3d) via the 2-D Dubiner Vandermonde of each face;
* LIFT = M^-1 [M^{A1} ... M^{A4}] embedded at the face rows (PAPER.md:170-216,
  fig:lifting-matrix), computed as HW's  LIFT = V (V^T Emat).

Reference tet: vertices v0=(-1,-1,-1), v1=(1,-1,-1), v2=(-1,1,-1), v3=(-1,-1,1).
Faces (0-based): 0: t=-1 (v0 v1 v2), 1: s=-1 (v0 v1 v3), 2: r+s+t=-1 (v1 v2 v3),
3: r=-1 (v0 v2 v3)  (HW Fmask order; reading R7).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

NODETOL = 1e-10

# HW Nodes3D alpha_opt for N = 1..15 (we use 1..9); reading R6.
ALPHA_OPT = [0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577, 1.1603,
             1.10153, 0.6080, 0.4523, 0.8856, 0.8717, 0.9655]


# ----------------------------------------------------------------------------- 1-D
def jacobi_p(x, alpha: float, beta: float, n: int):
    """Orthonormal Jacobi polynomial P_n^{(alpha,beta)}(x) on [-1,1] (HW JacobiP, Appendix A.1)."""
    x = np.asarray(x, dtype=np.float64)
    PL = np.zeros((n + 1,) + x.shape)
    gamma0 = (2.0 ** (alpha + beta + 1) / (alpha + beta + 1)
              * math.gamma(alpha + 1) * math.gamma(beta + 1) / math.gamma(alpha + beta + 1))
    PL[0] = 1.0 / math.sqrt(gamma0)
    if n == 0:
        return PL[0]
    gamma1 = (alpha + 1) * (beta + 1) / (alpha + beta + 3) * gamma0
    PL[1] = ((alpha + beta + 2) * x / 2 + (alpha - beta) / 2) / math.sqrt(gamma1)
    if n == 1:
        return PL[1]
    aold = 2.0 / (2 + alpha + beta) * math.sqrt((alpha + 1) * (beta + 1) / (alpha + beta + 3))
    for i in range(1, n):
        h1 = 2 * i + alpha + beta
        anew = 2.0 / (h1 + 2) * math.sqrt((i + 1) * (i + 1 + alpha + beta) * (i + 1 + alpha)
                                          * (i + 1 + beta) / (h1 + 1) / (h1 + 3))
        bnew = -(alpha * alpha - beta * beta) / h1 / (h1 + 2)
        PL[i + 1] = 1.0 / anew * (-aold * PL[i - 1] + (x - bnew) * PL[i])
        aold = anew
    return PL[n]


def grad_jacobi_p(x, alpha: float, beta: float, n: int):
    """d/dx P_n^{(alpha,beta)} = sqrt(n(n+alpha+beta+1)) P_{n-1}^{(alpha+1,beta+1)} (HW GradJacobiP)."""
    x = np.asarray(x, dtype=np.float64)
    if n == 0:
        return np.zeros_like(x)
    return math.sqrt(n * (n + alpha + beta + 1)) * jacobi_p(x, alpha + 1, beta + 1, n - 1)


def jacobi_gq(alpha: float, beta: float, N: int):
    """Gauss-Jacobi quadrature of order N (N+1 points) by Golub-Welsch (HW JacobiGQ)."""
    if N == 0:
        return np.array([-(alpha - beta) / (alpha + beta + 2)]), np.array([2.0])
    h1 = 2 * np.arange(N + 1) + alpha + beta
    with np.errstate(divide="ignore", invalid="ignore"):
        main = -0.5 * (alpha ** 2 - beta ** 2) / (h1 + 2) / h1
    ii = np.arange(1, N + 1)
    off = (2.0 / (h1[:N] + 2) * np.sqrt(ii * (ii + alpha + beta) * (ii + alpha) * (ii + beta)
                                        / (h1[:N] + 1) / (h1[:N] + 3)))
    if alpha + beta < 10 * np.finfo(float).eps:
        main[0] = 0.0
    J = np.diag(main) + np.diag(off, 1) + np.diag(off, -1)
    x, V = np.linalg.eigh(J)
    w = V[0, :] ** 2 * 2 ** (alpha + beta + 1) / (alpha + beta + 1) \
        * math.gamma(alpha + 1) * math.gamma(beta + 1) / math.gamma(alpha + beta + 1)
    return x, w


def jacobi_gl(alpha: float, beta: float, N: int):
    """Gauss-Lobatto-Jacobi points [-1, GQ(alpha+1,beta+1,N-2), 1] (HW JacobiGL)."""
    if N == 1:
        return np.array([-1.0, 1.0])
    xint, _ = jacobi_gq(alpha + 1, beta + 1, N - 2)
    return np.concatenate([[-1.0], xint, [1.0]])


# ------------------------------------------------------------------ warp & blend
def warp_factor(N: int, rout):
    """1-D warp: sum_i (x_i^GLL - x_i^eq) l_i^eq(r) / (1 - r^2)  (HW evalwarp)."""
    rout = np.asarray(rout, dtype=np.float64)
    xeq = np.array([-1.0 + 2.0 * (N - i) / N for i in range(N + 1)])  # +1 ... -1 (HW order)
    xgll = -jacobi_gl(0.0, 0.0, N)                                      # +1 ... -1
    warp = np.zeros_like(rout)
    for i in range(N + 1):
        d = np.full_like(rout, xgll[i] - xeq[i])
        for j in range(1, N):
            if i != j:
                d = d * (rout - xeq[j]) / (xeq[i] - xeq[j])
        if i != 0:
            d = -d / (xeq[i] - xeq[0])
        if i != N:
            d = d / (xeq[i] - xeq[N])
        warp = warp + d
    return warp


def eval_shift(N: int, pval: float, L1, L2, L3):
    """Warp & blend shift in the equilateral triangle (HW evalshift)."""
    blend1 = L2 * L3
    blend2 = L1 * L3
    blend3 = L1 * L2
    warpfactor1 = 4 * warp_factor(N, L3 - L2)
    warpfactor2 = 4 * warp_factor(N, L1 - L3)
    warpfactor3 = 4 * warp_factor(N, L2 - L1)
    warp1 = blend1 * warpfactor1 * (1 + (pval * L1) ** 2)
    warp2 = blend2 * warpfactor2 * (1 + (pval * L2) ** 2)
    warp3 = blend3 * warpfactor3 * (1 + (pval * L3) ** 2)
    dx = 1 * warp1 + math.cos(2 * math.pi / 3) * warp2 + math.cos(4 * math.pi / 3) * warp3
    dy = 0 * warp1 + math.sin(2 * math.pi / 3) * warp2 + math.sin(4 * math.pi / 3) * warp3
    return dx, dy


def equi_nodes_3d(N: int):
    """Equidistant lattice on the reference tet, r fastest, then s, then t (HW EquiNodes3D)."""
    r, s, t = [], [], []
    for l in range(N + 1):
        for m in range(N + 1 - l):
            for q in range(N + 1 - l - m):
                r.append(-1 + 2.0 * q / N)
                s.append(-1 + 2.0 * m / N)
                t.append(-1 + 2.0 * l / N)
    return np.array(r), np.array(s), np.array(t)


def nodes_3d(N: int):
    """Warp & blend nodes on the equilateral tet (HW Nodes3D).  Returns X, Y, Z.

    Interior / face-interior positions for N >= 4 are parity unpinned beyond
    invariants (GLL edges, 24-fold symmetry, vertex/midpoint cases, Appendix B
    fingerprints); see DESIGN.md."""
    alpha = ALPHA_OPT[N - 1] if N <= 15 else 1.0
    tol = 1e-10
    r, s, t = equi_nodes_3d(N)
    L1 = (1 + t) / 2
    L2 = (1 + s) / 2
    L3 = -(1 + r + s + t) / 2
    L4 = (1 + r) / 2
    v1 = np.array([-1.0, -1 / math.sqrt(3), -1 / math.sqrt(6)])
    v2 = np.array([1.0, -1 / math.sqrt(3), -1 / math.sqrt(6)])
    v3 = np.array([0.0, 2 / math.sqrt(3), -1 / math.sqrt(6)])
    v4 = np.array([0.0, 0.0, 3 / math.sqrt(6)])
    t1 = np.array([v2 - v1, v2 - v1, v3 - v2, v3 - v1])
    t2 = np.array([v3 - 0.5 * (v1 + v2), v4 - 0.5 * (v1 + v2), v4 - 0.5 * (v2 + v3), v4 - 0.5 * (v1 + v3)])
    for f in range(4):
        t1[f] /= np.linalg.norm(t1[f])
        t2[f] /= np.linalg.norm(t2[f])
    XYZ = np.outer(L3, v1) + np.outer(L4, v2) + np.outer(L2, v3) + np.outer(L1, v4)
    shift = np.zeros_like(XYZ)
    for face in range(4):
        if face == 0:
            La, Lb, Lc, Ld = L1, L2, L3, L4
        elif face == 1:
            La, Lb, Lc, Ld = L2, L1, L3, L4
        elif face == 2:
            La, Lb, Lc, Ld = L3, L1, L4, L2
        else:
            La, Lb, Lc, Ld = L4, L1, L3, L2
        warp1, warp2 = eval_shift(N, alpha, Lb, Lc, Ld)   # HW WarpShiftFace3D
        blend = Lb * Lc * Ld
        denom = (Lb + 0.5 * La) * (Lc + 0.5 * La) * (Ld + 0.5 * La)
        ids = denom > tol
        blend[ids] = (1 + (alpha * La[ids]) ** 2) * blend[ids] / denom[ids]
        shift = shift + np.outer(blend * warp1, t1[face]) + np.outer(blend * warp2, t2[face])
        ids = (La < tol) & (((Lb > tol).astype(int) + (Lc > tol).astype(int) + (Ld > tol).astype(int)) < 3)
        shift[ids] = np.outer(warp1[ids], t1[face]) + np.outer(warp2[ids], t2[face])
    XYZ = XYZ + shift
    return XYZ[:, 0], XYZ[:, 1], XYZ[:, 2]


def xyz_to_rst(X, Y, Z):
    """Equilateral -> bi-unit reference tet (HW xyztorst)."""
    v1 = np.array([-1.0, -1 / math.sqrt(3), -1 / math.sqrt(6)])
    v2 = np.array([1.0, -1 / math.sqrt(3), -1 / math.sqrt(6)])
    v3 = np.array([0.0, 2 / math.sqrt(3), -1 / math.sqrt(6)])
    v4 = np.array([0.0, 0.0, 3 / math.sqrt(6)])
    rhs = np.stack([X, Y, Z]) - 0.5 * (v2 + v3 + v4 - v1)[:, None]
    A = np.column_stack([0.5 * (v2 - v1), 0.5 * (v3 - v1), 0.5 * (v4 - v1)])
    RST = np.linalg.solve(A, rhs)
    return RST[0], RST[1], RST[2]


# ------------------------------------------------------------- Dubiner basis 3-D
def rst_to_abc(r, s, t):
    """Collapsed coordinates (HW rsttoabc)."""
    Np = len(r)
    a = np.zeros(Np); b = np.zeros(Np)
    for n in range(Np):
        a[n] = 2 * (1 + r[n]) / (-s[n] - t[n]) - 1 if (s[n] + t[n]) != 0 else -1.0
        b[n] = 2 * (1 + s[n]) / (1 - t[n]) - 1 if t[n] != 1 else -1.0
    return a, b, np.array(t, dtype=np.float64)


def simplex_3d_p(a, b, c, i, j, k):
    """Orthonormal Dubiner polynomial psi_ijk (HW Simplex3DP)."""
    h1 = jacobi_p(a, 0, 0, i)
    h2 = jacobi_p(b, 2 * i + 1, 0, j)
    h3 = jacobi_p(c, 2 * (i + j) + 2, 0, k)
    return 2 * math.sqrt(2) * h1 * h2 * ((1 - b) ** i) * h3 * ((1 - c) ** (i + j))


def grad_simplex_3d_p(a, b, c, id_, jd, kd):
    """Gradient of psi_ijk w.r.t. (r,s,t) (HW GradSimplex3DP)."""
    fa = jacobi_p(a, 0, 0, id_); dfa = grad_jacobi_p(a, 0, 0, id_)
    gb = jacobi_p(b, 2 * id_ + 1, 0, jd); dgb = grad_jacobi_p(b, 2 * id_ + 1, 0, jd)
    hc = jacobi_p(c, 2 * (id_ + jd) + 2, 0, kd); dhc = grad_jacobi_p(c, 2 * (id_ + jd) + 2, 0, kd)
    V3Dr = dfa * (gb * hc)
    if id_ > 0:
        V3Dr = V3Dr * ((0.5 * (1 - b)) ** (id_ - 1))
    if id_ + jd > 0:
        V3Dr = V3Dr * ((0.5 * (1 - c)) ** (id_ + jd - 1))
    V3Ds = 0.5 * (1 + a) * V3Dr
    tmp = dgb * ((0.5 * (1 - b)) ** id_)
    if id_ > 0:
        tmp = tmp + (-0.5 * id_) * (gb * (0.5 * (1 - b)) ** (id_ - 1))
    if id_ + jd > 0:
        tmp = tmp * ((0.5 * (1 - c)) ** (id_ + jd - 1))
    tmp = fa * (tmp * hc)
    V3Ds = V3Ds + tmp
    V3Dt = 0.5 * (1 + a) * V3Dr + 0.5 * (1 + b) * tmp
    tmp = dhc * ((0.5 * (1 - c)) ** (id_ + jd))
    if id_ + jd > 0:
        tmp = tmp - 0.5 * (id_ + jd) * (hc * ((0.5 * (1 - c)) ** (id_ + jd - 1)))
    tmp = fa * (gb * tmp)
    tmp = tmp * ((0.5 * (1 - b)) ** id_)
    V3Dt = V3Dt + tmp
    scale = 2 ** (2 * id_ + jd + 1.5)
    return V3Dr * scale, V3Ds * scale, V3Dt * scale


def vandermonde_3d(N, r, s, t):
    """V_ij = psi_j(x_i), modes ordered i, then j, then k (HW Vandermonde3D)."""
    a, b, c = rst_to_abc(r, s, t)
    cols = []
    for i in range(N + 1):
        for j in range(N + 1 - i):
            for k in range(N + 1 - i - j):
                cols.append(simplex_3d_p(a, b, c, i, j, k))
    return np.column_stack(cols)


def grad_vandermonde_3d(N, r, s, t):
    """Vr, Vs, Vt (HW GradVandermonde3D)."""
    a, b, c = rst_to_abc(r, s, t)
    cr, cs, ct = [], [], []
    for i in range(N + 1):
        for j in range(N + 1 - i):
            for k in range(N + 1 - i - j):
                dr, ds, dt = grad_simplex_3d_p(a, b, c, i, j, k)
                cr.append(dr); cs.append(ds); ct.append(dt)
    return np.column_stack(cr), np.column_stack(cs), np.column_stack(ct)


# ------------------------------------------------------------- Dubiner basis 2-D
def rs_to_ab(r, s):
    """Collapsed triangle coordinates (HW rstoab)."""
    a = np.zeros(len(r))
    for n in range(len(r)):
        a[n] = 2 * (1 + r[n]) / (1 - s[n]) - 1 if s[n] != 1 else -1.0
    return a, np.array(s, dtype=np.float64)


def simplex_2d_p(a, b, i, j):
    """Orthonormal triangle polynomial (HW Simplex2DP)."""
    h1 = jacobi_p(a, 0, 0, i)
    h2 = jacobi_p(b, 2 * i + 1, 0, j)
    return math.sqrt(2.0) * h1 * h2 * (1 - b) ** i


def vandermonde_2d(N, r, s):
    """2-D Vandermonde (HW Vandermonde2D)."""
    a, b = rs_to_ab(r, s)
    cols = []
    for i in range(N + 1):
        for j in range(N + 1 - i):
            cols.append(simplex_2d_p(a, b, i, j))
    return np.column_stack(cols)


# ------------------------------------------------------------------- element
@dataclass
class RefElement:
    N: int
    Np: int
    Nfp: int
    r: np.ndarray
    s: np.ndarray
    t: np.ndarray
    V: np.ndarray
    Dr: np.ndarray
    Ds: np.ndarray
    Dt: np.ndarray
    M: np.ndarray
    Fmask: np.ndarray      # [4][Nfp]
    face_mass: list        # 4 x [Nfp][Nfp], in face-parameter coordinates
    Emat: np.ndarray       # [Np][4 Nfp]
    LIFT: np.ndarray       # [Np][4 Nfp]


def face_coordinates(ref_r, ref_s, ref_t, Fmask, f):
    """Face-parameter coordinates of face f's nodes: (r,s), (r,t), (s,t), (s,t) (HW Lift3D)."""
    ids = Fmask[f]
    if f == 0:
        return ref_r[ids], ref_s[ids]
    if f == 1:
        return ref_r[ids], ref_t[ids]
    return ref_s[ids], ref_t[ids]


def build_reference(N: int) -> RefElement:
    """Reference element of order N (HW StartUp3D / Lift3D)."""
    if not (1 <= N <= 9):
        raise ValueError("order N must be in 1..9")
    Np = (N + 1) * (N + 2) * (N + 3) // 6
    Nfp = (N + 1) * (N + 2) // 2
    X, Y, Z = nodes_3d(N)
    r, s, t = xyz_to_rst(X, Y, Z)
    V = vandermonde_3d(N, r, s, t)
    Vr, Vs, Vt = grad_vandermonde_3d(N, r, s, t)
    Vinv = np.linalg.inv(V)
    Dr = Vr @ Vinv
    Ds = Vs @ Vinv
    Dt = Vt @ Vinv
    M = np.linalg.inv(V @ V.T)
    Fmask = np.array([
        np.nonzero(np.abs(1 + t) < NODETOL)[0],
        np.nonzero(np.abs(1 + s) < NODETOL)[0],
        np.nonzero(np.abs(1 + r + s + t) < NODETOL)[0],
        np.nonzero(np.abs(1 + r) < NODETOL)[0],
    ])
    assert Fmask.shape == (4, Nfp)
    Emat = np.zeros((Np, 4 * Nfp))
    face_mass = []
    for f in range(4):
        fr, fs = face_coordinates(r, s, t, Fmask, f)
        VFace = vandermonde_2d(N, fr, fs)
        massFace = np.linalg.inv(VFace @ VFace.T)
        face_mass.append(massFace)
        Emat[np.ix_(Fmask[f], np.arange(f * Nfp, (f + 1) * Nfp))] += massFace
    LIFT = V @ (V.T @ Emat)
    return RefElement(N, Np, Nfp, r, s, t, V, Dr, Ds, Dt, M, Fmask, face_mass, Emat, LIFT)
