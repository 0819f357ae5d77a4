"""Oracle Maxwell operator and LSERK4 (test infrastructure only; see oracle/__init__.py).

Semi-discrete DG operator, eq. (4) of PAPER.md:157-169:

    d_t u^k = - sum_nu D^{k,d nu}[F(u^k)] + L^k [ n.F - (n.F)^* ]|_{A subset dD_k}

for Maxwell in vacuum, eps = mu = 1 (reading R3):  d_t E = curl H,
d_t H = -curl E.  The four stages of fig:dg-subtasks are
written out in the paper's order:

1. F(u) + local differentiation (volume): ur = Dr u, us = Ds u, ut = Dt u per
   element, chain rule with the per-element affine factors (eq. 6),
   then the curl.
2. flux gather (eq. 5): traces u- = u[vmapM], u+ = u[vmapP]
   picked from the volume nodes; PEC walls E+ = -E-, H+ = H-
   (reading R4); the Maxwell upwind flux of fig:flux-code a

       n.(F - F*)_E = 1/2 [ n x ( [[H]] - alpha n x [[E]] ) ]

   with [[u]] = u+ - u- (reading R1) and its H counterpart (reading R2)

       n.(F - F*)_H = 1/2 [ -n x ( [[E]] + alpha n x [[H]] ) ]

   each scaled by Fscale = sJ/J.
3. flux lifting: LIFT applied to the face buffer.
4. assembly: rhs = volume term + lifted flux.

LSERK4: the 5-stage, 2N-storage Carpenter-Kennedy scheme (reading R5; "RK4
time stepping" PAPER.md:1179-1181), coefficients as in HW:

    res <- a_s res + dt rhs(u);   u <- u + b_s res,     s = 0..4.
"""
from __future__ import annotations

import numpy as np

from .mesh import Setup


def lserk4_coefficients():
    """(a, b, c) of the (5,4) low-storage RK of Carpenter & Kennedy, as tabulated in HW."""
    a = np.array([0.0,
                  -567301805773.0 / 1357537059087.0,
                  -2404267990393.0 / 2016746695238.0,
                  -3550918686646.0 / 2091501179385.0,
                  -1275806237668.0 / 842570457699.0])
    b = np.array([1432997174477.0 / 9575080441755.0,
                  5161836677717.0 / 13612068292357.0,
                  1720146321549.0 / 2090206949498.0,
                  3134564353537.0 / 4481467310338.0,
                  2277821191437.0 / 14882151754819.0])
    c = np.array([0.0,
                  1432997174477.0 / 9575080441755.0,
                  2526269341429.0 / 6820363962896.0,
                  2006345519317.0 / 3224310063776.0,
                  2802321613138.0 / 2924317926251.0])
    return a, b, c


def _grad(st: Setup, u):
    """Physical gradient of a scalar nodal field u [K][Np] (eq. 6 chain rule)."""
    ref = st.ref
    ur = u @ ref.Dr.T
    us = u @ ref.Ds.T
    ut = u @ ref.Dt.T
    ux = st.rx[:, None] * ur + st.sx[:, None] * us + st.tx[:, None] * ut
    uy = st.ry[:, None] * ur + st.sy[:, None] * us + st.ty[:, None] * ut
    uz = st.rz[:, None] * ur + st.sz[:, None] * us + st.tz[:, None] * ut
    return ux, uy, uz


def curl(st: Setup, ux, uy, uz):
    """curl of a nodal vector field (HW Curl3D)."""
    _, uxy, uxz = _grad(st, ux)
    uyx, _, uyz = _grad(st, uy)
    uzx, uzy, _ = _grad(st, uz)
    return uzy - uyz, uxz - uzx, uyx - uxy


def surface_flux(st: Setup, U, alpha: float = 1.0):
    """Stage 2 (flux gather): Fscale * n.(F - F*) / 2 at every face node, [6][K][4 Nfp]."""
    K, Nfp = st.K, st.Nfp
    vM = st.vmapM.reshape(K, 4 * Nfp)
    vP = st.vmapP.reshape(K, 4 * Nfp)
    B = st.mapB.reshape(K, 4 * Nfp)
    flat = [U[c].ravel() for c in range(6)]
    d = [flat[c][vP] - flat[c][vM] for c in range(6)]          # [[u]] = u+ - u-
    # PEC: E+ = -E-, H+ = H-
    for c in range(3):
        d[c][B] = -2.0 * flat[c][vM][B]
    for c in range(3, 6):
        d[c][B] = 0.0
    nx = np.repeat(st.nx, Nfp, axis=1)
    ny = np.repeat(st.ny, Nfp, axis=1)
    nz = np.repeat(st.nz, Nfp, axis=1)
    Fs = np.repeat(st.Fscale, Nfp, axis=1)
    fl = upwind_flux((nx, ny, nz), d[0:3], d[3:6], alpha)
    return np.stack(fl) * (Fs / 2.0)[None]


def upwind_flux(n, dE, dH, alpha: float = 1.0):
    """Pointwise 2 n.(F - F*) for Maxwell (fig:flux-code a), jumps d = u+ - u-:

        fluxE =  n x dH + alpha (dE - (n.dE) n)      [= n x (dH - alpha n x dE)]
        fluxH = -n x dE + alpha (dH - (n.dH) n)      [= -n x (dE + alpha n x dH)]

    Returns (fluxEx, fluxEy, fluxEz, fluxHx, fluxHy, fluxHz); the caller halves and scales by Fscale."""
    nx, ny, nz = n
    dEx, dEy, dEz = dE
    dHx, dHy, dHz = dH
    ndotdH = nx * dHx + ny * dHy + nz * dHz
    ndotdE = nx * dEx + ny * dEy + nz * dEz
    fluxEx = (ny * dHz - nz * dHy) + alpha * (dEx - ndotdE * nx)
    fluxEy = (nz * dHx - nx * dHz) + alpha * (dEy - ndotdE * ny)
    fluxEz = (nx * dHy - ny * dHx) + alpha * (dEz - ndotdE * nz)
    fluxHx = -(ny * dEz - nz * dEy) + alpha * (dHx - ndotdH * nx)
    fluxHy = -(nz * dEx - nx * dEz) + alpha * (dHy - ndotdH * ny)
    fluxHz = -(nx * dEy - ny * dEx) + alpha * (dHz - ndotdH * nz)
    return fluxEx, fluxEy, fluxEz, fluxHx, fluxHy, fluxHz


def rhs(st: Setup, U, alpha: float = 1.0):
    """d_t u for fields U [6][K][Np] (Ex,Ey,Ez,Hx,Hy,Hz), eq. (4)."""
    U = np.asarray(U, dtype=np.float64)
    Ex, Ey, Ez, Hx, Hy, Hz = U
    flux = surface_flux(st, U, alpha)                    # stage 2
    cHx, cHy, cHz = curl(st, Hx, Hy, Hz)                 # stage 1 (volume)
    cEx, cEy, cEz = curl(st, Ex, Ey, Ez)
    LIFT = st.ref.LIFT
    lifted = np.stack([flux[c] @ LIFT.T for c in range(6)])   # stage 3
    return np.stack([cHx, cHy, cHz, -cEx, -cEy, -cEz]) + lifted   # stage 4


def lserk_integrate(f, U, dt: float, nsteps: int, callback=None):
    """Generic 2N-storage LSERK4 loop for u' = f(u): res <- a_s res + dt f(u); u <- u + b_s res."""
    a, b, _ = lserk4_coefficients()
    U = np.array(U, dtype=np.result_type(U, np.float64), copy=True)
    res = np.zeros_like(U)
    for step in range(nsteps):
        for s in range(5):
            R = f(U)
            res = a[s] * res + dt * R
            U = U + b[s] * res
        if callback is not None:
            callback(step, U)
    return U


def lserk4(st: Setup, U, dt: float, nsteps: int, alpha: float = 1.0, callback=None):
    """Advance fields U [6][K][Np] by nsteps LSERK4 steps of size dt; res starts at zero (a_0 = 0)."""
    return lserk_integrate(lambda V: rhs(st, V, alpha), U, dt, nsteps, callback)


def energy(st: Setup, U):
    """Discrete EM energy 1/2 sum_k J_k sum_c u_c^T M u_c (M = reference mass, eq. 6a)."""
    M = st.ref.M
    e = 0.0
    for c in range(6):
        e += np.einsum("k,ki,ij,kj->", st.J, U[c], M, U[c])
    return 0.5 * e
