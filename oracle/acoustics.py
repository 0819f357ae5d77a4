"""Oracle for the second linear hyperbolic system: linear acoustics (test infrastructure
only; see oracle/__init__.py).  SURVEY §8f NEXT-3: "a second linear hyperbolic system
through the same diff/lift kernels" — PAPER.md:105-115 poses the method for any
u_t + div F(u) = 0 (eq. claw) and lists the systems it covers.

System (reading R16): nondimensional linear acoustics, rho0 = c = 1,
u = (p, vx, vy, vz),

    p_t + div v   = 0,        v_t + grad p = 0,

i.e. F(u) = (v, p I), so n.F(u) = A_n u with A_n = [[0, n^T], [n, 0]] (eigenvalues
+1, -1, 0, 0; |A_n| = [[1, 0], [0, n n^T]]).

Same semi-discrete form as Maxwell, eq. (4), in the same four
stages (fig:dg-subtasks):

1. volume: -div F(u^k) with the per-element chain rule (eq. 6):
   rhs_p = -(d_x vx + d_y vy + d_z vz),  rhs_v = -grad p;
2. flux gather: jumps [[u]] = u+ - u- (reading R1's convention) at every face node
   and the upwind flux (Lax-Friedrichs/Riemann form with the paper's alpha of
   fig:flux-code a, applied to this system):

       n.F* = 1/2 A_n (u- + u+) - alpha/2 |A_n| (u+ - u-)
       2 n.(F - F*) = -A_n [[u]] + alpha |A_n| [[u]]
         p:  -n.[[v]] + alpha [[p]]
         v:  -n [[p]] + alpha n (n.[[v]])

   scaled by Fscale / 2 as for Maxwell;
3. lift (LIFT) and 4. assembly.

Walls (reading R17): rigid (sound-hard) walls v.n = 0, imposed by the mirror state
p+ = p-, v+ = v- - 2 (n.v-) n, the acoustic counterpart of PEC.

Pins: tests/test_oracle_acoustics.py (exact RHS of polynomial fields, skew /
negative-semidefinite dense operator in the M_g inner product, h-convergence to the
exact rigid-wall cavity mode, energy behaviour).
"""
from __future__ import annotations

import numpy as np

from .maxwell import _grad, lserk_integrate
from .mesh import Setup

NFIELDS = 4


def surface_flux(st: Setup, U, alpha: float = 1.0):
    """Stage 2: Fscale * n.(F - F*) / 2 at every face node, [4][K][4 Nfp]."""
    K, Nfp = st.K, st.Nfp
    vM = st.vmapM.reshape(K, 4 * Nfp)
    vP = st.vmapP.reshape(K, 4 * Nfp)
    B = st.mapB.reshape(K, 4 * Nfp)
    nx = np.repeat(st.nx, Nfp, axis=1)
    ny = np.repeat(st.ny, Nfp, axis=1)
    nz = np.repeat(st.nz, Nfp, axis=1)
    flat = [U[c].ravel() for c in range(4)]
    d = [flat[c][vP] - flat[c][vM] for c in range(4)]           # [[u]] = u+ - u-
    # rigid wall: p+ = p-, v+ = v- - 2 (n.v-) n
    ndotv = nx * flat[1][vM] + ny * flat[2][vM] + nz * flat[3][vM]
    d[0][B] = 0.0
    d[1][B] = (-2.0 * ndotv * nx)[B]
    d[2][B] = (-2.0 * ndotv * ny)[B]
    d[3][B] = (-2.0 * ndotv * nz)[B]
    fl = upwind_flux((nx, ny, nz), d[0], d[1:4], alpha)
    Fs = np.repeat(st.Fscale, Nfp, axis=1)
    return np.stack(fl) * (Fs / 2.0)[None]


def upwind_flux(n, dp, dv, alpha: float = 1.0):
    """Pointwise 2 n.(F - F*) = (-A_n + alpha |A_n|) [[u]] for acoustics."""
    nx, ny, nz = n
    dvx, dvy, dvz = dv
    ndotdv = nx * dvx + ny * dvy + nz * dvz
    fp = -ndotdv + alpha * dp
    fvx = -nx * dp + alpha * nx * ndotdv
    fvy = -ny * dp + alpha * ny * ndotdv
    fvz = -nz * dp + alpha * nz * ndotdv
    return fp, fvx, fvy, fvz


def rhs(st: Setup, U, alpha: float = 1.0):
    """d_t u for fields U [4][K][Np] (p, vx, vy, vz)."""
    U = np.asarray(U, dtype=np.float64)
    p, vx, vy, vz = U
    flux = surface_flux(st, U, alpha)                             # stage 2
    px, py, pz = _grad(st, p)                                     # stage 1 (volume)
    div = _grad(st, vx)[0] + _grad(st, vy)[1] + _grad(st, vz)[2]
    LIFT = st.ref.LIFT
    lifted = np.stack([flux[c] @ LIFT.T for c in range(4)])       # stage 3
    return np.stack([-div, -px, -py, -pz]) + lifted               # stage 4


def lserk4(st: Setup, U, dt: float, nsteps: int, alpha: float = 1.0, callback=None):
    """Advance acoustic fields U [4][K][Np] by nsteps LSERK4 steps (same scheme as Maxwell)."""
    return lserk_integrate(lambda V: rhs(st, V, alpha), U, dt, nsteps, callback)


def energy(st: Setup, U):
    """Discrete acoustic energy 1/2 sum_k J_k sum_c u_c^T M u_c."""
    M = st.ref.M
    return 0.5 * sum(np.einsum("k,ki,ij,kj->", st.J, U[c], M, U[c]) for c in range(4))
