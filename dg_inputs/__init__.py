"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

This module holds NONE of the DG method's arithmetic (no nodes, no operators, no
flux, no time stepping).  It only produces *inputs*: tetrahedral box meshes,
element/vertex permutations, vertex jitter, seeded random field arrays, the
closed-form PEC cavity eigenmodes used as initial data / exact solutions, and
the harness's time-step rule.  Both `oracle/` and the `paper_1211_0582_b200`
binding consume these; neither is imported from here.

Recipes (stated again in DESIGN.md §"Input recipe"):

* Kuhn box mesh: the box [0,L]^3 split into n^3 cubes,
  each cube into the 6 "Kuhn" tetrahedra (one per permutation of the axes), all
  positively oriented, conforming.  The paper's meshes are "large 3D Maxwell
  problem" meshes that it does not specify; this is the
  stand-in (reading R9).
* `shuffle_elements`: seeded random element permutation (emulates the poor
  locality of an unstructured mesh numbering).
* `rotate_local_vertices`: a seeded *even* permutation of each tet's 4 local
  vertices (keeps the orientation positive, exercises every face-node
  orientation in the trace gather).
* `jitter_interior`: seeded uniform displacement of interior vertices by at most
  0.1*h per coordinate, so elements are no longer congruent (geometry varies).
* `random_fields`: U(-1,1) fields of shape [6][K][Np] (component-major, the
  C-ABI host layout).
* `cavity_mode_101`, `cavity_mode_111`: exact PEC eigenmodes of the unit cube
  (SURVEY.md Appendix A.9), eps = mu = 1.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "np_of", "nfp_of", "kuhn_box", "shuffle_elements", "rotate_local_vertices",
    "jitter_interior", "random_fields", "cavity_mode_101", "cavity_mode_111",
    "dt_rule", "FIELD_NAMES",
]

FIELD_NAMES = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")

# The 12 even permutations of (0,1,2,3): applying one to a tet's vertex list
# keeps the sign of its volume.
_EVEN_PERMS = np.array([
    (0, 1, 2, 3), (0, 2, 3, 1), (0, 3, 1, 2),
    (1, 0, 3, 2), (1, 2, 0, 3), (1, 3, 2, 0),
    (2, 0, 1, 3), (2, 1, 3, 0), (2, 3, 0, 1),
    (3, 0, 2, 1), (3, 1, 0, 2), (3, 2, 1, 0),
], dtype=np.int64)


def np_of(N: int) -> int:
    """Np = dim P_N on a tetrahedron."""
    return (N + 1) * (N + 2) * (N + 3) // 6


def nfp_of(N: int) -> int:
    """Nfp = dim P_N on a triangle face."""
    return (N + 1) * (N + 2) // 2


def _signed_volume6(VX, tet):
    a, b, c, d = (VX[v] for v in tet)
    return float(np.dot(b - a, np.cross(c - a, d - a)))


def kuhn_box(n: int, L: float = 1.0, nz: int | None = None):
    """Kuhn box mesh of [0,L]^2 x [0, L*nz/n]: returns (VX [nv][3] float64, EToV [K][4] int64),
    K = 6 n^2 nz (nz defaults to n: the cube [0,L]^3).

    Vertex id(i,j,k) = i + (n+1)(j + (n+1)k); cells ordered k, j, i (i fastest);
    each cell emits one tet per axis permutation p (lexicographic order), with
    vertices origin, +e_p0, +e_p0+e_p1, +e_p0+e_p1+e_p2; a negative signed
    volume swaps the last two vertices.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    nz = n if nz is None else nz
    m = n + 1
    idx = np.arange(m)
    kk, jj, ii = np.meshgrid(np.arange(nz + 1), idx, idx, indexing="ij")
    VX = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.float64) * (L / n)
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    step = (1, m, m * m)
    # orientation of each permutation's tet is cell-independent: fix it once
    proto = []
    for p in perms:
        o = 0
        t = [o]
        for ax in p:
            o += step[ax]
            t.append(o)
        if _signed_volume6(VX, t) < 0:
            t[2], t[3] = t[3], t[2]
        proto.append(t)
    proto = np.array(proto, dtype=np.int64)  # [6][4] relative to the cell-origin vertex
    # cells ordered k, j, i with i fastest
    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(n), np.arange(n), indexing="ij")
    origin = (ci + m * (cj + m * ck)).ravel()
    EToV = (origin[:, None, None] + proto[None, :, :]).reshape(-1, 4)
    return VX, EToV.astype(np.int64)


def shuffle_elements(EToV, seed: int):
    """Seeded random permutation of the element order.  Returns (EToV', perm) with EToV' = EToV[perm]."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(EToV.shape[0])
    return EToV[perm].copy(), perm


def rotate_local_vertices(EToV, seed: int):
    """Apply a seeded even permutation to each element's local vertex order (orientation preserved)."""
    rng = np.random.default_rng(seed)
    choice = rng.integers(0, len(_EVEN_PERMS), size=EToV.shape[0])
    P = _EVEN_PERMS[choice]
    return np.take_along_axis(EToV, P, axis=1).copy()


def jitter_interior(VX, n: int, seed: int, L: float = 1.0, amp: float = 0.1):
    """Move every interior vertex by U(-amp*h, amp*h) per coordinate (h = L/n), seeded.

    With amp = 0.1 every Kuhn tet stays positively oriented (max vertex move
    0.17h against a minimum vertex-to-face height of 0.707h)."""
    rng = np.random.default_rng(seed)
    h = L / n
    VX = VX.copy()
    tol = 1e-12 * L
    interior = np.all((VX > tol) & (VX < L - tol), axis=1)
    d = rng.uniform(-amp * h, amp * h, size=VX.shape)
    VX[interior] += d[interior]
    return VX


def random_fields(K: int, N: int, seed: int = 0, nfields: int = 6):
    """U(-1,1) fields, shape [nfields][K][Np], float64 (C-ABI host layout); nfields = 6
    for Maxwell (Ex..Hz), 4 for acoustics (p, vx, vy, vz)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(nfields, K, np_of(N)))


def random_fields_local(ids, K: int, N: int, seed: int = 0, nfields: int = 6):
    """random_fields(K, N, seed, nfields)[:, ids] without materialising the global array:
    the PCG64 stream behind rng.uniform is one 64-bit draw per value, so the values of global
    element k, field c are draws (c K + k) Np .. + Np, reached with bit_generator.advance
    (per-rank host memory O(K_local), for multi-GPU runs)."""
    Np = np_of(N)
    ids = np.asarray(ids, dtype=np.int64)
    out = np.empty((nfields, ids.size, Np))
    if ids.size == 0:
        return out
    order = np.argsort(ids, kind="stable")
    for c in range(nfields):
        bg = np.random.PCG64(seed)
        pos = 0
        i = 0
        while i < ids.size:  # runs of consecutive global ids in one draw
            j = i
            while j + 1 < ids.size and ids[order[j + 1]] == ids[order[j]] + 1:
                j += 1
            start = (c * K + int(ids[order[i]])) * Np
            bg.advance(start - pos)
            vals = np.random.Generator(bg).uniform(-1.0, 1.0, size=(j - i + 1) * Np).reshape(j - i + 1, Np)
            out[c, order[i:j + 1]] = vals
            pos = start + (j - i + 1) * Np
            i = j + 1
    return out


def cavity_mode_101(x, y, z, t=0.0):
    """Exact PEC eigenmode (1,0,1) of the unit cube, omega = pi*sqrt(2).

    Returns an array [6][...] ordered (Ex,Ey,Ez,Hx,Hy,Hz)."""
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64); z = np.asarray(z, dtype=np.float64)
    pi = math.pi
    w = pi * math.sqrt(2.0)
    zero = np.zeros_like(x)
    Ey = np.sin(pi * x) * np.sin(pi * z) * math.cos(w * t)
    Hx = (pi / w) * np.sin(pi * x) * np.cos(pi * z) * math.sin(w * t)
    Hz = -(pi / w) * np.cos(pi * x) * np.sin(pi * z) * math.sin(w * t)
    return np.stack([zero, Ey, zero, Hx, zero, Hz])


def cavity_mode_111(x, y, z, t=0.0, A=1.0, B=-0.5, C=-0.5):
    """Exact PEC eigenmode (1,1,1) of the unit cube with A+B+C = 0, omega = pi*sqrt(3).

    E = (A cos(px) sin(py) sin(pz), B sin(px) cos(py) sin(pz), C sin(px) sin(py) cos(pz)) cos(wt),
    H = -(curl E0 / w) sin(wt)."""
    if abs(A + B + C) > 1e-14:
        raise ValueError("need A+B+C = 0 (divergence-free)")
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64); z = np.asarray(z, dtype=np.float64)
    pi = math.pi
    w = pi * math.sqrt(3.0)
    cx, sx = np.cos(pi * x), np.sin(pi * x)
    cy, sy = np.cos(pi * y), np.sin(pi * y)
    cz, sz = np.cos(pi * z), np.sin(pi * z)
    ct, st = math.cos(w * t), math.sin(w * t)
    Ex = A * cx * sy * sz * ct
    Ey = B * sx * cy * sz * ct
    Ez = C * sx * sy * cz * ct
    # curl E0 (E0 = E at t=0 without the time factor)
    cEx = pi * (C * sx * cy * cz - B * sx * cy * cz)      # dEz/dy - dEy/dz
    cEy = pi * (A * cx * sy * cz - C * cx * sy * cz)      # dEx/dz - dEz/dx
    cEz = pi * (B * cx * cy * sz - A * cx * cy * sz)      # dEy/dx - dEx/dy
    Hx = -(cEx / w) * st
    Hy = -(cEy / w) * st
    Hz = -(cEz / w) * st
    return np.stack([Ex, Ey, Ez, Hx, Hy, Hz])


def acoustic_mode(x, y, z, t=0.0, lmn=(1, 1, 1)):
    """Exact rigid-wall (v.n = 0) eigenmode of linear acoustics (rho0 = c = 1) in the unit
    cube: p = cos(l pi x) cos(m pi y) cos(n pi z) cos(w t), v = -(sin(w t)/w) grad p0,
    w = pi sqrt(l^2 + m^2 + n^2).  Returns [4][...] ordered (p, vx, vy, vz)."""
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64); z = np.asarray(z, dtype=np.float64)
    l, m, n = lmn
    pi = math.pi
    w = pi * math.sqrt(l * l + m * m + n * n)
    cx, sx = np.cos(l * pi * x), np.sin(l * pi * x)
    cy, sy = np.cos(m * pi * y), np.sin(m * pi * y)
    cz, sz = np.cos(n * pi * z), np.sin(n * pi * z)
    st = math.sin(w * t) / w
    p = cx * cy * cz * math.cos(w * t)
    vx = l * pi * sx * cy * cz * st
    vy = m * pi * cx * sy * cz * st
    vz = n * pi * cx * cy * sz * st
    return np.stack([p, vx, vy, vz])


def dt_rule(VX, EToV, N: int, C: float = 0.25):
    """Harness time step dt = C * h_min / N^2, h_min = 2 * min inradius (PAPER.md:350 'dt ~ dx/N^2';
    SURVEY.md §8(c) reading 10).  r_in = 3 V / (sum of face areas)."""
    a = VX[EToV[:, 0]]; b = VX[EToV[:, 1]]; c = VX[EToV[:, 2]]; d = VX[EToV[:, 3]]
    vol = np.abs(np.einsum("ij,ij->i", b - a, np.cross(c - a, d - a))) / 6.0

    def area(p, q, r):
        return 0.5 * np.linalg.norm(np.cross(q - p, r - p), axis=1)

    S = area(a, b, c) + area(a, b, d) + area(b, c, d) + area(a, c, d)
    rin = 3.0 * vol / S
    return C * 2.0 * float(rin.min()) / (N * N)
