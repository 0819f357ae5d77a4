"""Oracle mesh setup (test infrastructure only; see oracle/__init__.py).

Affine geometry, normals and connectivity for straight-sided tetrahedra,
following PAPER.md:117-124 (conforming tets), 246-255 (nodal trace picking
through vmapM/vmapP), 290-308 (eq. 6: per-element J_k and dr/dx factors times
shared reference matrices), and HW's StartUp3D / GeometricFactors3D /
Normals3D / tiConnect3D / BuildMaps3D, written out plainly:

* node coordinates x = 1/2[-(1+r+s+t) v_a + (1+r) v_b + (1+s) v_c + (1+t) v_d];
* A = [v_b-v_a, v_c-v_a, v_d-v_a]/2 = dx/dr, J = det A, [grad r; grad s; grad t] = A^-1;
* raw outward normals of faces 0..3: -grad t, -grad s, grad r+grad s+grad t, -grad r;
  Fscale = |raw| (= sJ/J), n = raw/|raw|;
* EToE/EToF by matching sorted global vertex triples; a boundary face points to itself;
* vmapM[k][f][i] = k*Np + Fmask[f][i]; vmapP by coordinate matching of face
  nodes with a relative tolerance 1e-8 (reading R8); on boundary faces
  vmapP = vmapM.
"""
from __future__ import annotations

import numpy as np

from .refelem import RefElement, build_reference

FACE_VERTS = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))


class MeshError(ValueError):
    pass


class Setup:
    """Everything the oracle RHS needs for one mesh and order N."""

    def __init__(self, VX, EToV, N: int, ref: RefElement | None = None):
        VX = np.asarray(VX, dtype=np.float64)
        EToV = np.asarray(EToV, dtype=np.int64)
        self.ref = ref if ref is not None else build_reference(N)
        ref = self.ref
        self.N, self.Np, self.Nfp = ref.N, ref.Np, ref.Nfp
        K = EToV.shape[0]
        self.K = K
        self.VX, self.EToV = VX, EToV
        va, vb, vc, vd = (VX[EToV[:, i]] for i in range(4))          # [K][3]
        r, s, t = ref.r, ref.s, ref.t
        # node coordinates [K][Np] per coordinate
        X = 0.5 * (-(1 + r + s + t)[None, :, None] * va[:, None, :] + (1 + r)[None, :, None] * vb[:, None, :]
                   + (1 + s)[None, :, None] * vc[:, None, :] + (1 + t)[None, :, None] * vd[:, None, :])
        self.x, self.y, self.z = X[..., 0], X[..., 1], X[..., 2]
        # affine Jacobian
        A = np.stack([vb - va, vc - va, vd - va], axis=2) / 2.0          # A[k][:,mu] = dx/dr_mu
        J = np.linalg.det(A)
        if np.any(J <= 0):
            raise MeshError("element with non-positive Jacobian")
        G = np.linalg.inv(A)                                              # rows: grad r, grad s, grad t
        self.J = J
        self.rx, self.ry, self.rz = G[:, 0, 0], G[:, 0, 1], G[:, 0, 2]
        self.sx, self.sy, self.sz = G[:, 1, 0], G[:, 1, 1], G[:, 1, 2]
        self.tx, self.ty, self.tz = G[:, 2, 0], G[:, 2, 1], G[:, 2, 2]
        raw = np.stack([-G[:, 2, :], -G[:, 1, :], G[:, 0, :] + G[:, 1, :] + G[:, 2, :], -G[:, 0, :]], axis=1)  # [K][4][3]
        Fs = np.linalg.norm(raw, axis=2)                                  # [K][4]
        self.Fscale = Fs
        self.nx, self.ny, self.nz = raw[..., 0] / Fs, raw[..., 1] / Fs, raw[..., 2] / Fs
        self._connect()
        self._maps()

    # -- face connectivity by sorted vertex triples -----------------------------
    def _connect(self):
        K = self.K
        EToE = np.tile(np.arange(K)[:, None], (1, 4))
        EToF = np.tile(np.arange(4)[None, :], (K, 1))
        seen = {}
        for k in range(K):
            for f, fv in enumerate(FACE_VERTS):
                key = tuple(sorted(int(self.EToV[k, v]) for v in fv))
                if key in seen:
                    k2, f2 = seen[key]
                    if k2 < 0:
                        raise MeshError("face shared by more than two elements")
                    EToE[k, f], EToF[k, f] = k2, f2
                    EToE[k2, f2], EToF[k2, f2] = k, f
                    seen[key] = (-1, -1)
                else:
                    seen[key] = (k, f)
        self.EToE, self.EToF = EToE, EToF

    # -- volume-to-face maps by coordinate matching -----------------------------
    def _maps(self):
        K, Np, Nfp = self.K, self.Np, self.Nfp
        Fmask = self.ref.Fmask
        vmapM = (np.arange(K)[:, None, None] * Np + Fmask[None, :, :]).astype(np.int64)  # [K][4][Nfp]
        vmapP = vmapM.copy()
        xf, yf, zf = self.x.ravel(), self.y.ravel(), self.z.ravel()
        for k in range(K):
            vk = self.VX[self.EToV[k]]
            h = max(np.linalg.norm(vk[a] - vk[b]) for a in range(4) for b in range(a + 1, 4))
            tol2 = (1e-8 * h) ** 2
            for f in range(4):
                k2, f2 = self.EToE[k, f], self.EToF[k, f]
                if k2 == k and f2 == f:
                    continue                      # boundary face: vmapP = vmapM
                idM = vmapM[k, f]
                idP = vmapM[k2, f2]
                # d2[i, j] = |x(face node i of k) - x(face node j of k2)|^2
                d2 = ((xf[idM][:, None] - xf[idP][None, :]) ** 2 + (yf[idM][:, None] - yf[idP][None, :]) ** 2
                      + (zf[idM][:, None] - zf[idP][None, :]) ** 2)
                hit = d2 < tol2
                if not np.all(hit.sum(axis=1) == 1):
                    raise MeshError("unmatched face node")
                vmapP[k, f] = idP[np.argmax(hit, axis=1)]
        self.vmapM, self.vmapP = vmapM, vmapP
        self.mapB = vmapP == vmapM                                  # [K][4][Nfp] boundary slots
