"""Pins of the oracle's geometry, connectivity and maps (closed forms, brute force, invariants)."""
import itertools
import os

import numpy as np
import pytest

import dg_inputs as di
from oracle import build_reference
from oracle.mesh import MeshError, Setup

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _meshes():
    out = []
    for n in (1, 2, 3):
        VX, E = di.kuhn_box(n)
        out.append((f"kuhn{n}", n, VX, E))
    VX, E = di.kuhn_box(2)
    E2, _ = di.shuffle_elements(E, 1)
    E2 = di.rotate_local_vertices(E2, 3)
    out.append(("kuhn2-shuffled-rotated", 2, VX, E2))
    VXj = di.jitter_interior(VX, 2, seed=2)
    out.append(("kuhn2-jittered", 2, VXj, E2))
    return out


MESHES = _meshes()


@pytest.fixture(scope="module")
def ref3():
    return build_reference(3)


def test_kuhn_first_cell_golden():
    rows = []
    with open(os.path.join(GOLD, "kuhn_n2_first_cell.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                rows.append([int(v) for v in line.split()])
    _, E = di.kuhn_box(2)
    assert E[:6].tolist() == rows


@pytest.mark.parametrize("name,n,VX,E", MESHES, ids=[m[0] for m in MESHES])
def test_geometry_and_maps(name, n, VX, E, ref3):
    st = Setup(VX, E, 3, ref=ref3)
    K = st.K
    # total volume = |[0,1]^3| = sum_k J_k |ref tet| (eq. 6a with 1^T M 1 = 4/3)
    assert abs((st.J * 4.0 / 3.0).sum() - 1.0) < 1e-13
    # per element closed surface: sum_f area_f n_f = 0 with area_f = 2 J Fscale_f
    S = np.stack([st.nx, st.ny, st.nz], 2) * (2 * st.J[:, None] * st.Fscale)[..., None]
    assert np.abs(S.sum(axis=1)).max() < 1e-13
    # unit normals
    assert np.abs(st.nx ** 2 + st.ny ** 2 + st.nz ** 2 - 1).max() < 1e-14
    # face counts on the Kuhn box: interior 12n^3 - 6n^2, boundary 12n^2 (combinatorics)
    bnd = (st.EToE == np.arange(K)[:, None]).sum()
    assert bnd == 12 * n * n
    assert (4 * K - bnd) // 2 == 12 * n ** 3 - 6 * n ** 2
    # antiparallel normals and equal Fscale*J (shared face area) across interior faces
    for k in range(K):
        for f in range(4):
            k2, f2 = st.EToE[k, f], st.EToF[k, f]
            if k2 == k:
                continue
            n1 = np.array([st.nx[k, f], st.ny[k, f], st.nz[k, f]])
            n2 = np.array([st.nx[k2, f2], st.ny[k2, f2], st.nz[k2, f2]])
            assert np.abs(n1 + n2).max() < 1e-13
            assert abs(st.J[k] * st.Fscale[k, f] - st.J[k2] * st.Fscale[k2, f2]) < 1e-14
    # x[vmapM] == x[vmapP]
    for c in (st.x, st.y, st.z):
        f = c.ravel()
        assert np.abs(f[st.vmapM] - f[st.vmapP]).max() < 1e-14
    # vmapP is an involution on face-node slots; boundary slots are exactly the boundary faces
    for k in range(K):
        for f in range(4):
            k2, f2 = st.EToE[k, f], st.EToF[k, f]
            isb = (k2 == k and f2 == f)
            assert np.all(st.mapB[k, f] == isb)
            if isb:
                continue
            for i in range(st.Nfp):
                hit = np.nonzero(st.vmapM[k2, f2] == st.vmapP[k, f, i])[0]
                assert len(hit) == 1
                assert st.vmapP[k2, f2, hit[0]] == st.vmapM[k, f, i]


def test_connectivity_matches_brute_force():
    VX, E = di.kuhn_box(2)
    E, _ = di.shuffle_elements(E, 5)
    E = di.rotate_local_vertices(E, 6)
    st = Setup(VX, E, 1)
    fv = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))
    K = E.shape[0]
    for k in range(K):
        for f in range(4):
            a = set(E[k, list(fv[f])].tolist())
            hits = [(k2, f2) for k2 in range(K) for f2 in range(4)
                    if (k2, f2) != (k, f) and set(E[k2, list(fv[f2])].tolist()) == a]
            if hits:
                assert hits == [(st.EToE[k, f], st.EToF[k, f])]
            else:
                assert (st.EToE[k, f], st.EToF[k, f]) == (k, f)


def test_kuhn_geometry_closed_forms():
    # n=2: h = 1/2; each tet volume h^3/6 = J * 4/3  ->  J = 1/64
    VX, E = di.kuhn_box(2)
    st = Setup(VX, E, 1)
    assert np.allclose(st.J, 1.0 / 64.0, rtol=0, atol=1e-16)
    # Kuhn tet 0 = (0, e_x, e_x+e_y, e_x+e_y+e_z)*h: grad r etc. are rows of A^-1
    assert np.allclose(st.Fscale[0], [4, 4 * np.sqrt(2), 4, 4 * np.sqrt(2)], atol=1e-13)


def test_mesh_errors():
    VX, E = di.kuhn_box(1)
    bad = E.copy()
    bad[0, [2, 3]] = bad[0, [3, 2]]                  # negative orientation
    with pytest.raises(MeshError):
        Setup(VX, bad, 1)
    # a face shared by three tets
    VX3 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]], float)
    E3 = np.array([[0, 1, 2, 3], [0, 2, 1, 4], [0, 1, 2, 5]])
    # orient the third positively (it may already be)
    a, b, c, d = VX3[E3[2]]
    if np.dot(b - a, np.cross(c - a, d - a)) < 0:
        E3[2, [2, 3]] = E3[2, [3, 2]]
    with pytest.raises(MeshError):
        Setup(VX3, E3, 1)


def test_node_coordinates_affine_vertices():
    # vertex nodes land on the element vertices
    VX, E = di.kuhn_box(2)
    VX = di.jitter_interior(VX, 2, 4)
    st = Setup(VX, E, 2)
    B = np.stack([-(1 + st.ref.r + st.ref.s + st.ref.t) / 2, (1 + st.ref.r) / 2,
                  (1 + st.ref.s) / 2, (1 + st.ref.t) / 2], 1)
    for v in range(4):
        n = int(np.argmax(B[:, v]))
        P = np.stack([st.x[:, n], st.y[:, n], st.z[:, n]], 1)
        assert np.abs(P - VX[E[:, v]]).max() < 1e-15
