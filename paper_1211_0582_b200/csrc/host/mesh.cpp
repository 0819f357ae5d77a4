// Mesh validation, connectivity, maps and affine geometry (see mesh.h).
#include "mesh.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>

namespace dg {

namespace {

// the 6 permutations of (0,1,2), lexicographic; code = index
constexpr int kPerm3[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

struct FaceKey {
  int64_t g[3];
  int64_t slot;  // k*4 + f
};

}  // namespace

std::string build_mesh(const RefElem& ref, int64_t nv, const double* VX, int64_t K,
                       const int64_t* EToV, MeshData& m) {
  const int N = ref.N, Np = ref.Np, Nfp = ref.Nfp;
  if (nv <= 0 || K <= 0 || !VX || !EToV) return "empty mesh";
  m = MeshData();
  m.K = K; m.nv = nv; m.N = N; m.Np = Np; m.Nfp = Nfp;
  m.VX.assign(VX, VX + 3 * nv);
  m.EToV.assign(EToV, EToV + 4 * K);
  for (int64_t i = 0; i < 4 * K; ++i)
    if (EToV[i] < 0 || EToV[i] >= nv) return "EToV entry out of range at element " + std::to_string(i / 4);

  // ---- affine geometry: A = [vb-va, vc-va, vd-va]/2 = dx/dr (columns), J = det A,
  //      rows of A^-1 = grad r, grad s, grad t  (eq. 6)
  m.J.resize(K);
  m.rst_x.resize(9 * K);
  m.nrm.resize(16 * K);
  for (int64_t k = 0; k < K; ++k) {
    const double* va = VX + 3 * EToV[4 * k + 0];
    const double* vb = VX + 3 * EToV[4 * k + 1];
    const double* vc = VX + 3 * EToV[4 * k + 2];
    const double* vd = VX + 3 * EToV[4 * k + 3];
    double A[3][3];
    for (int d = 0; d < 3; ++d) {
      A[d][0] = 0.5 * (vb[d] - va[d]);
      A[d][1] = 0.5 * (vc[d] - va[d]);
      A[d][2] = 0.5 * (vd[d] - va[d]);
    }
    const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
    const double c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2];
    const double c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    const double J = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
    if (!(J > 0.0)) return "element " + std::to_string(k) + " has non-positive Jacobian";
    m.J[k] = J;
    const double iJ = 1.0 / J;
    // inverse = adj(A)/J ; G[i][j] = d r_i / d x_j
    double G[3][3];
    G[0][0] = c00 * iJ;
    G[1][0] = c01 * iJ;
    G[2][0] = c02 * iJ;
    G[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) * iJ;
    G[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) * iJ;
    G[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) * iJ;
    G[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) * iJ;
    G[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) * iJ;
    G[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) * iJ;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) m.rst_x[9 * k + 3 * i + j] = G[i][j];
    // raw outward normals: -grad t, -grad s, grad r + grad s + grad t, -grad r
    double raw[4][3];
    for (int d = 0; d < 3; ++d) {
      raw[0][d] = -G[2][d];
      raw[1][d] = -G[1][d];
      raw[2][d] = G[0][d] + G[1][d] + G[2][d];
      raw[3][d] = -G[0][d];
    }
    for (int f = 0; f < 4; ++f) {
      const double Fs = std::sqrt(raw[f][0] * raw[f][0] + raw[f][1] * raw[f][1] + raw[f][2] * raw[f][2]);
      double* o = &m.nrm[16 * k + 4 * f];
      o[0] = raw[f][0] / Fs;
      o[1] = raw[f][1] / Fs;
      o[2] = raw[f][2] / Fs;
      o[3] = Fs;
    }
  }

  // ---- face connectivity: sort faces by their sorted global vertex triple
  std::vector<FaceKey> keys(4 * K);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) {
      FaceKey& fk = keys[4 * k + f];
      for (int p = 0; p < 3; ++p) fk.g[p] = EToV[4 * k + kFaceVerts[f][p]];
      std::sort(fk.g, fk.g + 3);
      fk.slot = 4 * k + f;
    }
  std::sort(keys.begin(), keys.end(), [](const FaceKey& a, const FaceKey& b) {
    if (a.g[0] != b.g[0]) return a.g[0] < b.g[0];
    if (a.g[1] != b.g[1]) return a.g[1] < b.g[1];
    if (a.g[2] != b.g[2]) return a.g[2] < b.g[2];
    return a.slot < b.slot;
  });
  m.EToE.resize(4 * K);
  m.EToF.resize(4 * K);
  m.orient.assign(4 * K, 0);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) { m.EToE[4 * k + f] = k; m.EToF[4 * k + f] = (int8_t)f; }
  auto same = [](const FaceKey& a, const FaceKey& b) {
    return a.g[0] == b.g[0] && a.g[1] == b.g[1] && a.g[2] == b.g[2];
  };
  for (size_t i = 0; i < keys.size();) {
    size_t j = i + 1;
    while (j < keys.size() && same(keys[i], keys[j])) ++j;
    if (j - i > 2) return "face shared by more than two elements";
    if (j - i == 2) {
      const int64_t s1 = keys[i].slot, s2 = keys[i + 1].slot;
      if (s1 / 4 == s2 / 4) return "element " + std::to_string(s1 / 4) + " has a repeated face";
      m.EToE[s1] = s2 / 4; m.EToF[s1] = (int8_t)(s2 % 4);
      m.EToE[s2] = s1 / 4; m.EToF[s2] = (int8_t)(s1 % 4);
    }
    i = j;
  }

  // ---- face-node permutation tables.  Every face enumerates its nodes with the
  // same face-local weight pattern W(i) = (N-x-y, x, y) (y outer, x inner) at its
  // local vertex positions (0,1,2); for a vertex correspondence sigma (position p
  // of this face <-> position sigma[p] of the neighbour face) the neighbour node
  // is the j with W(j)[sigma[p]] = W(i)[p].
  std::vector<std::array<int, 3>> W(Nfp);
  {
    int i = 0;
    for (int y = 0; y <= N; ++y)
      for (int x = 0; x <= N - y; ++x) W[i++] = {N - x - y, x, y};
  }
  // consistency: Fmask enumeration of every face follows W
  for (int f = 0; f < 4; ++f)
    for (int i = 0; i < Nfp; ++i) {
      const auto& L = ref.lattice[ref.Fmask[f * Nfp + i]];
      for (int p = 0; p < 3; ++p)
        if (L[kFaceVerts[f][p]] != W[i][p]) return "internal: face enumeration mismatch";
    }
  m.fperm.assign(6 * Nfp, -1);
  for (int c = 0; c < 6; ++c)
    for (int i = 0; i < Nfp; ++i) {
      std::array<int, 3> want;
      for (int p = 0; p < 3; ++p) want[kPerm3[c][p]] = W[i][p];
      for (int j = 0; j < Nfp; ++j)
        if (W[j] == want) { m.fperm[c * Nfp + i] = j; break; }
      if (m.fperm[c * Nfp + i] < 0) return "internal: face permutation";
    }

  // ---- orientation codes (the per-node maps are built on demand by build_maps: they are
  // O(K Nfp) int64 per rank, 7.9 GB for C5 at N = 9, and only the parity export needs them)
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = m.EToE[4 * k + f];
      const int f2 = m.EToF[4 * k + f];
      int code = 0;
      if (!(k2 == k && f2 == f)) {
        int64_t g[3], h[3];
        for (int p = 0; p < 3; ++p) {
          g[p] = EToV[4 * k + kFaceVerts[f][p]];
          h[p] = EToV[4 * k2 + kFaceVerts[f2][p]];
        }
        int sig[3];
        for (int p = 0; p < 3; ++p) {
          sig[p] = -1;
          for (int q = 0; q < 3; ++q)
            if (h[q] == g[p]) sig[p] = q;
          if (sig[p] < 0) return "unmatched face nodes";
        }
        code = -1;
        for (int c = 0; c < 6; ++c)
          if (kPerm3[c][0] == sig[0] && kPerm3[c][1] == sig[1] && kPerm3[c][2] == sig[2]) code = c;
        if (code < 0) return "unmatched face nodes";
      }
      m.orient[4 * k + f] = (int8_t)code;
    }
  return "";
}

void build_maps(const RefElem& ref, MeshData& m) {
  if (!m.vmapM.empty() || m.K == 0) return;
  const int Np = ref.Np, Nfp = ref.Nfp;
  const int64_t K = m.K;
  m.vmapM.resize(4 * K * Nfp);
  m.vmapP.resize(4 * K * Nfp);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = m.EToE[4 * k + f];
      const int f2 = m.EToF[4 * k + f];
      const int code = m.orient[4 * k + f];
      for (int i = 0; i < Nfp; ++i) {
        const int64_t slot = (4 * k + f) * Nfp + i;
        m.vmapM[slot] = k * Np + ref.Fmask[f * Nfp + i];
        if (k2 == k && f2 == f)
          m.vmapP[slot] = m.vmapM[slot];
        else
          m.vmapP[slot] = k2 * Np + ref.Fmask[f2 * Nfp + m.fperm[code * Nfp + i]];
      }
    }
}

void node_coords(const RefElem& ref, const MeshData& m, double* x, double* y, double* z) {
  const int Np = ref.Np;
  for (int64_t k = 0; k < m.K; ++k) {
    const double* va = &m.VX[3 * m.EToV[4 * k + 0]];
    const double* vb = &m.VX[3 * m.EToV[4 * k + 1]];
    const double* vc = &m.VX[3 * m.EToV[4 * k + 2]];
    const double* vd = &m.VX[3 * m.EToV[4 * k + 3]];
    for (int n = 0; n < Np; ++n) {
      const double r = ref.r[n], s = ref.s[n], t = ref.t[n];
      const double ca = -(1 + r + s + t), cb = 1 + r, cc = 1 + s, cd = 1 + t;
      x[k * Np + n] = 0.5 * (ca * va[0] + cb * vb[0] + cc * vc[0] + cd * vd[0]);
      y[k * Np + n] = 0.5 * (ca * va[1] + cb * vb[1] + cc * vc[1] + cd * vd[1]);
      z[k * Np + n] = 0.5 * (ca * va[2] + cb * vb[2] + cc * vc[2] + cd * vd[2]);
    }
  }
}

}  // namespace dg
