// Partition, ghost-face plan and gather indices (see partition.h).
#include "partition.h"

#include <algorithm>
#include <map>

namespace dg {

namespace {
uint64_t spread3(uint64_t v) {  // 21-bit -> every third bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}
// sort [b, e) of ids by the Morton code of the element centroids (bounding box of all elements)
void morton_sort(const MeshData& m, std::vector<int64_t>& ids, size_t b, size_t e) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t v = 0; v < m.nv; ++v)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], m.VX[3 * v + d]);
      hi[d] = std::max(hi[d], m.VX[3 * v + d]);
    }
  std::vector<std::pair<uint64_t, int64_t>> key;
  key.reserve(e - b);
  for (size_t i = b; i < e; ++i) {
    const int64_t k = ids[i];
    uint64_t code = 0;
    for (int d = 0; d < 3; ++d) {
      double c = 0;
      for (int q = 0; q < 4; ++q) c += m.VX[3 * m.EToV[4 * k + q] + d];
      c *= 0.25;
      const double t = (c - lo[d]) / std::max(hi[d] - lo[d], 1e-300);
      const uint64_t g = uint64_t(std::min(std::max(t, 0.0), 1.0) * double((1 << 21) - 1));
      code |= spread3(g) << d;
    }
    key.push_back({code, k});
  }
  std::sort(key.begin(), key.end());
  for (size_t i = b; i < e; ++i) ids[i] = key[i - b].second;
}
}  // namespace

void rcb_owners(const MeshData& m, int nranks, std::vector<int32_t>& owner) {
  const int64_t K = m.K;
  std::vector<double> cen(static_cast<size_t>(3 * K));
  for (int64_t k = 0; k < K; ++k)
    for (int d = 0; d < 3; ++d) {
      double c = 0;
      for (int q = 0; q < 4; ++q) c += m.VX[3 * m.EToV[4 * k + q] + d];
      cen[3 * k + d] = 0.25 * c;
    }
  std::vector<int64_t> ids(static_cast<size_t>(K));
  for (int64_t k = 0; k < K; ++k) ids[k] = k;
  owner.assign(size_t(K), 0);
  struct Job { size_t b, e; int r0, nr; };
  std::vector<Job> stack{{0, size_t(K), 0, nranks}};
  while (!stack.empty()) {
    const Job j = stack.back();
    stack.pop_back();
    if (j.nr == 1 || j.e - j.b <= 1) {
      for (size_t i = j.b; i < j.e; ++i) owner[ids[i]] = j.r0;
      continue;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (size_t i = j.b; i < j.e; ++i)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], cen[3 * ids[i] + d]);
        hi[d] = std::max(hi[d], cen[3 * ids[i] + d]);
      }
    int ax = 0;
    for (int d = 1; d < 3; ++d)
      if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;  // largest extent; ties keep the lower axis
    const int nl = j.nr / 2;
    const size_t cut = j.b + size_t((j.e - j.b) * uint64_t(nl) / uint64_t(j.nr));
    std::nth_element(ids.begin() + j.b, ids.begin() + cut, ids.begin() + j.e, [&](int64_t a, int64_t b) {
      const double ca = cen[3 * a + ax], cb = cen[3 * b + ax];
      return ca < cb || (ca == cb && a < b);
    });
    stack.push_back({j.b, cut, j.r0, nl});
    stack.push_back({cut, j.e, j.r0 + nl, j.nr - nl});
  }
}

std::string build_partition(const MeshData& m, int rank, int nranks, const int32_t* owner,
                            Partition& P, bool reorder) {
  const int64_t K = m.K;
  P = Partition();
  P.rank = rank;
  P.nranks = nranks;
  P.K_global = K;
  std::vector<int32_t> own(K);
  for (int64_t k = 0; k < K; ++k) {
    own[k] = owner ? owner[k] : int32_t((k * nranks) / K);
    if (own[k] < 0 || own[k] >= nranks) return "partition owner out of range at element " + std::to_string(k);
  }
  // per rank pair: cross faces keyed by the lower-rank side's slot
  std::map<int, std::vector<std::pair<int64_t, int64_t>>> cross;  // peer -> (key, my slot)
  std::vector<char> is_bnd(K, 0);
  for (int64_t k = 0; k < K; ++k) {
    if (own[k] != rank) continue;
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = m.EToE[4 * k + f];
      const int f2 = m.EToF[4 * k + f];
      const int q = own[k2];
      if (q == rank) continue;
      is_bnd[k] = 1;
      const int64_t mine = 4 * k + f, theirs = 4 * k2 + f2;
      const int64_t key = rank < q ? mine : theirs;
      cross[q].push_back({key, mine});
    }
  }
  // boundary-first: a stage writes the boundary elements' fields in its first tiles, so the
  // next stage's trace exchange starts while the interior tiles are still running
  for (int64_t k = 0; k < K; ++k)
    if (own[k] == rank && is_bnd[k]) P.local_ids.push_back(k);
  P.K_boundary = int64_t(P.local_ids.size());
  for (int64_t k = 0; k < K; ++k)
    if (own[k] == rank && !is_bnd[k]) P.local_ids.push_back(k);
  P.K_local = int64_t(P.local_ids.size());
  if (reorder) {
    morton_sort(m, P.local_ids, 0, size_t(P.K_boundary));
    morton_sort(m, P.local_ids, size_t(P.K_boundary), size_t(P.K_local));
  }
  P.g2l.assign(K, -1);
  for (int64_t l = 0; l < P.K_local; ++l) P.g2l[P.local_ids[l]] = l;
  P.ghost_of.assign(4 * P.K_local, -1);
  int64_t off = 0;
  for (auto& kv : cross) {
    auto& v = kv.second;
    std::sort(v.begin(), v.end());
    PeerPlan pp;
    pp.rank = kv.first;
    pp.nfaces = int64_t(v.size());
    pp.send_off = off;
    pp.recv_off = off;  // symmetric: the peer has the same cross faces
    for (size_t i = 0; i < v.size(); ++i) {
      const int64_t slot = v[i].second;
      const int64_t l = P.g2l[slot / 4];
      P.send_elem.push_back(l);
      P.send_face.push_back(int8_t(slot % 4));
      P.ghost_of[4 * l + slot % 4] = off + int64_t(i);
    }
    off += pp.nfaces;
    P.peers.push_back(pp);
  }
  P.n_ghost_faces = off;
  return "";
}

void build_gather_index(const RefElem& ref, const MeshData& m, const Partition& P, const TileLayout& L,
                        int64_t ghost_base, std::vector<int32_t>& gidx) {
  const int Nfp = ref.Nfp;
  gidx.assign(size_t(L.ntiles(P.K_local)) * L.E * 4 * Nfp, -1);
  for (int64_t l = 0; l < P.K_local; ++l) {
    const int64_t k = P.local_ids[l];
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = m.EToE[4 * k + f];
      const int f2 = m.EToF[4 * k + f];
      if (k2 == k && f2 == f) continue;  // PEC wall
      const int code = m.orient[4 * k + f];
      const int64_t g = P.ghost_of[4 * l + f];
      for (int i = 0; i < Nfp; ++i) {
        const int j = m.fperm[code * Nfp + i];  // neighbour face-node position
        int64_t v;
        const int64_t l2 = g >= 0 ? -1 : P.g2l[k2];
        if (L.perm >= 1 && l2 >= 0 && l2 / L.E == l / L.E)
          v = TileLayout::intra(int(l2 % L.E), ref.Fmask[f2 * Nfp + j]);
        else if (L.perm == 2)
          v = g >= 0 ? (TileLayout::GHOST_FLAG | (g * L.nc * Nfp + j))
                     : ((P.g2l[k2] << 8) | ref.Fmask[f2 * Nfp + j]);
        else if (g >= 0)
          v = ghost_base + g * L.nc * Nfp + j;
        else
          v = L.off(P.g2l[k2], 0, ref.Fmask[f2 * Nfp + j]);
        const int64_t mm = int64_t(f) * Nfp + i;  // face-node slot of element l
        if (L.perm == 3)  // FFMA tiles store the index [tile][m][e] (elements fastest)
          gidx[(l / L.E) * L.E * 4 * Nfp + mm * L.E + l % L.E] = int32_t(v);
        else
          gidx[4 * l * Nfp + mm] = int32_t(v);
      }
    }
  }
}

void build_face_connectivity(const RefElem& ref, const MeshData& m, const Partition& P, const TileLayout& L,
                             std::vector<int32_t>& fbase, std::vector<uint8_t>& fcode, std::vector<int16_t>& ftab) {
  const int Nfp = ref.Nfp, NF = 4 * Nfp;
  const int64_t Kpad = L.ntiles(P.K_local) * L.E;
  fbase.assign(size_t(Kpad) * 4, -1);
  fcode.assign(size_t(Kpad) * 4, 0);
  for (int64_t l = 0; l < P.K_local; ++l) {
    const int64_t k = P.local_ids[l];
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = m.EToE[4 * k + f];
      const int f2 = m.EToF[4 * k + f];
      if (k2 == k && f2 == f) continue;  // PEC wall
      const int code = m.orient[4 * k + f];
      const int64_t g = P.ghost_of[4 * l + f];
      if (g >= 0) {
        fbase[4 * l + f] = TileLayout::ghost_code(g * L.nc * Nfp);  // negative: local bases reach 2^31 - 1
        fcode[4 * l + f] = uint8_t(code);
      } else {
        fbase[4 * l + f] = int32_t(L.off(P.g2l[k2], 0, 0));
        fcode[4 * l + f] = uint8_t(f2 * 6 + code);
      }
    }
  }
  ftab.assign(size_t(NF) + 30 * Nfp, 0);
  for (int i = 0; i < NF; ++i) ftab[i] = int16_t(ref.Fmask[i]);
  for (int f2 = 0; f2 < 4; ++f2)
    for (int o = 0; o < 6; ++o)
      for (int i = 0; i < Nfp; ++i)
        ftab[NF + (f2 * 6 + o) * Nfp + i] = int16_t(ref.Fmask[f2 * Nfp + m.fperm[o * Nfp + i]]);
  for (int o = 0; o < 6; ++o)
    for (int i = 0; i < Nfp; ++i) ftab[NF + 24 * Nfp + o * Nfp + i] = int16_t(m.fperm[o * Nfp + i]);
}

}  // namespace dg
