// Mesh partition for multi-GPU runs (distributed DG, one
// exchange of face data per stage; volume ~ N^3 vs surface ~ N^2).
//
// Each rank owns a set of elements.  Local storage order: the partition-boundary
// elements (a face on another rank) first, then the interior elements, each group
// in ascending global id.  A stage kernel writes the boundary elements in its first
// tiles and signals their completion, so the next stage's trace exchange runs while
// the interior tiles are still being computed.
//
// Ghost faces: for every rank pair (r, q) the cross faces are ordered by the
// global slot 4k+f of the face on the LOWER rank; rank r sends, for each of its
// cross faces in that order, the 6*Nfp traces u[k][c][Fmask[f][j]] in its own
// face-node order (record [c][j]); the receiver reads its u+ from the record
// through the same orientation permutation it uses for a local neighbour.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "mesh.h"
#include "../kernels/stage_params.h"

namespace dg {

struct PeerPlan {
  int rank = -1;            // peer rank
  int64_t nfaces = 0;       // cross faces with this peer
  int64_t send_off = 0;     // offset (faces) into this rank's send buffer
  int64_t recv_off = 0;     // offset (faces) into this rank's ghost region
};

struct Partition {
  int rank = 0, nranks = 1;
  int64_t K_global = 0, K_local = 0, K_boundary = 0;
  std::vector<int64_t> local_ids;   // [K_local] global id of local element l (storage order)
  std::vector<int64_t> g2l;         // [K_global] local index or -1
  std::vector<PeerPlan> peers;      // ascending peer rank
  int64_t n_ghost_faces = 0;        // total received faces (= total sent faces)
  // send list: for send face s (in buffer order) the local element and face
  std::vector<int64_t> send_elem;   // [n_ghost_faces]
  std::vector<int8_t> send_face;    // [n_ghost_faces]
  // for local element l, face f: ghost record index (or -1 if not a cross face)
  std::vector<int64_t> ghost_of;    // [K_local][4]
};

// owner: [K] rank per element, or empty -> contiguous ranges.  reorder: sort each group
// (boundary, interior) by the Morton code of the element centroids.  Returns "" or an error.
std::string build_partition(const MeshData& m, int rank, int nranks, const int32_t* owner,
                            Partition& out, bool reorder = false);

// Recursive coordinate bisection: owner[k] for every element, by recursively
// splitting the element set at the rank-weighted median centroid coordinate along the axis
// of largest extent (ties broken by element id, so every rank computes the same owners).
void rcb_owners(const MeshData& m, int nranks, std::vector<int32_t>& owner);

// Gather index of the exterior trace for every local face node (see
// stage_params.h): L.off(k2_local, 0, n2), or ghost_base + g*6*Nfp + j, or -1
// (PEC).  Rows are padded to ntiles*E elements (padding rows = -1).
void build_gather_index(const RefElem& ref, const MeshData& m, const Partition& P, const TileLayout& L,
                        int64_t ghost_base, std::vector<int32_t>& gidx);

// Compressed face connectivity of the TC kernel (perm 4), per local (element, face):
// fbase = L.off(k2_local, 0, 0) (word offset of the neighbour's node 0, component 0),
// or GHOST_FLAG | g*nc*Nfp (its ghost record), or -1 (PEC); fcode = f2*6 + orientation
// (ghost: orientation).  ftab = Fmask [4Nfp] | node of neighbour face node i, by
// (f2*6 + orientation) [24][Nfp] | ghost-record position, by orientation [6][Nfp].
// Together they rebuild exactly the nodes of build_gather_index (SURVEY §7 hard part 5).
void build_face_connectivity(const RefElem& ref, const MeshData& m, const Partition& P, const TileLayout& L,
                             std::vector<int32_t>& fbase, std::vector<uint8_t>& fcode, std::vector<int16_t>& ftab);

}  // namespace dg
