// Host-side mesh setup for straight-sided tetrahedra (FP64, one-off, not timed).
//
// PAPER.md:117-124 (conforming tets), 246-255 (nodal trace picking through
// vmapM/vmapP), 290-308 (eq. 6: per-element affine factors), 720-743
// (face-granular gather metadata).  Face-node matching uses exact integer
// lattice labels instead of coordinates (reading R8).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "refelem.h"

namespace dg {

struct MeshData {
  int64_t K = 0, nv = 0;
  int N = 0, Np = 0, Nfp = 0;
  std::vector<double> VX;        // [nv][3]
  std::vector<int64_t> EToV;     // [K][4]
  std::vector<int64_t> EToE;     // [K][4]  (boundary face: self)
  std::vector<int8_t> EToF;      // [K][4]  (boundary face: self)
  std::vector<int8_t> orient;    // [K][4]  face-node permutation code (0..5), 0 on boundary
  std::vector<double> J;         // [K]
  std::vector<double> rst_x;     // [K][9]  rx ry rz sx sy sz tx ty tz
  std::vector<double> nrm;       // [K][4][4]  nx ny nz Fscale
  std::vector<int64_t> vmapM;    // [K][4][Nfp]  global node id k*Np + n (built on demand: build_maps)
  std::vector<int64_t> vmapP;    // [K][4][Nfp]
  std::vector<int32_t> fperm;    // [6][Nfp]  neighbour face-node index for each orientation code
};

// Validates and builds everything; returns "" on success, else an error message
// (non-positive Jacobian, face shared by > 2 elements, unmatched face nodes, bad ids).
std::string build_mesh(const RefElem& ref, int64_t nv, const double* VX, int64_t K,
                       const int64_t* EToV, MeshData& out);

// vmapM / vmapP of the global mesh from EToE, EToF, orient and fperm (parity export only;
// the device path uses the compressed per-face connectivity or the local gather index).
void build_maps(const RefElem& ref, MeshData& m);

// Physical node coordinates [K][Np] of element k: x = 1/2[-(1+r+s+t)va + (1+r)vb + (1+s)vc + (1+t)vd]
void node_coords(const RefElem& ref, const MeshData& m, double* x, double* y, double* z);

}  // namespace dg
