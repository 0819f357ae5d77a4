// Reference tetrahedron of order N for the nodal DG method (host, FP64).
//
// PAPER.md:141-156 (eq. 3: M, S, D = M^-1 S, face mass M^A), 170-216
// (fig:lifting-matrix: L = M^-1 [M^{A1} .. M^{A4}]), 290-308 (eq. 6: shared
// reference matrices).  The node family is the warp & blend set the paper cites
// ([warburton_explicit_2006]) with HW's alpha_opt table
// (reading R6).
//
// Route (deliberately different from the oracle's Vandermonde/Dubiner route,
// so agreement cross-validates both):
//   * basis: collapsed-coordinate Jacobi products written as HOMOGENEOUS
//     polynomials (no singular collapse), unnormalised, derivatives by
//     forward-mode dual numbers;
//   * Dr/Ds/Dt = Vr V^-1 etc.;
//   * M and the face masses by collapsed Gauss-Legendre quadrature of the
//     Lagrange basis (exact to degree 2N); LIFT = M^-1 Emat by LU.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "linalg.h"

namespace dg {

// local face -> local vertices (face f is opposite to the vertex not listed):
// 0: t=-1 {0,1,2}; 1: s=-1 {0,1,3}; 2: r+s+t=-1 {1,2,3}; 3: r=-1 {0,2,3}
constexpr int kFaceVerts[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {0, 2, 3}};

inline int np_of(int N) { return (N + 1) * (N + 2) * (N + 3) / 6; }
inline int nfp_of(int N) { return (N + 1) * (N + 2) / 2; }

struct RefElem {
  int N = 0, Np = 0, Nfp = 0;
  std::vector<double> r, s, t;                 // [Np] nodes on the bi-unit tet
  std::vector<std::array<int, 4>> lattice;     // [Np] integer barycentric weights (v0..v3), sum N
  std::vector<int> Fmask;                      // [4][Nfp]
  Mat Dr, Ds, Dt;                              // [Np][Np]
  Mat M;                                       // [Np][Np]
  std::array<Mat, 4> face_mass;                // [Nfp][Nfp] in face-parameter coordinates
  Mat LIFT;                                    // [Np][4 Nfp]
};

// Throws std::runtime_error on an unsupported order (1..9) or a numerical failure.
RefElem build_ref_elem(int N);

// Gauss-Lobatto-Legendre points (ascending) and Gauss-Legendre rule, by Newton.
std::vector<double> gll_points(int N);
void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w);

}  // namespace dg
