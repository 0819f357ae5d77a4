// Small dense FP64 linear algebra for the host-side setup (reference element,
// affine geometry).  Row-major std::vector<double>; LU with partial pivoting.
#pragma once
#include <cmath>
#include <stdexcept>
#include <vector>

namespace dg {

struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(size_t(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) * cols + j]; }
  double operator()(int i, int j) const { return a[size_t(i) * cols + j]; }
};

inline Mat matmul(const Mat& A, const Mat& B) {
  if (A.cols != B.rows) throw std::runtime_error("matmul: shape mismatch");
  Mat C(A.rows, B.cols);
  for (int i = 0; i < A.rows; ++i)
    for (int k = 0; k < A.cols; ++k) {
      const double aik = A(i, k);
      for (int j = 0; j < B.cols; ++j) C(i, j) += aik * B(k, j);
    }
  return C;
}

inline Mat transpose(const Mat& A) {
  Mat T(A.cols, A.rows);
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j) T(j, i) = A(i, j);
  return T;
}

// LU factorisation with partial pivoting, in place.
struct LU {
  Mat lu;
  std::vector<int> piv;
  explicit LU(const Mat& A) : lu(A), piv(A.rows) {
    const int n = A.rows;
    if (A.cols != n) throw std::runtime_error("LU: not square");
    for (int i = 0; i < n; ++i) piv[i] = i;
    for (int k = 0; k < n; ++k) {
      int p = k;
      double best = std::fabs(lu(k, k));
      for (int i = k + 1; i < n; ++i)
        if (std::fabs(lu(i, k)) > best) { best = std::fabs(lu(i, k)); p = i; }
      if (best == 0.0) throw std::runtime_error("LU: singular matrix");
      if (p != k) {
        for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
        std::swap(piv[k], piv[p]);
      }
      const double inv = 1.0 / lu(k, k);
      for (int i = k + 1; i < n; ++i) {
        const double l = lu(i, k) * inv;
        lu(i, k) = l;
        if (l != 0.0)
          for (int j = k + 1; j < n; ++j) lu(i, j) -= l * lu(k, j);
      }
    }
  }
  // Solve A X = B (B: n x m), returns X.
  Mat solve(const Mat& B) const {
    const int n = lu.rows, m = B.cols;
    Mat X(n, m);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < m; ++j) X(i, j) = B(piv[i], j);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) {
        const double l = lu(i, k);
        if (l != 0.0)
          for (int j = 0; j < m; ++j) X(i, j) -= l * X(k, j);
      }
    for (int i = n - 1; i >= 0; --i) {
      for (int k = i + 1; k < n; ++k) {
        const double u = lu(i, k);
        if (u != 0.0)
          for (int j = 0; j < m; ++j) X(i, j) -= u * X(k, j);
      }
      const double inv = 1.0 / lu(i, i);
      for (int j = 0; j < m; ++j) X(i, j) *= inv;
    }
    return X;
  }
};

// X with X A = B  (i.e. X = B A^-1), via A^T X^T = B^T.
inline Mat right_solve(const Mat& B, const Mat& A) {
  LU f(transpose(A));
  return transpose(f.solve(transpose(B)));
}

}  // namespace dg
