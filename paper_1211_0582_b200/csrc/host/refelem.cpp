// Reference element construction (see refelem.h for the route and citations).
#include "refelem.h"

#include <cmath>
#include <stdexcept>

namespace dg {

namespace {

// forward-mode dual number in (r, s, t)
struct D4 {
  double v, dr, ds, dt;
};
inline D4 cst(double c) { return {c, 0, 0, 0}; }
inline D4 operator+(D4 a, D4 b) { return {a.v + b.v, a.dr + b.dr, a.ds + b.ds, a.dt + b.dt}; }
inline D4 operator-(D4 a, D4 b) { return {a.v - b.v, a.dr - b.dr, a.ds - b.ds, a.dt - b.dt}; }
inline D4 operator*(double c, D4 a) { return {c * a.v, c * a.dr, c * a.ds, c * a.dt}; }
inline D4 operator*(D4 a, D4 b) {
  return {a.v * b.v, a.dr * b.v + a.v * b.dr, a.ds * b.v + a.v * b.ds, a.dt * b.v + a.v * b.dt};
}

// Homogeneous Jacobi polynomial H_n(u,v) = v^n P_n^{(al,be)}(u/v), classical
// (unnormalised) three-term recurrence multiplied through by powers of v.
D4 hjacobi(int n, double al, double be, D4 u, D4 v) {
  D4 p0 = cst(1.0);
  if (n == 0) return p0;
  D4 p1 = 0.5 * ((al + be + 2.0) * u + (al - be) * v);
  for (int k = 2; k <= n; ++k) {
    const double c = 2.0 * k + al + be;
    const double a1 = 2.0 * k * (k + al + be) * (c - 2.0);
    const double a2 = (c - 1.0) * (al * al - be * be);
    const double a3 = (c - 1.0) * c * (c - 2.0);
    const double a4 = 2.0 * (k + al - 1.0) * (k + be - 1.0) * c;
    D4 p2 = (1.0 / a1) * ((a3 * u + a2 * v) * p1 - a4 * (v * v * p0));
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

// PKD-type basis function (i,j,k) at (r,s,t), as a polynomial in r,s,t:
//   H_i^{(0,0)}(2+2r+s+t, -s-t) * H_j^{(2i+1,0)}(1+2s+t, 1-t) * P_k^{(2i+2j+2,0)}(t)
D4 basis3d(int i, int j, int k, double r, double s, double t) {
  const D4 R = {r, 1, 0, 0}, S = {s, 0, 1, 0}, T = {t, 0, 0, 1};
  const D4 one = cst(1.0);
  D4 f = hjacobi(i, 0.0, 0.0, cst(2.0) + 2.0 * R + S + T, cst(0.0) - S - T);
  D4 g = hjacobi(j, 2.0 * i + 1.0, 0.0, one + 2.0 * S + T, one - T);
  D4 h = hjacobi(k, 2.0 * (i + j) + 2.0, 0.0, T, one);
  return f * g * h;
}

void basis_rows(int N, const std::vector<double>& r, const std::vector<double>& s,
                const std::vector<double>& t, Mat* V, Mat* Vr, Mat* Vs, Mat* Vt) {
  const int n = (int)r.size();
  const int Np = np_of(N);
  if (V) *V = Mat(n, Np);
  if (Vr) *Vr = Mat(n, Np);
  if (Vs) *Vs = Mat(n, Np);
  if (Vt) *Vt = Mat(n, Np);
  for (int p = 0; p < n; ++p) {
    int m = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j)
        for (int k = 0; k <= N - i - j; ++k, ++m) {
          D4 b = basis3d(i, j, k, r[p], s[p], t[p]);
          if (V) (*V)(p, m) = b.v;
          if (Vr) (*Vr)(p, m) = b.dr;
          if (Vs) (*Vs)(p, m) = b.ds;
          if (Vt) (*Vt)(p, m) = b.dt;
        }
  }
}

// Legendre P_n and P_{n-1} at x
void legendre2(int n, double x, double& pn, double& pnm1) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { pn = 1.0; pnm1 = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  pn = p1;
  pnm1 = p0;
}

// 1-D warp function of SURVEY.md A.2:
//   warp(x) = sum_{interior i} (x_i^GLL - x_i^eq) * l_i^eq(x) / (1 - x^2)
// with the endpoint factors of l_i cancelled analytically.
double warp1d(int N, const std::vector<double>& xgll, double x) {
  std::vector<double> xeq(N + 1);
  for (int i = 0; i <= N; ++i) xeq[i] = -1.0 + 2.0 * i / N;
  double w = 0.0;
  for (int i = 1; i < N; ++i) {
    double l = 1.0;
    for (int j = 1; j < N; ++j)
      if (j != i) l *= (x - xeq[j]) / (xeq[i] - xeq[j]);
    // l_i(x)/(1-x^2) = l_int(x) * (x+1)(x-1)/((xi+1)(xi-1)) / (1-x^2) = -l_int(x)/((xi+1)(xi-1))
    l = -l / ((xeq[i] + 1.0) * (xeq[i] - 1.0));
    w += (xgll[i] - xeq[i]) * l;
  }
  return w;
}

void eval_shift(int N, const std::vector<double>& xgll, double alpha, double L1, double L2,
                double L3, double& dx, double& dy) {
  const double w1 = 4.0 * L2 * L3 * warp1d(N, xgll, L3 - L2) * (1.0 + (alpha * L1) * (alpha * L1));
  const double w2 = 4.0 * L1 * L3 * warp1d(N, xgll, L1 - L3) * (1.0 + (alpha * L2) * (alpha * L2));
  const double w3 = 4.0 * L1 * L2 * warp1d(N, xgll, L2 - L1) * (1.0 + (alpha * L3) * (alpha * L3));
  const double pi = 3.14159265358979323846;
  dx = w1 + std::cos(2.0 * pi / 3.0) * w2 + std::cos(4.0 * pi / 3.0) * w3;
  dy = std::sin(2.0 * pi / 3.0) * w2 + std::sin(4.0 * pi / 3.0) * w3;
}

const double kAlphaOpt[9] = {0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577, 1.1603};

void warp_blend_nodes(int N, RefElem& E) {
  const double tol = 1e-10;
  const double alpha = kAlphaOpt[N - 1];
  const std::vector<double> xgll = gll_points(N);
  const double s3 = std::sqrt(3.0), s6 = std::sqrt(6.0);
  const double v[4][3] = {{-1.0, -1.0 / s3, -1.0 / s6}, {1.0, -1.0 / s3, -1.0 / s6},
                          {0.0, 2.0 / s3, -1.0 / s6}, {0.0, 0.0, 3.0 / s6}};
  double t1[4][3], t2[4][3];
  for (int d = 0; d < 3; ++d) {
    t1[0][d] = v[1][d] - v[0][d];
    t1[1][d] = v[1][d] - v[0][d];
    t1[2][d] = v[2][d] - v[1][d];
    t1[3][d] = v[2][d] - v[0][d];
    t2[0][d] = v[2][d] - 0.5 * (v[0][d] + v[1][d]);
    t2[1][d] = v[3][d] - 0.5 * (v[0][d] + v[1][d]);
    t2[2][d] = v[3][d] - 0.5 * (v[1][d] + v[2][d]);
    t2[3][d] = v[3][d] - 0.5 * (v[0][d] + v[2][d]);
  }
  for (int f = 0; f < 4; ++f) {
    double a = 0, b = 0;
    for (int d = 0; d < 3; ++d) { a += t1[f][d] * t1[f][d]; b += t2[f][d] * t2[f][d]; }
    a = std::sqrt(a); b = std::sqrt(b);
    for (int d = 0; d < 3; ++d) { t1[f][d] /= a; t2[f][d] /= b; }
  }
  // 3x3 map back: [(v2-v1)/2 (v3-v1)/2 (v4-v1)/2] (r,s,t)^T = X - (v2+v3+v4-v1)/2
  Mat A(3, 3);
  for (int d = 0; d < 3; ++d) {
    A(d, 0) = 0.5 * (v[1][d] - v[0][d]);
    A(d, 1) = 0.5 * (v[2][d] - v[0][d]);
    A(d, 2) = 0.5 * (v[3][d] - v[0][d]);
  }
  LU Af(A);
  for (int l = 0; l <= N; ++l)
    for (int m = 0; m <= N - l; ++m)
      for (int q = 0; q <= N - l - m; ++q) {
        const double r0 = -1.0 + 2.0 * q / N, s0 = -1.0 + 2.0 * m / N, t0 = -1.0 + 2.0 * l / N;
        const double L1 = (1 + t0) / 2, L2 = (1 + s0) / 2, L3 = -(1 + r0 + s0 + t0) / 2, L4 = (1 + r0) / 2;
        double X[3], sh[3] = {0, 0, 0};
        for (int d = 0; d < 3; ++d) X[d] = L3 * v[0][d] + L4 * v[1][d] + L2 * v[2][d] + L1 * v[3][d];
        const double Ls[4][4] = {{L1, L2, L3, L4}, {L2, L1, L3, L4}, {L3, L1, L4, L2}, {L4, L1, L3, L2}};
        for (int f = 0; f < 4; ++f) {
          const double La = Ls[f][0], Lb = Ls[f][1], Lc = Ls[f][2], Ld = Ls[f][3];
          double w1, w2;
          eval_shift(N, xgll, alpha, Lb, Lc, Ld, w1, w2);
          double blend = Lb * Lc * Ld;
          const double denom = (Lb + 0.5 * La) * (Lc + 0.5 * La) * (Ld + 0.5 * La);
          if (denom > tol) blend = (1.0 + (alpha * La) * (alpha * La)) * blend / denom;
          for (int d = 0; d < 3; ++d) sh[d] += blend * w1 * t1[f][d] + blend * w2 * t2[f][d];
          const int nin = (Lb > tol) + (Lc > tol) + (Ld > tol);
          if (La < tol && nin < 3)
            for (int d = 0; d < 3; ++d) sh[d] = w1 * t1[f][d] + w2 * t2[f][d];
        }
        Mat rhs(3, 1);
        for (int d = 0; d < 3; ++d)
          rhs(d, 0) = X[d] + sh[d] - 0.5 * (v[1][d] + v[2][d] + v[3][d] - v[0][d]);
        Mat rst = Af.solve(rhs);
        E.r.push_back(rst(0, 0));
        E.s.push_back(rst(1, 0));
        E.t.push_back(rst(2, 0));
        E.lattice.push_back({N - q - m - l, q, m, l});
      }
}

}  // namespace

std::vector<double> gll_points(int N) {
  // interior GLL points = roots of P_N'; Newton on (x P_N - P_{N-1}) from Chebyshev-GL guesses
  std::vector<double> x(N + 1);
  for (int i = 0; i <= N; ++i) x[i] = -std::cos(3.14159265358979323846 * i / N);
  for (int i = 1; i < N; ++i) {
    double xi = x[i];
    for (int it = 0; it < 100; ++it) {
      double pn, pnm1;
      legendre2(N, xi, pn, pnm1);
      const double dx = (xi * pn - pnm1) / ((N + 1) * pn);
      xi -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    x[i] = xi;
  }
  x[0] = -1.0;
  x[N] = 1.0;
  // enforce exact symmetry (the point set is symmetric about 0)
  for (int i = 0; i <= N / 2; ++i) {
    const double a = 0.5 * (x[N - i] - x[i]);
    x[i] = -a;
    x[N - i] = a;
  }
  if (N % 2 == 0) x[N / 2] = 0.0;
  return x;
}

void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w) {
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < q; ++i) {
    double xi = -std::cos(pi * (i + 0.75) / (q + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double pn, pnm1;
      legendre2(q, xi, pn, pnm1);
      dp = q * (xi * pn - pnm1) / (xi * xi - 1.0);
      const double dx = pn / dp;
      xi -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    double pn, pnm1;
    legendre2(q, xi, pn, pnm1);
    dp = q * (xi * pn - pnm1) / (xi * xi - 1.0);
    x[i] = xi;
    w[i] = 2.0 / ((1.0 - xi * xi) * dp * dp);
  }
}

RefElem build_ref_elem(int N) {
  if (N < 1 || N > 9) throw std::runtime_error("order N must be in 1..9");
  RefElem E;
  E.N = N;
  E.Np = np_of(N);
  E.Nfp = nfp_of(N);
  const int Np = E.Np, Nfp = E.Nfp;
  warp_blend_nodes(N, E);
  if ((int)E.r.size() != Np) throw std::runtime_error("node count mismatch");

  // Fmask from the exact integer lattice labels (a face node has weight 0 at the opposite vertex)
  const int opposite[4] = {3, 2, 0, 1};
  E.Fmask.resize(4 * Nfp);
  for (int f = 0; f < 4; ++f) {
    int c = 0;
    for (int n = 0; n < Np; ++n)
      if (E.lattice[n][opposite[f]] == 0) {
        if (c >= Nfp) throw std::runtime_error("Fmask overflow");
        E.Fmask[f * Nfp + c++] = n;
      }
    if (c != Nfp) throw std::runtime_error("Fmask count mismatch");
  }

  Mat V, Vr, Vs, Vt;
  basis_rows(N, E.r, E.s, E.t, &V, &Vr, &Vs, &Vt);
  E.Dr = right_solve(Vr, V);
  E.Ds = right_solve(Vs, V);
  E.Dt = right_solve(Vt, V);

  // collapsed Gauss-Legendre quadrature on the tet, exact for degree 2N integrands
  const int q = N + 2;
  std::vector<double> gx, gw;
  gauss_legendre(q, gx, gw);
  std::vector<double> qr, qs, qt, qw;
  for (int ia = 0; ia < q; ++ia)
    for (int ib = 0; ib < q; ++ib)
      for (int ic = 0; ic < q; ++ic) {
        const double a = gx[ia], b = gx[ib], c = gx[ic];
        qr.push_back(0.25 * (1 + a) * (1 - b) * (1 - c) - 1.0);
        qs.push_back(0.5 * (1 + b) * (1 - c) - 1.0);
        qt.push_back(c);
        qw.push_back(gw[ia] * gw[ib] * gw[ic] * (1 - b) * (1 - c) * (1 - c) / 8.0);
      }
  Mat Phi;
  basis_rows(N, qr, qs, qt, &Phi, nullptr, nullptr, nullptr);
  Mat Lq = right_solve(Phi, V);  // Lagrange basis at quadrature points [nq][Np]
  E.M = Mat(Np, Np);
  for (size_t p = 0; p < qw.size(); ++p)
    for (int i = 0; i < Np; ++i) {
      const double li = Lq(p, i) * qw[p];
      for (int j = 0; j < Np; ++j) E.M(i, j) += li * Lq(p, j);
    }

  // face masses in face-parameter coordinates (area-2 reference triangle)
  Mat Emat(Np, 4 * Nfp);
  for (int f = 0; f < 4; ++f) {
    std::vector<double> fr, fs, ft, fw;
    for (int ia = 0; ia < q; ++ia)
      for (int ib = 0; ib < q; ++ib) {
        const double a = gx[ia], b = gx[ib];
        const double u = 0.5 * (1 + a) * (1 - b) - 1.0, v = b;
        const double w = gw[ia] * gw[ib] * (1 - b) / 2.0;
        double r, s, t;
        if (f == 0) { r = u; s = v; t = -1.0; }
        else if (f == 1) { r = u; s = -1.0; t = v; }
        else if (f == 2) { s = u; t = v; r = -1.0 - u - v; }
        else { r = -1.0; s = u; t = v; }
        fr.push_back(r); fs.push_back(s); ft.push_back(t); fw.push_back(w);
      }
    Mat Pf;
    basis_rows(N, fr, fs, ft, &Pf, nullptr, nullptr, nullptr);
    Mat Lf = right_solve(Pf, V);
    Mat Mf(Nfp, Nfp);
    for (size_t p = 0; p < fw.size(); ++p)
      for (int i = 0; i < Nfp; ++i) {
        const double li = Lf(p, E.Fmask[f * Nfp + i]) * fw[p];
        for (int j = 0; j < Nfp; ++j) Mf(i, j) += li * Lf(p, E.Fmask[f * Nfp + j]);
      }
    for (int i = 0; i < Nfp; ++i)
      for (int j = 0; j < Nfp; ++j) Emat(E.Fmask[f * Nfp + i], f * Nfp + j) += Mf(i, j);
    E.face_mass[f] = Mf;
  }
  LU Mf(E.M);
  E.LIFT = Mf.solve(Emat);
  return E;
}

}  // namespace dg
