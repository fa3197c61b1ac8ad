// Small dense host linear algebra for the rational Krylov solver (rksm.cu): the k x k and
// nt x m problems that stay on the host (the reference does them with Eigen dense types).
// Column-major storage throughout.
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace stkg {
namespace hla {

using Mat = std::vector<double>;  // column-major, dimensions carried by the caller

inline double& at(Mat& a, int ld, int i, int j) { return a[static_cast<size_t>(j) * ld + i]; }
inline double at(const Mat& a, int ld, int i, int j) { return a[static_cast<size_t>(j) * ld + i]; }

// C (m x p) = A (m x q) * B (q x p)
inline Mat matmul(const Mat& A, const Mat& B, int m, int q, int p) {
  Mat C(static_cast<size_t>(m) * p, 0.0);
  for (int j = 0; j < p; ++j)
    for (int l = 0; l < q; ++l) {
      const double b = B[static_cast<size_t>(j) * q + l];
      if (b == 0.0) continue;
      const double* a = &A[static_cast<size_t>(l) * m];
      double* c = &C[static_cast<size_t>(j) * m];
      for (int i = 0; i < m; ++i) c[i] += a[i] * b;
    }
  return C;
}

inline Mat transpose(const Mat& A, int m, int n) {
  Mat T(static_cast<size_t>(m) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) T[static_cast<size_t>(i) * n + j] = A[static_cast<size_t>(j) * m + i];
  return T;
}

inline double frob(const Mat& A) {
  double s = 0.0;
  for (double x : A) s += x * x;
  return std::sqrt(s);
}

// Diagonally pivoted Cholesky of a symmetric positive semi-definite Gram matrix G (m x m):
// G(perm, perm) = R^T R with R upper (rank x m, stored m x m).  Stops when the next pivot
// is <= tol^2 * (largest pivot) -- the Gram-matrix analogue of a rank-revealing QR with
// relative threshold tol on |R_ii|.  Returns the rank.
inline int pivoted_cholesky(Mat G, int m, double tol, std::vector<int>& perm, Mat& R) {
  perm.resize(m);
  std::iota(perm.begin(), perm.end(), 0);
  R.assign(static_cast<size_t>(m) * m, 0.0);
  double first = -1.0;
  int rank = 0;
  for (int k = 0; k < m; ++k) {
    int piv = k;
    for (int i = k + 1; i < m; ++i)
      if (at(G, m, i, i) > at(G, m, piv, piv)) piv = i;
    const double d = at(G, m, piv, piv);
    if (first < 0.0) first = d;
    if (!(d > tol * tol * first) || !(d > 0.0)) break;
    if (piv != k) {  // symmetric swap of rows/cols k and piv, and of the computed R columns
      for (int i = 0; i < m; ++i) std::swap(at(G, m, i, k), at(G, m, i, piv));
      for (int j = 0; j < m; ++j) std::swap(at(G, m, k, j), at(G, m, piv, j));
      for (int i = 0; i < k; ++i) std::swap(at(R, m, i, k), at(R, m, i, piv));
      std::swap(perm[k], perm[piv]);
    }
    const double rkk = std::sqrt(at(G, m, k, k));
    at(R, m, k, k) = rkk;
    for (int j = k + 1; j < m; ++j) at(R, m, k, j) = at(G, m, k, j) / rkk;
    for (int i = k + 1; i < m; ++i)
      for (int j = k + 1; j < m; ++j) at(G, m, i, j) -= at(R, m, k, i) * at(R, m, k, j);
    rank = k + 1;
  }
  return rank;
}

// Plain Cholesky G = R^T R (R upper).  Returns false when G is not (numerically) s.p.d.
inline bool cholesky_upper(const Mat& G, int m, Mat& R) {
  R.assign(static_cast<size_t>(m) * m, 0.0);
  for (int j = 0; j < m; ++j) {
    for (int i = 0; i <= j; ++i) {
      double s = at(G, m, i, j);
      for (int k = 0; k < i; ++k) s -= at(R, m, k, i) * at(R, m, k, j);
      if (i == j) {
        if (!(s > 0.0)) return false;
        at(R, m, j, j) = std::sqrt(s);
      } else {
        at(R, m, i, j) = s / at(R, m, i, i);
      }
    }
  }
  return true;
}

// Inverse of an upper triangular r x r matrix stored with leading dimension ld.
inline Mat upper_inverse(const Mat& R, int r, int ld) {
  Mat X(static_cast<size_t>(r) * r, 0.0);
  for (int j = r - 1; j >= 0; --j) {
    at(X, r, j, j) = 1.0 / at(R, ld, j, j);
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += at(R, ld, i, k) * at(X, r, k, j);
      at(X, r, i, j) = -s / at(R, ld, i, i);
    }
  }
  return X;
}

// R factor (n x n upper) of a Householder QR of A (m x n, m >= n); A is destroyed.
inline Mat householder_r(Mat A, int m, int n) {
  const int kmax = std::min(m, n);
  for (int k = 0; k < kmax; ++k) {
    double norm = 0.0;
    for (int i = k; i < m; ++i) norm += at(A, m, i, k) * at(A, m, i, k);
    norm = std::sqrt(norm);
    if (norm == 0.0) continue;
    const double alpha = at(A, m, k, k) > 0 ? -norm : norm;
    std::vector<double> v(m - k);
    for (int i = k; i < m; ++i) v[i - k] = at(A, m, i, k);
    v[0] -= alpha;
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn == 0.0) continue;
    for (int j = k; j < n; ++j) {
      double s = 0.0;
      for (int i = k; i < m; ++i) s += v[i - k] * at(A, m, i, j);
      s = 2.0 * s / vn;
      for (int i = k; i < m; ++i) at(A, m, i, j) -= s * v[i - k];
    }
  }
  Mat R(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= std::min(j, m - 1); ++i) at(R, n, i, j) = at(A, m, i, j);
  return R;
}

// One-sided Jacobi SVD of A (m x n, m >= n): A = U diag(s) V^T, s descending.
inline void jacobi_svd(Mat A, int m, int n, std::vector<double>& s, Mat& U, Mat& V) {
  V.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) at(V, n, i, i) = 1.0;
  const double eps = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = 0; i < m; ++i) {
          const double x = at(A, m, i, p), y = at(A, m, i, q);
          a += x * x;
          b += y * y;
          c += x * y;
        }
        if (c == 0.0 || std::abs(c) <= eps * std::sqrt(a * b)) continue;
        off = std::max(off, std::abs(c) / std::sqrt(a * b));
        const double zeta = (b - a) / (2.0 * c);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (int i = 0; i < m; ++i) {
          const double x = at(A, m, i, p), y = at(A, m, i, q);
          at(A, m, i, p) = cs * x - sn * y;
          at(A, m, i, q) = sn * x + cs * y;
        }
        for (int i = 0; i < n; ++i) {
          const double x = at(V, n, i, p), y = at(V, n, i, q);
          at(V, n, i, p) = cs * x - sn * y;
          at(V, n, i, q) = sn * x + cs * y;
        }
      }
    if (off <= eps) break;
  }
  s.assign(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double x = 0.0;
    for (int i = 0; i < m; ++i) x += at(A, m, i, j) * at(A, m, i, j);
    s[j] = std::sqrt(x);
  }
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return s[x] > s[y]; });
  Mat U2(static_cast<size_t>(m) * n, 0.0), V2(static_cast<size_t>(n) * n), s2(n);
  for (int c = 0; c < n; ++c) {
    const int j = order[c];
    s2[c] = s[j];
    for (int i = 0; i < m; ++i) at(U2, m, i, c) = s[j] > 0 ? at(A, m, i, j) / s[j] : 0.0;
    for (int i = 0; i < n; ++i) at(V2, n, i, c) = at(V, n, i, j);
  }
  s = s2;
  U = U2;
  V = V2;
}

}  // namespace hla
}  // namespace stkg
