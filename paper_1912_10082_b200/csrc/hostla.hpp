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
  // columns of C are independent: threads split them once the product is large enough
#pragma omp parallel for schedule(static) if (static_cast<double>(m) * q * p > 4e6)
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
