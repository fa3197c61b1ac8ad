// Host-side assembly (layer L1 of SURVEY §1) for the B200 plans: the temporal and spatial
// factors and eigenpairs the GPU kernels consume.  This is product code (not the oracle):
// it restates, without Eigen, the reference functions cited per entry point, producing
// plain arrays for the C ABI of include/stk_gpu.h.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "../../include/stk_gpu.h"

namespace stkg {
void set_error(const std::string& msg);  // errors.cpp
}

namespace {

struct Failure {
  int code;
  std::string msg;
};

template <typename F>
int run(F&& body) {
  try {
    body();
    return STKG_OK;
  } catch (const Failure& f) {
    stkg::set_error(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    stkg::set_error(e.what());
    return STKG_NUMERIC;
  }
}

[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

// ------------------------------------------------------------------ Gauss-Legendre --
// gauss_legendre (stk/quadrature.hpp:17-64): Newton iteration on the three-term Legendre
// recurrence from the Chebyshev-like initial guess, symmetric fill, affine map to (a,b).
// The operation sequence is kept identical so the spline Gram bands are bit-identical to
// the reference's (checked against oracle/_ref by
// tests/test_host_cpu.py::test_wave_bands_bit_identical_to_reference).
struct Rule {
  std::vector<double> x, w;
};

void legendre_at(int n, double x, double& pn, double& pnm1) {
  double p_prev = 1.0, p = x;
  for (int k = 2; k <= n; ++k) {
    const double p_next = ((2.0 * k - 1.0) * x * p - (k - 1.0) * p_prev) / k;
    p_prev = p;
    p = p_next;
  }
  pn = p;
  pnm1 = p_prev;
}

Rule gauss_rule(int n, double a, double b) {
  if (n < 1) fail(STKG_ARGUMENT, "gauss_legendre: npoints must be >= 1");
  Rule r;
  r.x.assign(n, 0.0);
  r.w.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double pn, pm;
      legendre_at(n, x, pn, pm);
      const double dp = n * (x * pn - pm) / (x * x - 1.0);
      const double dx = pn / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    double pn, pm;
    legendre_at(n, x, pn, pm);
    const double dp = n * (x * pn - pm) / (x * x - 1.0);
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    r.x[i] = -x;
    r.x[n - 1 - i] = x;
    r.w[i] = w;
    r.w[n - 1 - i] = w;
  }
  if (n % 2 == 1) r.x[n / 2] = 0.0;
  const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
  for (int i = 0; i < n; ++i) {
    r.x[i] = mid + half * r.x[i];
    r.w[i] *= half;
  }
  return r;
}

// ------------------------------------------------------------------ B-spline basis --
// Clamped uniform B-spline space of SplineBasis (stk/splines.hpp:17-119): knots = degree
// copies of a, the n_elems+1 uniform breakpoints, degree copies of b; end conditions by
// dropping functions (last two: rho(T)=rho'(T)=0; first and last: zero at both ends).
class Splines {
 public:
  enum Ends { kNone, kRightValueSlope, kBothValues };

  Splines(int degree, int n_elems, double a, double b, Ends ends)
      : p_(degree), ne_(n_elems), a_(a), b_(b) {
    if (degree != 2 && degree != 3) fail(STKG_ARGUMENT, "SplineBasis: degree must be 2 or 3");
    if (n_elems < 1) fail(STKG_ARGUMENT, "SplineBasis: need at least one element");
    if (!(b > a)) fail(STKG_ARGUMENT, "SplineBasis: empty interval");
    const double h = (b - a) / n_elems;
    t_.assign(degree, a);
    for (int i = 0; i <= n_elems; ++i) t_.push_back(a + i * h);
    t_.insert(t_.end(), degree, b);
    const int full = n_elems + degree;
    int first = 0, last = full;  // active = [first, last)
    if (ends == kRightValueSlope) last = full - 2;
    if (ends == kBothValues) first = 1, last = full - 1;
    if (last - first < 1)
      fail(STKG_ARGUMENT, "SplineBasis: too few basis functions left after end conditions");
    first_ = first;
    last_ = last;
  }

  int degree() const { return p_; }
  int elems() const { return ne_; }
  int active() const { return last_ - first_; }
  double h() const { return (b_ - a_) / ne_; }
  double left(int e) const { return a_ + e * h(); }
  double right(int e) const { return a_ + (e + 1) * h(); }

  // (active index, full index) pairs supported on element e, ascending.
  void on_element(int e, std::vector<std::pair<int, int>>& out) const {
    out.clear();
    for (int i = std::max(e, first_); i <= std::min(e + p_, last_ - 1); ++i)
      out.emplace_back(i - first_, i);
  }

  // d-th derivative of full-basis function i at x (Cox-de Boor recursion).
  double eval(int i, int k, int d, double x) const {
    if (k == 0) {
      if (d != 0) return 0.0;
      const double lo = t_[i], hi = t_[i + 1];
      if (lo <= x && x < hi) return 1.0;
      if (x == b_ && lo < hi && hi == b_) return 1.0;  // closed last interval
      return 0.0;
    }
    const double span_l = t_[i + k] - t_[i];
    const double span_r = t_[i + k + 1] - t_[i + 1];
    double acc = 0.0;
    if (d > 0) {
      if (span_l > 0.0) acc += eval(i, k - 1, d - 1, x) / span_l;
      if (span_r > 0.0) acc -= eval(i + 1, k - 1, d - 1, x) / span_r;
      return k * acc;
    }
    if (span_l > 0.0) acc += (x - t_[i]) / span_l * eval(i, k - 1, 0, x);
    if (span_r > 0.0) acc += (t_[i + k + 1] - x) / span_r * eval(i + 1, k - 1, 0, x);
    return acc;
  }

 private:
  int p_, ne_;
  double a_, b_;
  std::vector<double> t_;
  int first_ = 0, last_ = 0;
};

// spline_gram (stk/discretize.hpp:111-131) accumulated straight into a 7-diagonal band:
// band[(c - r + 3) * n + r] = sum over (element, quad point) of w * B_r^(dr) * B_c^(dc), in
// the reference's triplet order (element, quad point, row, column), which is the order in
// which setFromTriplets sums duplicate entries.
void gram_band(const Splines& s, int dr, int dc, double* band) {
  const int n = s.active();
  std::fill(band, band + 7 * static_cast<size_t>(n), 0.0);
  const Rule ref = gauss_rule(s.degree() + 1, 0.0, 1.0);
  std::vector<std::pair<int, int>> funcs;
  for (int e = 0; e < s.elems(); ++e) {
    s.on_element(e, funcs);
    const double xl = s.left(e), xr = s.right(e);
    for (size_t q = 0; q < ref.x.size(); ++q) {
      const double x = xl + (xr - xl) * ref.x[q];
      const double w = (xr - xl) * ref.w[q];
      for (const auto& [ja, ia] : funcs) {
        const double vi = s.eval(ia, s.degree(), dr, x);
        for (const auto& [jb, ib] : funcs) {
          const double vj = s.eval(ib, s.degree(), dc, x);
          band[static_cast<size_t>(jb - ja + 3) * n + ja] += w * vi * vj;
        }
      }
    }
  }
}

// ------------------------------------------------------------- dense eigensolver ----
// Householder tridiagonalisation of a symmetric matrix (row-major a, overwritten by the
// accumulated orthogonal transform) followed by implicit QL with Wilkinson-type shifts.
// Together: a = Z diag(d) Z^T with the eigenvectors in the columns of a (row-major).
void householder_tridiag(int n, std::vector<double>& a, std::vector<double>& d,
                         std::vector<double>& e) {
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) * n + j]; };
  d.assign(n, 0.0);
  e.assign(n, 0.0);
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    double h = 0.0;
    if (l > 0) {
      double scale = 0.0;
      for (int k = 0; k <= l; ++k) scale += std::abs(A(i, k));
      if (scale == 0.0) {
        e[i] = A(i, l);
      } else {
        for (int k = 0; k <= l; ++k) {
          A(i, k) /= scale;
          h += A(i, k) * A(i, k);
        }
        const double f = A(i, l);
        const double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        A(i, l) = f - g;
        double fsum = 0.0;
        for (int j = 0; j <= l; ++j) {
          A(j, i) = A(i, j) / h;
          double gj = 0.0;
          for (int k = 0; k <= j; ++k) gj += A(j, k) * A(i, k);
          for (int k = j + 1; k <= l; ++k) gj += A(k, j) * A(i, k);
          e[j] = gj / h;
          fsum += e[j] * A(i, j);
        }
        const double hh = fsum / (h + h);
        for (int j = 0; j <= l; ++j) {
          const double fj = A(i, j);
          const double gj = e[j] - hh * fj;
          e[j] = gj;
          for (int k = 0; k <= j; ++k) A(j, k) -= fj * e[k] + gj * A(i, k);
        }
      }
    } else {
      e[i] = A(i, l);
    }
    d[i] = h;
  }
  d[0] = 0.0;
  e[0] = 0.0;
  for (int i = 0; i < n; ++i) {
    const int l = i - 1;
    if (d[i] != 0.0) {
      for (int j = 0; j <= l; ++j) {
        double g = 0.0;
        for (int k = 0; k <= l; ++k) g += A(i, k) * A(k, j);
        for (int k = 0; k <= l; ++k) A(k, j) -= g * A(k, i);
      }
    }
    d[i] = A(i, i);
    A(i, i) = 1.0;
    for (int j = 0; j <= l; ++j) A(j, i) = A(i, j) = 0.0;
  }
}

// zt holds Z^T (row k = eigenvector k), so each plane rotation touches two contiguous rows.
void tridiag_ql(int n, std::vector<double>& d, std::vector<double>& e,
                std::vector<double>& zt) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  if (n > 0) e[n - 1] = 0.0;
  const double eps = std::numeric_limits<double>::epsilon();
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
        if (std::abs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (iter++ == 60) fail(STKG_NUMERIC, "sym_gen_eig: eigendecomposition did not converge");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          double* zi = &zt[static_cast<size_t>(i) * n];
          double* zi1 = &zt[static_cast<size_t>(i + 1) * n];
          for (int k = 0; k < n; ++k) {
            f = zi1[k];
            zi1[k] = s * zi[k] + c * f;
            zi[k] = c * zi[k] - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
}

void require_symmetric(int n, const double* a, const char* who) {
  double asym = 0.0, scale = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double x = a[static_cast<size_t>(j) * n + i], y = a[static_cast<size_t>(i) * n + j];
      asym += (x - y) * (x - y);
      scale += x * x;
    }
  if (std::sqrt(asym) > 1e-12 * (scale > 0 ? std::sqrt(scale) : 1.0))
    fail(STKG_ARGUMENT, std::string(who) + ": matrix is not symmetric");
}

double sinpi_ratio(int64_t r, int64_t N) {
  // sin(pi * r / N) for integer r, with exact integer range reduction
  int64_t m = r % (2 * N);
  if (m < 0) m += 2 * N;
  double sign = 1.0;
  if (m >= N) {
    m -= N;
    sign = -1.0;
  }
  if (2 * m > N) m = N - m;
  return sign * std::sin(M_PI * static_cast<double>(m) / static_cast<double>(N));
}

}  // namespace

extern "C" {

int stkg_heat_time_matrices(int nt, double T, double* d_diag, double* d_sup, double* c_diag,
                            double* c_sup) {
  return run([&] {
    if (nt < 1) fail(STKG_ARGUMENT, "TimeGrid: nt must be >= 1");
    if (!(T > 0)) fail(STKG_ARGUMENT, "TimeGrid: T must be positive");
    const double dt = T / nt;  // TimeGrid::dt (stk/discretize.hpp:22)
    for (int k = 0; k < nt; ++k) {
      d_diag[k] = 1.0;
      c_diag[k] = dt / 2.0;
      if (k + 1 < nt) {
        d_sup[k] = -1.0;
        c_sup[k] = dt / 2.0;
      }
    }
  });
}

int stkg_fem1d_matrices(double a, double b, int nh, double* m_diag, double* m_off,
                        double* a_diag, double* a_off) {
  return run([&] {
    if (!(b > a)) fail(STKG_ARGUMENT, "SpaceGrid1D: empty interval");
    if (nh < 1) fail(STKG_ARGUMENT, "SpaceGrid1D: nh must be >= 1");
    const double h = (b - a) / (nh + 1);  // SpaceGrid1D::fem_h (stk/discretize.hpp:38)
    for (int i = 0; i < nh; ++i) {
      m_diag[i] = 2.0 * h / 3.0;
      a_diag[i] = 2.0 / h;
      if (i + 1 < nh) {
        m_off[i] = h / 6.0;
        a_off[i] = -1.0 / h;
      }
    }
  });
}

int stkg_p1_eigpair(double a, double b, int nh, double* X, double* lambdas) {
  return run([&] {
    if (!(b > a)) fail(STKG_ARGUMENT, "SpaceGrid1D: empty interval");
    if (nh < 1) fail(STKG_ARGUMENT, "SpaceGrid1D: nh must be >= 1");
    const int64_t N = nh + 1;
    const double h = (b - a) / N;
    const double norm = std::sqrt(2.0 / static_cast<double>(N));
    for (int k = 1; k <= nh; ++k) {
      const double s_half = sinpi_ratio(k, 2 * N);  // sin(theta_k / 2)
      const double c = std::cos(M_PI * static_cast<double>(k) / static_cast<double>(N));
      const double mu = (h / 3.0) * (2.0 + c);       // eigenvalue of M_h
      lambdas[k - 1] = 12.0 * s_half * s_half / (h * h * (2.0 + c));
      const double scale = norm / std::sqrt(mu);
      double* col = X + static_cast<size_t>(k - 1) * nh;
      for (int i = 1; i <= nh; ++i) col[i - 1] = scale * sinpi_ratio(static_cast<int64_t>(i) * k, N);
    }
  });
}

int stkg_sym_gen_eig(int n, const double* Q, const double* M, double* lambdas, double* X) {
  return run([&] {
    if (n < 1) fail(STKG_ARGUMENT, "sym_gen_eig: size mismatch");
    require_symmetric(n, Q, "sym_gen_eig(Q)");
    require_symmetric(n, M, "sym_gen_eig(M)");
    const size_t nn = static_cast<size_t>(n) * n;
    // Cholesky M = L L^T, L stored row-major lower.
    std::vector<double> L(nn, 0.0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        double s = M[static_cast<size_t>(j) * n + i];
        for (int k = 0; k < j; ++k) s -= L[static_cast<size_t>(i) * n + k] * L[static_cast<size_t>(j) * n + k];
        if (i == j) {
          if (!(s > 0.0)) fail(STKG_DEFINITENESS, "sym_gen_eig: M is not s.p.d.");
          L[static_cast<size_t>(i) * n + i] = std::sqrt(s);
        } else {
          L[static_cast<size_t>(i) * n + j] = s / L[static_cast<size_t>(j) * n + j];
        }
      }
    // W = L^-1 Q (column by column), then B = L^-1 W^T = L^-1 Q L^-T.  Row-major work arrays.
    std::vector<double> W(nn), B(nn);
    auto forward = [&](const double* rhs_col, size_t stride, double* out_row_major_col) {
      // solve L y = rhs; rhs element i at rhs_col[i*stride]; y written to out[i*n]
      for (int i = 0; i < n; ++i) {
        double s = rhs_col[i * stride];
        const double* li = &L[static_cast<size_t>(i) * n];
        for (int k = 0; k < i; ++k) s -= li[k] * out_row_major_col[static_cast<size_t>(k) * n];
        out_row_major_col[static_cast<size_t>(i) * n] = s / li[i];
      }
    };
    for (int j = 0; j < n; ++j) forward(Q + static_cast<size_t>(j) * n, 1, &W[j]);  // W(i,j)
    // B(:, j) = L^-1 (W^T)(:, j) = L^-1 W(j, :)^T
    for (int j = 0; j < n; ++j) forward(&W[static_cast<size_t>(j) * n], 1, &B[j]);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) {
        const double s = 0.5 * (B[static_cast<size_t>(i) * n + j] + B[static_cast<size_t>(j) * n + i]);
        B[static_cast<size_t>(i) * n + j] = s;
        B[static_cast<size_t>(j) * n + i] = s;
      }
    std::vector<double> d, e;
    householder_tridiag(n, B, d, e);
    // B now holds Z (row-major, eigenvectors in columns); QL rotates Z^T rows.
    std::vector<double> zt(nn);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) zt[static_cast<size_t>(j) * n + i] = B[static_cast<size_t>(i) * n + j];
    tridiag_ql(n, d, e, zt);
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d[x] < d[y]; });
    // X = L^-T V: back substitution L^T x = v per eigenvector.
    std::vector<double> v(n);
    for (int c = 0; c < n; ++c) {
      const int k = order[c];
      lambdas[c] = d[k];
      const double* zk = &zt[static_cast<size_t>(k) * n];
      double* xc = X + static_cast<size_t>(c) * n;
      for (int i = n - 1; i >= 0; --i) {
        double s = zk[i];
        for (int r = i + 1; r < n; ++r) s -= L[static_cast<size_t>(r) * n + i] * xc[r];
        xc[i] = s / L[static_cast<size_t>(i) * n + i];
      }
    }
  });
}

int stkg_wave_space_matrices(double a, double b, int nh, int degree, double* bands) {
  return run([&] {
    const int n_elems = nh + 2 - degree;  // wave_space_basis (stk/discretize.hpp:99-104)
    if (n_elems < 1) fail(STKG_ARGUMENT, "wave_space_basis: nh too small for degree");
    if (degree < 2) fail(STKG_ARGUMENT, "wave_space_matrices: degree >= 2 required");
    Splines s(degree, n_elems, a, b, Splines::kBothValues);
    const size_t w = 7 * static_cast<size_t>(s.active());
    gram_band(s, 0, 0, bands);          // M = (psi, psi)
    gram_band(s, 1, 1, bands + w);      // A = (psi', psi')
    gram_band(s, 2, 2, bands + 2 * w);  // Q = (psi'', psi'')
  });
}

int stkg_wave_time_dim(int nt, int degree) { return nt + degree - 2; }

int stkg_wave_time_matrices(int nt, double T, int degree, double* bands) {
  return run([&] {
    if (nt < 1) fail(STKG_ARGUMENT, "TimeGrid: nt must be >= 1");
    if (!(T > 0)) fail(STKG_ARGUMENT, "TimeGrid: T must be positive");
    Splines s(degree, nt, 0.0, T, Splines::kRightValueSlope);  // wave_time_basis (:92-95)
    const size_t w = 7 * static_cast<size_t>(s.active());
    gram_band(s, 2, 2, bands);          // Q = (rho'', rho'')
    gram_band(s, 2, 0, bands + w);      // D = (rho'', rho)
    gram_band(s, 0, 0, bands + 2 * w);  // M = (rho, rho)
  });
}

}  // extern "C"
