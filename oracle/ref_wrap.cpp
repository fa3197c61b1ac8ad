// ref_wrap.cpp -- TEST INFRASTRUCTURE: a C shim over the parts of the reference that compile
// here as-is (stk/splines.hpp, stk/quadrature.hpp, stk/errors.hpp).  Built by
// oracle/Makefile straight from the sources under /root/reference into oracle/_ref/; the
// reference sources are never copied into this repository.
//
// spline_gram (stk/discretize.hpp:111-131) cannot be compiled (discretize.hpp pulls in
// Eigen through types.hpp), so its loop is restated here verbatim in structure, but every
// basis value and quadrature node comes from the reference's own SplineBasis/gauss_legendre.
#include <cstring>
#include <stdexcept>

#include "stk/quadrature.hpp"
#include "stk/splines.hpp"

namespace {
// triplet-order accumulation == Eigen setFromTriplets' duplicate summation order
void gram(const stk::SplineBasis& basis, int d_row, int d_col, double* band) {
  const int n = basis.num_active();
  std::memset(band, 0, sizeof(double) * 7 * n);
  const stk::QuadRule ref = stk::gauss_legendre(basis.degree() + 1, 0.0, 1.0);
  for (int e = 0; e < basis.num_elems(); ++e) {
    const auto funcs = basis.active_on_element(e);
    const double xl = basis.elem_left(e), xr = basis.elem_right(e);
    for (size_t qi = 0; qi < ref.nodes.size(); ++qi) {
      const double x = xl + (xr - xl) * ref.nodes[qi];
      const double w = (xr - xl) * ref.weights[qi];
      for (const auto& [ja, ia] : funcs) {
        const double vi = basis.eval_full(ia, x, d_row);
        for (const auto& [jb, ib] : funcs) {
          const double vj = basis.eval_full(ib, x, d_col);
          band[(jb - ja + 3) * n + ja] += w * vi * vj;
        }
      }
    }
  }
}
}  // namespace

extern "C" {

// wave_space_matrices(wave_space_basis(SpaceGrid1D(a,b,nh), degree)): [M | A | Q]
int ref_wave_space_bands(double a, double b, int nh, int degree, double* bands) {
  try {
    const int n_elems = nh + 2 - degree;
    stk::SplineBasis basis(degree, n_elems, a, b, stk::SplineBasis::EndConditions::zero_value_both);
    const int n = basis.num_active();
    gram(basis, 0, 0, bands);
    gram(basis, 1, 1, bands + 7 * n);
    gram(basis, 2, 2, bands + 14 * n);
    return n;
  } catch (const std::exception&) {
    return -1;
  }
}

// wave_time_matrices(wave_time_basis(TimeGrid(nt,T), degree)): [Q | D | M]
int ref_wave_time_bands(int nt, double T, int degree, double* bands) {
  try {
    stk::SplineBasis basis(degree, nt, 0.0, T,
                           stk::SplineBasis::EndConditions::zero_value_slope_right);
    const int n = basis.num_active();
    gram(basis, 2, 2, bands);
    gram(basis, 2, 0, bands + 7 * n);
    gram(basis, 0, 0, bands + 14 * n);
    return n;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_gauss_legendre(int npoints, double a, double b, double* nodes, double* weights) {
  try {
    const stk::QuadRule r = stk::gauss_legendre(npoints, a, b);
    for (int i = 0; i < npoints; ++i) {
      nodes[i] = r.nodes[i];
      weights[i] = r.weights[i];
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// value/derivative of active function j of a basis (ec: 0 none, 1 right value+slope, 2 both)
int ref_spline_eval(int degree, int n_elems, double a, double b, int ec, int j, double x,
                    int deriv, double* out) {
  try {
    stk::SplineBasis basis(degree, n_elems, a, b,
                           static_cast<stk::SplineBasis::EndConditions>(ec));
    *out = basis.eval(j, x, deriv);
    return basis.num_active();
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
