// stk_gpu.hpp -- header-only C++ host layer over the C ABI (stk_gpu.h).
//
// Re-exposes the GPU hot path under the reference library's own names and semantics
// (namespace stk, /root/reference/proj/include/stk):
//   solve_projected_heat_with   stk/sylvester.hpp:117-142   -> stk::gpu::solve_projected_heat_with
//   KronOp::apply (heat)        stk/sylvester.hpp:32-38     -> stk::gpu::HeatPlan::apply
//   TwoTermPrecond::solve       stk/sylvester.hpp:168-176   -> stk::gpu::WavePlan::two_term_solve
//   (new) modal banded preconditioner                      -> stk::gpu::WavePlan::modal_banded_solve
//   WaveOperator::apply         stk/outer_krylov.hpp:178-186 -> stk::gpu::WavePlan::apply
//   gmres(VecOp, VecOp, b, cfg) stk/outer_krylov.hpp:75-164 -> stk::gpu::gmres
// Failures are rethrown as the reference's exception classes (stk/errors.hpp:9-42).  When
// this header is compiled inside the reference tree those classes are reused; otherwise
// equivalent ones are declared here.  No Eigen dependency: matrices are column-major
// std::vector<double> on the host or raw device pointers.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <ostream>
#include <vector>

#include "stk_gpu.h"

#if __has_include("stk/errors.hpp")
#include "stk/errors.hpp"
#else
namespace stk {
class ArgumentError : public std::invalid_argument {
 public:
  explicit ArgumentError(const std::string& m) : std::invalid_argument(m) {}
};
class DefinitenessError : public std::runtime_error {
 public:
  explicit DefinitenessError(const std::string& m) : std::runtime_error(m) {}
};
class SingularityError : public std::runtime_error {
 public:
  explicit SingularityError(const std::string& m) : std::runtime_error(m) {}
};
class SolvabilityError : public std::runtime_error {
 public:
  explicit SolvabilityError(const std::string& m) : std::runtime_error(m) {}
};
class NumericError : public std::runtime_error {
 public:
  explicit NumericError(const std::string& m) : std::runtime_error(m) {}
};
}  // namespace stk
#endif

namespace stk {
namespace gpu {

class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int status) {
  if (status == STKG_OK) return;
  const std::string msg = stkg_last_error_message();
  switch (status) {
    case STKG_ARGUMENT: throw ArgumentError(msg);
    case STKG_DEFINITENESS: throw DefinitenessError(msg);
    case STKG_SINGULARITY: throw SingularityError(msg);
    case STKG_SOLVABILITY: throw SolvabilityError(msg);
    case STKG_NUMERIC: throw NumericError(msg);
    default: throw CudaError(msg);
  }
}

// ----------------------------------------------------------------- host containers --
struct Bidiagonal {   // upper bidiagonal: diag (n), sup (n-1)
  std::vector<double> diag, sup;
};
struct Tridiagonal {  // symmetric tridiagonal: diag (n), off (n-1)
  std::vector<double> diag, off;
};
struct EigPair {      // stk/types.hpp:126-129; X is n x n column-major
  std::vector<double> lambdas;
  std::vector<double> X;
  int64_t n() const { return static_cast<int64_t>(lambdas.size()); }
};
struct Band7 {        // band[d * n + i] = A(i, i + d - 3)
  std::vector<double> band;
  int64_t n = 0;
};

inline std::pair<Bidiagonal, Bidiagonal> heat_time_matrices(int nt, double T) {
  Bidiagonal d, c;
  d.diag.resize(nt);
  c.diag.resize(nt);
  d.sup.resize(nt > 1 ? nt - 1 : 1);
  c.sup.resize(nt > 1 ? nt - 1 : 1);
  check(stkg_heat_time_matrices(nt, T, d.diag.data(), d.sup.data(), c.diag.data(), c.sup.data()));
  d.sup.resize(nt > 1 ? nt - 1 : 0);
  c.sup.resize(nt > 1 ? nt - 1 : 0);
  return {d, c};
}

inline std::pair<Tridiagonal, Tridiagonal> fem1d_matrices(double a, double b, int nh) {
  Tridiagonal m, s;
  m.diag.resize(nh);
  s.diag.resize(nh);
  m.off.resize(nh > 1 ? nh - 1 : 1);
  s.off.resize(nh > 1 ? nh - 1 : 1);
  check(stkg_fem1d_matrices(a, b, nh, m.diag.data(), m.off.data(), s.diag.data(), s.off.data()));
  m.off.resize(nh > 1 ? nh - 1 : 0);
  s.off.resize(nh > 1 ? nh - 1 : 0);
  return {m, s};
}

inline EigPair p1_eigpair(double a, double b, int nh) {
  EigPair e;
  e.lambdas.resize(nh);
  e.X.resize(static_cast<size_t>(nh) * nh);
  check(stkg_p1_eigpair(a, b, nh, e.X.data(), e.lambdas.data()));
  return e;
}

inline EigPair sym_gen_eig(const std::vector<double>& Q, const std::vector<double>& M, int n) {
  if (Q.size() != static_cast<size_t>(n) * n || M.size() != Q.size())
    throw ArgumentError("sym_gen_eig: size mismatch");
  EigPair e;
  e.lambdas.resize(n);
  e.X.resize(Q.size());
  check(stkg_sym_gen_eig(n, Q.data(), M.data(), e.lambdas.data(), e.X.data()));
  return e;
}

// ------------------------------------------------------------------- device memory --
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t count) : n_(count) {
    void* p = nullptr;
    check(stkg_device_alloc(&p, count * sizeof(double)));
    p_ = static_cast<double*>(p);
  }
  explicit DeviceBuffer(const std::vector<double>& host) : DeviceBuffer(host.size()) {
    upload(host);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p_) stkg_device_free(p_);
  }
  void upload(const std::vector<double>& host) {
    if (host.size() != n_) throw ArgumentError("DeviceBuffer::upload: size mismatch");
    check(stkg_memcpy_h2d(p_, host.data(), n_ * sizeof(double)));
  }
  std::vector<double> download() const {
    std::vector<double> h(n_);
    check(stkg_device_synchronize());
    check(stkg_memcpy_d2h(h.data(), p_, n_ * sizeof(double)));
    return h;
  }
  double* data() { return p_; }
  const double* data() const { return p_; }
  size_t size() const { return n_; }

 private:
  double* p_ = nullptr;
  size_t n_ = 0;
};

// ------------------------------------------------------------------------ heat -------
// Transform backend of a heat plan (stkg_heat_desc::transform).
enum class Transform {
  Dense = STKG_TRANSFORM_DENSE,  // any EigPair: each axis a DMMA GEMM with X / X^T
  P1Dst = STKG_TRANSFORM_P1_DST  // uniform P1 grids: FP64 fast sine transforms (X not read)
};

class HeatPlan {
 public:
  // axes: per-axis EigPairs of the tensor pencil (x slowest); m/a: per-axis 1D factors of
  // KronOp (optional; needed for apply/residual).  transform = P1Dst needs the grid spacing
  // of every axis in p1_h (the closed-form uniform-P1 basis; n + 1 a power of two).
  HeatPlan(const std::vector<EigPair>& axes, const Bidiagonal& d, const Bidiagonal& c,
           const std::vector<Tridiagonal>* m = nullptr, const std::vector<Tridiagonal>* a = nullptr,
           void* stream = nullptr, int64_t time_chunk = 0, Transform transform = Transform::Dense,
           const std::vector<double>* p1_h = nullptr) {
    if (axes.empty() || axes.size() > 3) throw ArgumentError("HeatPlan: 1 to 3 spatial axes");
    if (c.diag.size() != d.diag.size())
      throw ArgumentError("solve_projected_heat: D and C sizes differ");
    stkg_heat_desc desc{};
    desc.ndim = static_cast<int>(axes.size());
    nt_ = static_cast<int64_t>(d.diag.size());
    desc.nt = nt_;
    nx_ = 1;
    for (int i = 0; i < 3; ++i) desc.n[i] = 1;
    for (size_t i = 0; i < axes.size(); ++i) {
      desc.n[i] = axes[i].n();
      nx_ *= axes[i].n();
      if (axes[i].X.size() != static_cast<size_t>(axes[i].n() * axes[i].n()))
        throw ArgumentError("solve_projected_heat: EigPair X shape mismatch");
      desc.X[i] = axes[i].X.data();
      desc.lambdas[i] = axes[i].lambdas.data();
      if (m && a) {
        desc.m_diag[i] = (*m)[i].diag.data();
        desc.m_off[i] = (*m)[i].off.empty() ? (*m)[i].diag.data() : (*m)[i].off.data();
        desc.a_diag[i] = (*a)[i].diag.data();
        desc.a_off[i] = (*a)[i].off.empty() ? (*a)[i].diag.data() : (*a)[i].off.data();
      }
    }
    desc.d_diag = d.diag.data();
    desc.c_diag = c.diag.data();
    desc.d_sup = d.sup.empty() ? d.diag.data() : d.sup.data();
    desc.c_sup = c.sup.empty() ? c.diag.data() : c.sup.data();
    desc.time_chunk = time_chunk;
    desc.transform = static_cast<int>(transform);
    if (transform == Transform::P1Dst) {
      if (!p1_h || p1_h->size() != axes.size())
        throw ArgumentError("HeatPlan: Transform::P1Dst needs p1_h per axis");
      for (size_t i = 0; i < axes.size(); ++i) desc.p1_h[i] = (*p1_h)[i];
    }
    check(stkg_heat_create(&h_, &desc, stream));
  }
  HeatPlan(const HeatPlan&) = delete;
  HeatPlan& operator=(const HeatPlan&) = delete;
  ~HeatPlan() {
    if (h_) stkg_heat_destroy(h_);
  }

  int64_t space_dim() const { return nx_; }
  // STKG_SCHEDULE_* of stkg_heat_solve for this plan (separate passes / fused transform pass /
  // line-solve pass)
  int schedule() const { return stkg_heat_schedule(h_); }
  int64_t time_dim() const { return nt_; }

  void solve(const double* F_dev, double* U_dev) { check(stkg_heat_solve(h_, F_dev, U_dev)); }
  std::vector<double> solve_host(const std::vector<double>& F) {
    if (F.size() != static_cast<size_t>(nx_ * nt_))
      throw ArgumentError("solve_projected_heat: G shape mismatch");
    std::vector<double> U(F.size());
    check(stkg_heat_solve_host(h_, F.data(), U.data()));
    return U;
  }
  void apply(const double* U_dev, double* out_dev) { check(stkg_heat_apply(h_, U_dev, out_dev)); }
  // F = L R^T given as device factors (L: N_h x r, R: N_t x r, column-major): U (N_h x N_t).
  void solve_factored(int64_t rank, const double* L_dev, const double* R_dev, double* U_dev) {
    check(stkg_heat_solve_factored(h_, rank, L_dev, R_dev, U_dev));
  }
  stkg_heat* handle() { return h_; }
  double residual(const double* U_dev, const double* F_dev, double* fnorm = nullptr) {
    double rel = 0.0, fn = 0.0;
    check(stkg_heat_residual(h_, U_dev, F_dev, &rel, &fn));
    if (fnorm) *fnorm = fn;
    return rel;
  }

 private:
  stkg_heat* h_ = nullptr;
  int64_t nx_ = 0, nt_ = 0;
};

// The tensor P1/Q1 heat plan of ndim uniform axes (n interior nodes on (a, b)) and n_t
// backward-difference steps on (0, T), with the spatial factors for apply/residual.
inline std::unique_ptr<HeatPlan> heat_plan_p1_uniform(int ndim, int n, int nt, double T = 1.0,
                                                      double a = 0.0, double b = 1.0,
                                                      Transform transform = Transform::P1Dst,
                                                      void* stream = nullptr) {
  auto dc = heat_time_matrices(nt, T);
  auto ma = fem1d_matrices(a, b, n);
  const EigPair e = p1_eigpair(a, b, n);
  const std::vector<EigPair> axes(static_cast<size_t>(ndim), e);
  const std::vector<Tridiagonal> ms(static_cast<size_t>(ndim), ma.first);
  const std::vector<Tridiagonal> as(static_cast<size_t>(ndim), ma.second);
  const std::vector<double> h(static_cast<size_t>(ndim), (b - a) / (n + 1));
  return std::make_unique<HeatPlan>(axes, dc.first, dc.second, &ms, &as, stream, 0, transform,
                                    &h);
}

// solve_projected_heat_with(eig, d, c, g) with a tensor EigPair and host G (N_h x N_t).
inline std::vector<double> solve_projected_heat_with(const std::vector<EigPair>& axes,
                                                     const Bidiagonal& d, const Bidiagonal& c,
                                                     const std::vector<double>& g) {
  HeatPlan plan(axes, d, c);
  return plan.solve_host(g);
}

// ------------------------------------------------------------------------ wave -------
struct GmresConfig {  // stk/outer_krylov.hpp:18-28
  double tol = 1e-8;
  int maxit = 200;
  int restart = 0;
};

struct SolveReport {  // stk/report.hpp:11-20
  int iterations = 0;
  std::vector<double> rel_res_history;
  int mu_mem = 0;
  int rank = 0;
  double wall_time_s = 0.0;
  double final_relres = 0.0;
  bool converged = false;
  bool stagnated = false;
};

// write_history_csv (stk/report.hpp:22-26)
inline void write_history_csv(std::ostream& os, const SolveReport& report) {
  os << "iter,relres\n";
  for (size_t i = 0; i < report.rel_res_history.size(); ++i)
    os << i + 1 << "," << report.rel_res_history[i] << "\n";
}

namespace detail {
inline SolveReport to_report(const stkg_report& r, std::vector<double>& hist) {
  SolveReport out;
  out.iterations = r.iterations;
  out.mu_mem = r.mu_mem;
  out.final_relres = r.final_relres;
  out.wall_time_s = r.wall_time_s;
  out.converged = r.converged != 0;
  out.stagnated = r.stagnated != 0;
  hist.resize(static_cast<size_t>(std::min(r.history_length, r.history_capacity)));
  out.rel_res_history = hist;
  return out;
}
}  // namespace detail

// rksm_solve (stk/rksm.hpp:104-234) on a HeatPlan built with the spatial factors.
struct RksmOptions {
  double tol = 1e-8;
  int maxit = 100;
  int fixed_iters = 0;  // > 0: preconditioner mode (exactly that many expansions)
  double trunc_tol = 1e-10;
};

// Device low-rank factors U = left * right^T (left: N_h x rank, right: N_t x rank).
struct LowRankDev {
  DeviceBuffer left, right;
  int64_t rank = 0;
};

inline LowRankDev rksm_solve(HeatPlan& plan, int64_t rank, const double* L_dev,
                             const double* R_dev, const RksmOptions& opts = {},
                             SolveReport* report = nullptr) {
  const int64_t cap = std::max<int64_t>(
      1, std::min<int64_t>(std::min(plan.space_dim(), plan.time_dim()),
                           rank * (std::max(opts.maxit, opts.fixed_iters) + 1)));
  LowRankDev out;
  out.left = DeviceBuffer(static_cast<size_t>(cap * plan.space_dim()));
  out.right = DeviceBuffer(static_cast<size_t>(cap * plan.time_dim()));
  stkg_rksm_options o{opts.tol, opts.maxit, opts.fixed_iters, opts.trunc_tol};
  std::vector<double> hist(static_cast<size_t>(std::max(opts.maxit, opts.fixed_iters) + 1));
  stkg_report rep{};
  rep.rel_res_history = hist.data();
  rep.history_capacity = static_cast<int>(hist.size());
  check(stkg_heat_rksm(plan.handle(), rank, L_dev, R_dev, &o, out.left.data(), out.right.data(),
                       cap, &out.rank, &rep));
  if (report) {
    *report = detail::to_report(rep, hist);
    report->rank = static_cast<int>(out.rank);
  }
  return out;
}

class WavePlan {
 public:
  // space = {M_h, A_h, Q_h}, time = {Q_t, D_t, M_t} (wave_space_matrices / wave_time_matrices);
  // with_precond builds TwoTermPrecond's eigenpairs (stk/sylvester.hpp:155-161) on the host.
  WavePlan(const Band7 space[3], const Band7 time[3], bool with_precond = true,
           void* stream = nullptr) {
    nh_ = space[0].n;
    nt_ = time[0].n;
    std::vector<double> sb, tb;
    for (int k = 0; k < 3; ++k) {
      sb.insert(sb.end(), space[k].band.begin(), space[k].band.end());
      tb.insert(tb.end(), time[k].band.begin(), time[k].band.end());
    }
    stkg_wave_desc desc{};
    desc.nh = nh_;
    desc.nt = nt_;
    desc.space_bands = sb.data();
    desc.time_bands = tb.data();
    EigPair es, et;
    if (with_precond) {
      es = sym_gen_eig(dense(space[2]), dense(space[0]), static_cast<int>(nh_));  // (Q_h, M_h)
      et = sym_gen_eig(dense(time[0]), dense(time[2]), static_cast<int>(nt_));    // (Q_t, M_t)
      desc.Xs = es.X.data();
      desc.lambdas = es.lambdas.data();
      desc.Xt = et.X.data();
      desc.thetas = et.lambdas.data();
    }
    stream_ = stream;
    check(stkg_wave_create(&w_, &desc, stream));
  }
  WavePlan(const WavePlan&) = delete;
  WavePlan& operator=(const WavePlan&) = delete;
  ~WavePlan() {
    if (w_) stkg_wave_destroy(w_);
  }

  int64_t space_dim() const { return nh_; }
  int64_t time_dim() const { return nt_; }

  void apply(const double* x, double* y) { check(stkg_wave_apply(w_, x, y)); }
  void two_term_solve(const double* v, double* w) { check(stkg_two_term_solve(w_, v, w)); }
  // The space-modal time-banded preconditioner (no reference counterpart, K2d).
  void modal_banded_solve(const double* v, double* w) {
    check(stkg_modal_banded_solve(w_, v, w));
  }
  // What gmres / pcg / solve_refined apply: false = TwoTermPrecond (default), true = modal.
  void use_modal_banded(bool on) { check(stkg_wave_set_precond(w_, on ? 1 : 0)); }

  SolveReport gmres(const double* b, double* x, const GmresConfig& cfg = {}, bool precond = true) {
    stkg_gmres_config c{cfg.tol, cfg.maxit, cfg.restart, precond ? 1 : 0};
    std::vector<double> hist(static_cast<size_t>(cfg.maxit) + 1);
    stkg_report r{};
    r.rel_res_history = hist.data();
    r.history_capacity = static_cast<int>(hist.size());
    check(stkg_gmres(w_, b, x, &c, &r));
    return detail::to_report(r, hist);
  }
  SolveReport pcg(const double* b, double* x, double tol, int maxit) {
    std::vector<double> hist(static_cast<size_t>(maxit) + 1);
    stkg_report r{};
    r.rel_res_history = hist.data();
    r.history_capacity = static_cast<int>(hist.size());
    check(stkg_pcg(w_, b, x, tol, maxit, &r));
    return detail::to_report(r, hist);
  }
  // ||b - B (x_hi + x_lo)|| / ||b|| with the residual in double-double (x_lo may be null).
  double residual_dd(const double* b, const double* x_hi, const double* x_lo = nullptr,
                     double* r = nullptr) {
    double rel = 0.0;
    check(stkg_wave_residual_dd(w_, b, x_hi, x_lo, r, &rel));
    return rel;
  }
  // Mixed-precision iterative refinement; the solution is the pair x_hi + x_lo.
  SolveReport solve_refined(const double* b, double* x_hi, double* x_lo, double tol = 1e-10,
                            int max_refine = 6, double inner_tol = 1e-6, int inner_maxit = 6000) {
    std::vector<double> hist(static_cast<size_t>(max_refine) + 2);
    stkg_report r{};
    r.rel_res_history = hist.data();
    r.history_capacity = static_cast<int>(hist.size());
    check(stkg_wave_solve_refined(w_, b, x_hi, x_lo, tol, max_refine, inner_tol, inner_maxit, &r));
    return detail::to_report(r, hist);
  }

  static std::vector<double> dense(const Band7& b) {
    std::vector<double> m(static_cast<size_t>(b.n * b.n), 0.0);
    for (int64_t d = 0; d < 7; ++d)
      for (int64_t i = 0; i < b.n; ++i) {
        const int64_t j = i + d - 3;
        if (j >= 0 && j < b.n) m[j * b.n + i] = b.band[d * b.n + i];
      }
    return m;
  }

 private:
  stkg_wave* w_ = nullptr;
  int64_t nh_ = 0, nt_ = 0;
  void* stream_ = nullptr;
};

inline std::pair<Band7, std::pair<Band7, Band7>> band_triple(const std::vector<double>& all, int64_t n) {
  Band7 a{std::vector<double>(all.begin(), all.begin() + 7 * n), n};
  Band7 b{std::vector<double>(all.begin() + 7 * n, all.begin() + 14 * n), n};
  Band7 c{std::vector<double>(all.begin() + 14 * n, all.end()), n};
  return {a, {b, c}};
}

// wave_space_matrices / wave_time_matrices (stk/discretize.hpp:141-161) as bands.
inline void wave_space_matrices(double a, double b, int nh, int degree, Band7 out[3]) {
  std::vector<double> all(static_cast<size_t>(21) * nh);
  check(stkg_wave_space_matrices(a, b, nh, degree, all.data()));
  auto t = band_triple(all, nh);
  out[0] = t.first;
  out[1] = t.second.first;
  out[2] = t.second.second;
}
inline void wave_time_matrices(int nt, double T, int degree, Band7 out[3]) {
  const int n = stkg_wave_time_dim(nt, degree);
  std::vector<double> all(static_cast<size_t>(21) * n);
  check(stkg_wave_time_matrices(nt, T, degree, all.data()));
  auto t = band_triple(all, n);
  out[0] = t.first;
  out[1] = t.second.first;
  out[2] = t.second.second;
}

// gmres(apply, precond, b, cfg) over arbitrary device operators -- the VecOp seam of
// stk/outer_krylov.hpp:30,75.  Operators take device pointers and the CUDA stream.
using DeviceVecOp = std::function<void(const double* x, double* y, void* stream)>;

namespace detail {
inline int call_op(void* user, const double* x, double* y, void* stream) {
  try {
    (*static_cast<const DeviceVecOp*>(user))(x, y, stream);
    return STKG_OK;
  } catch (const ArgumentError&) {
    return STKG_ARGUMENT;
  } catch (...) {
    return STKG_NUMERIC;
  }
}
}  // namespace detail

inline SolveReport gmres(int64_t n, const DeviceVecOp& apply, const DeviceVecOp* precond,
                         const double* b, double* x, const GmresConfig& cfg = {},
                         void* stream = nullptr) {
  stkg_gmres_config c{cfg.tol, cfg.maxit, cfg.restart, precond ? 1 : 0};
  std::vector<double> hist(static_cast<size_t>(cfg.maxit) + 1);
  stkg_report r{};
  r.rel_res_history = hist.data();
  r.history_capacity = static_cast<int>(hist.size());
  check(stkg_gmres_op(n, &detail::call_op, const_cast<DeviceVecOp*>(&apply),
                      precond ? &detail::call_op : nullptr, const_cast<DeviceVecOp*>(precond), b,
                      x, &c, &r, stream));
  return detail::to_report(r, hist);
}

}  // namespace gpu
}  // namespace stk
