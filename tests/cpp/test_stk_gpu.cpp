// C++ tests of the host layer stk_gpu.hpp over the C ABI, written against the reference's
// own names (namespace stk) and its SPEC.md known-answer examples.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "stk_gpu.hpp"

static int failures = 0;
#define EXPECT(cond)                                                      \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                         \
    }                                                                     \
  } while (0)

using namespace stk::gpu;

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

int main() {
  // SPEC.md:130 heat_time_matrices N_t=3, T=3
  auto [D, C] = heat_time_matrices(3, 3.0);
  EXPECT(D.diag == std::vector<double>({1, 1, 1}) && D.sup == std::vector<double>({-1, -1}));
  EXPECT(C.diag == std::vector<double>({.5, .5, .5}) && C.sup == std::vector<double>({.5, .5}));
  // SPEC.md:138 fem1d N_h=1 on (0,1): A=[4], M=[1/3]
  auto [M1, A1] = fem1d_matrices(0.0, 1.0, 1);
  EXPECT(std::abs(A1.diag[0] - 4.0) < 1e-15 && std::abs(M1.diag[0] - 1.0 / 3.0) < 1e-15);

  // SPEC.md:307 scalar solve_projected_heat: y = 1
  {
    EigPair e{{1.0}, {1.0}};
    Bidiagonal one{{1.0}, {}};
    auto y = solve_projected_heat_with({e}, one, one, {2.0});
    EXPECT(y.size() == 1 && y[0] == 1.0);
  }
  // 2D P1 heat through HeatPlan: GPU residual <= 1e-12 and host path == device path
  {
    const int n = 47, nt = 20;
    auto [M, A] = fem1d_matrices(0.0, 1.0, n);
    auto [Dt, Ct] = heat_time_matrices(nt, 1.0);
    EigPair e = p1_eigpair(0.0, 1.0, n);
    std::vector<Tridiagonal> ms{M, M}, as{A, A};
    HeatPlan plan({e, e}, Dt, Ct, &ms, &as);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> F(static_cast<size_t>(n) * n * nt);
    for (auto& v : F) v = nd(rng);
    DeviceBuffer dF(F), dU(F.size());
    plan.solve(dF.data(), dU.data());
    double fn = 0;
    const double rr = plan.residual(dU.data(), dF.data(), &fn);
    EXPECT(rr < 1e-12 && fn > 0);
    auto Uh = plan.solve_host(F);
    EXPECT(rel(Uh, dU.download()) == 0.0);
  }
  // rksm_solve: 1D, N_h=10, N_t=6, rank-1 F -> relres <= 1e-8, U matches the
  // direct solve to 1e-6
  {
    const int n = 10, nt = 6;
    auto [M, A] = fem1d_matrices(0.0, 1.0, n);
    auto [Dt, Ct] = heat_time_matrices(nt, 1.0);
    std::vector<Tridiagonal> ms{M}, as{A};
    HeatPlan plan({p1_eigpair(0.0, 1.0, n)}, Dt, Ct, &ms, &as);
    std::vector<double> l(n), r(nt);
    for (int i = 0; i < n; ++i) l[i] = std::sin(0.3 * i + 0.1);
    for (int j = 0; j < nt; ++j) r[j] = 1.0 + 0.5 * j;
    DeviceBuffer dl(l), dr(r), dU(static_cast<size_t>(n) * nt);
    SolveReport rep;
    LowRankDev u = rksm_solve(plan, 1, dl.data(), dr.data(), RksmOptions{}, &rep);
    EXPECT(rep.converged && rep.final_relres <= 1e-8 && u.rank >= 1);
    EXPECT(static_cast<int>(rep.rel_res_history.size()) == rep.iterations);
    std::ostringstream hist;
    write_history_csv(hist, rep);
    EXPECT(hist.str().rfind("iter,relres\n1,", 0) == 0);
    plan.solve_factored(1, dl.data(), dr.data(), dU.data());
    std::vector<double> ud = dU.download(), L = u.left.download(), R = u.right.download();
    std::vector<double> ur(ud.size(), 0.0);  // U (N_h x N_t) = left right^T
    for (int64_t c = 0; c < u.rank; ++c)
      for (int j = 0; j < nt; ++j)
        for (int i = 0; i < n; ++i) ur[static_cast<size_t>(j) * n + i] += L[c * n + i] * R[c * nt + j];
    EXPECT(rel(ur, ud) <= 1e-6);
  }
  // Transform::P1Dst (fast sine transforms) equals Transform::Dense on a 2D P1 grid
  {
    const int n = 63, nt = 8;
    auto pd = heat_plan_p1_uniform(2, n, nt, 1.0, 0.0, 1.0, Transform::Dense);
    auto ps = heat_plan_p1_uniform(2, n, nt, 1.0, 0.0, 1.0, Transform::P1Dst);
    std::mt19937_64 rng(11);
    std::normal_distribution<double> nd;
    std::vector<double> F(static_cast<size_t>(n) * n * nt);
    for (auto& v : F) v = nd(rng);
    DeviceBuffer dF(F), u1(F.size()), u2(F.size());
    pd->solve(dF.data(), u1.data());
    ps->solve(dF.data(), u2.data());
    EXPECT(rel(u2.download(), u1.download()) < 1e-12);
    EXPECT(ps->residual(u2.data(), dF.data()) < 1e-12);
    bool threw = false;
    try {
      auto e = p1_eigpair(0.0, 1.0, n);
      auto dc = heat_time_matrices(nt, 1.0);
      HeatPlan bad({e}, dc.first, dc.second, nullptr, nullptr, nullptr, 0, Transform::P1Dst);
    } catch (const stk::ArgumentError&) {
      threw = true;
    }
    EXPECT(threw);  // P1Dst without p1_h
  }
  // the line-solve schedule (stkg_heat_schedule): a 2D plan with at least 32 column tiles and
  // a mesh-proportional time step takes it, a small plan does not; same solve as Dense
  {
    const int n = 511, nt = 4;
    const double T = nt / 512.0;
    auto pd = heat_plan_p1_uniform(2, n, nt, T, 0.0, 1.0, Transform::Dense);
    auto ps = heat_plan_p1_uniform(2, n, nt, T, 0.0, 1.0, Transform::P1Dst);
    EXPECT(ps->schedule() == STKG_SCHEDULE_LINE_SOLVE);
    EXPECT(pd->schedule() == STKG_SCHEDULE_SEPARATE);
    EXPECT(heat_plan_p1_uniform(2, 63, 8, 1.0, 0.0, 1.0, Transform::P1Dst)->schedule() ==
           STKG_SCHEDULE_SEPARATE);
    std::mt19937_64 rng(13);
    std::normal_distribution<double> nd;
    std::vector<double> F(static_cast<size_t>(n) * n * nt);
    for (auto& v : F) v = nd(rng);
    DeviceBuffer dF(F), u1(F.size()), u2(F.size());
    pd->solve(dF.data(), u1.data());
    ps->solve(dF.data(), u2.data());
    EXPECT(rel(u2.download(), u1.download()) < 2e-12);
    EXPECT(ps->residual(u2.data(), dF.data()) < 1e-11);
  }
  // SingularityError (stk/sylvester.hpp:133-135)
  {
    EigPair e{{2.0}, {1.0}};
    Bidiagonal d{{1.0, 0.0}, {-1.0}}, c{{0.5, 0.0}, {0.5}};
    bool threw = false;
    try {
      solve_projected_heat_with({e}, d, c, {1.0, 1.0});
    } catch (const stk::SingularityError&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // ArgumentError on a shape mismatch
  {
    EigPair e{{1.0, 2.0}, {1, 0, 0, 1}};
    Bidiagonal d{{1.0}, {}};
    bool threw = false;
    try {
      solve_projected_heat_with({e}, d, d, {1.0, 2.0, 3.0});
    } catch (const stk::ArgumentError&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // Wave: the assembled system, PCG and GMRES (WaveOperator + TwoTermPrecond) and the
  // generic VecOp gmres agree on a small instance
  {
    Band7 sp[3], tm[3];
    wave_space_matrices(0.0, 1.0, 24, 3, sp);
    wave_time_matrices(24, 1.0, 3, tm);
    WavePlan plan(sp, tm);
    const int64_t N = plan.space_dim() * plan.time_dim();
    EXPECT(plan.time_dim() == 25);
    std::mt19937_64 rng(3);
    std::normal_distribution<double> nd;
    std::vector<double> b(N);
    for (auto& v : b) v = nd(rng);
    DeviceBuffer db(b), x1(N), x2(N), x3(N);
    GmresConfig cfg;
    cfg.tol = 1e-12;
    cfg.maxit = 500;
    SolveReport r1 = plan.gmres(db.data(), x1.data(), cfg);
    EXPECT(r1.converged && r1.final_relres < 1e-10);
    {
      DeviceBuffer xh(N), xl(N);
      SolveReport rr = plan.solve_refined(db.data(), xh.data(), xl.data(), 1e-13);
      EXPECT(rr.converged && rr.final_relres <= 1e-13);
      EXPECT(plan.residual_dd(db.data(), xh.data(), xl.data()) <= 1e-13);
    }
    for (size_t i = 1; i < r1.rel_res_history.size(); ++i)
      EXPECT(r1.rel_res_history[i] <= r1.rel_res_history[i - 1] * (1 + 1e-12));
    SolveReport r2 = plan.pcg(db.data(), x2.data(), 1e-12, 2000);
    EXPECT(r2.final_relres < 1e-10);
    DeviceVecOp op = [&](const double* x, double* y, void*) { plan.apply(x, y); };
    DeviceVecOp pc = [&](const double* x, double* y, void*) { plan.two_term_solve(x, y); };
    SolveReport r3 = gmres(N, op, &pc, db.data(), x3.data(), cfg);
    EXPECT(r3.converged && r3.iterations == r1.iterations);
    auto h1 = x1.download(), h2 = x2.download(), h3 = x3.download();
    EXPECT(rel(h3, h1) == 0.0);  // same kernels, same order: bit-identical
    EXPECT(rel(h2, h1) < 1e-8);
    {  // the modal banded preconditioner: far fewer PCG iterations, same solution
      DeviceBuffer x4(N);
      plan.use_modal_banded(true);
      SolveReport r4 = plan.pcg(db.data(), x4.data(), 1e-12, 2000);
      plan.use_modal_banded(false);
      EXPECT(r4.converged && r4.final_relres < 1e-10 && 3 * r4.iterations < r2.iterations);
      EXPECT(rel(x4.download(), h1) < 1e-8);
    }
  }
  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("stk_gpu.hpp tests: ALL OK\n");
  return 0;
}
