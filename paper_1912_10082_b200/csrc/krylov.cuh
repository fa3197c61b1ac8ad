// Krylov solvers on device vectors (K4 of SURVEY §2.1): the gmres of
// stk/outer_krylov.hpp:75-164 over arbitrary device operators, and a PCG variant.
// Vector work is deterministic (fixed-grid reductions); the small Hessenberg/Givens
// algebra runs on the host exactly as in the reference.
#pragma once

#include <functional>

#include "common.cuh"

namespace stkg {

using DevOp = std::function<void(const double* x, double* y)>;  // y = op(x), on the stream

struct Krylov {
  int64_t N = 0;
  cudaStream_t stream = nullptr;
  DevBuf V;         // basis, N x v_cap column-major
  int64_t v_cap = 0;
  DevBuf w, z, r, p, q, xk;
  DevBuf hvec, partials, scalars;
  double* pinned = nullptr;
  int pinned_cap = 0;
  // Device flag set when a device-side stopping test fires; operators built on library
  // kernels may pass it to their launches to turn the remaining queued work into no-ops.
  const int* skip = nullptr;
  DevBuf state_buf;  // PCG device scalars
  DevBuf hist_buf;   // device residual history
  Krylov() = default;
  Krylov(const Krylov&) = delete;
  Krylov& operator=(const Krylov&) = delete;
  ~Krylov();
  void ensure(int64_t basis_cols, int64_t hcap);
  void pin(int count);
};

// Deterministic ||x||_2 and x.y (host results).
double knorm(Krylov& k, const double* x);
double kdot(Krylov& k, const double* x, const double* y);

// gmres (stk/outer_krylov.hpp:75-164): same control flow, counters and report fields;
// MGS + one re-orthogonalisation pass run as two classical Gram-Schmidt GEMV passes.
void gmres_run(Krylov& k, const DevOp& apply, const DevOp* precond, const double* b, double* x,
               const stkg_gmres_config& cfg, stkg_report* rep);

// Preconditioned conjugate gradients (apply and precond s.p.d.).
void pcg_run(Krylov& k, const DevOp& apply, const DevOp& precond, const double* b, double* x,
             double tol, int maxit, stkg_report* rep);

}  // namespace stkg
