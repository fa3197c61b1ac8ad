// Internal view of a heat plan shared by the heat solve (heat.cu) and the rational Krylov
// solver (rksm.cu).  Not part of the C ABI.
#pragma once

#include <vector>

#include "common.cuh"

struct stkg_heat;

namespace stkg {

// lambda_i = lam_x[ix] + lam_y[iy] (+ lam_z[iz]) of tensor mode i = (ix*ny + iy)*nz + iz
struct ModeLambda {
  const double* l0;
  const double* l1;
  const double* l2;
  int64_t n1, n2;
  int ndim;
  __device__ __forceinline__ double operator()(int64_t i) const {
    if (ndim == 1) return l0[i];
    if (ndim == 2) return l0[i / n1] + l1[i % n1];
    const int64_t iz = i % n2, r = i / n2;
    return l0[r / n1] + l1[r % n1] + l2[iz];
  }
};


ModeLambda mode_lambda(const stkg_heat& h);
// One axis transform (forward: X_a^T, inverse: X_a) over ntc column blocks of n_x.
void axis_pass(stkg_heat& h, int a, bool forward, const double* src, double* dst, int64_t ntc);
// out_l = M (dd_l U_l + ds_{l-1} U_{l-1}) + A (cd_l U_l + cs_{l-1} U_{l-1}), l < nt, with
// caller-supplied device temporal factors (e.g. dd = 1, cd = 0: out = M U column-wise).
void apply_with_time(stkg_heat& h, const double* U, double* out, int64_t nt, const double* dd,
                     const double* ds, const double* cd, const double* cs);

}  // namespace stkg

struct stkg_heat {
  using DevBuf = stkg::DevBuf;
  int ndim = 0;
  int64_t n[3] = {1, 1, 1};
  int64_t nt = 0;
  int64_t nx = 0;  // spatial unknowns
  cudaStream_t stream = nullptr;
  DevBuf X[3], XT[3], lam[3];
  int transform = STKG_TRANSFORM_DENSE;
  DevBuf inv_mu[3];  // P1_DST: 1/mu_k per axis (folded into the recurrence)
  DevBuf twiddle[3];  // P1_DST: exp(-2 pi i m / 2N) per axis, as double2
  // P1_DST 2D/3D device solve: internal layout with the fastest axis stored at pitch
  // N = n + 1 (0: unpadded); lam/inv_mu of that axis extended by a 0 for the pad lane
  int64_t pitch = 0;
  DevBuf lam_pad, inv_mu_pad;
  DevBuf lam_col, w_col;  // fused axis-0 pass: per-column lambda sum / weight product
  // line-solve axis-0 pass (heat_tridiag.cuh): reciprocal pivots [N_0][columns] and the
  // axis-0 P1 stencil entries; tri_ok: the plan runs it instead of the transform-based pass
  DevBuf tri_iw;
  bool tri_ok = false;
  double tri_md = 0.0, tri_mo = 0.0, tri_ad = 0.0, tri_ao = 0.0;
  bool uniform_time = false;  // all temporal bidiagonal coefficients equal (factored scan)
  DevBuf d_diag, d_sup, c_diag, c_sup;
  // host copies used by the host-side parts of the rational Krylov solver
  std::vector<double> lam_h[3], d_diag_h, d_sup_h, c_diag_h, c_sup_h;
  std::vector<double> m_diag_h[3], m_off_h[3], a_diag_h[3], a_off_h[3];
  bool has_operator = false;
  // rational Krylov workspace (rksm.cu), kept across calls so that repeated solves do not
  // allocate: growable device scratch slots, fixed reduction buffers, pinned staging
  DevBuf rk_slots[16];
  DevBuf rk_partials, rk_hdev, rk_ones, rk_zeros;
  double* rk_pin = nullptr;
  size_t rk_pin_n = 0;
  DevBuf m_diag[3], m_off[3], a_diag[3], a_off[3];
  DevBuf scratch;   // nx * nt, device solve
  DevBuf lfac;      // 2 * nx * rank, transformed load factors (factored solve)
  DevBuf rt;        // nt * rp, the temporal factor transposed and zero-padded (factored solve)
  DevBuf carry;     // nx, modal state y_{l0-1} carried across time chunks
  DevBuf partials;  // reduction partials
  DevBuf scalars;   // device results of reductions
  double* pinned = nullptr;  // host mirror of scalars
  int singular = 0;
  double singular_lambda = 0.0;
  int64_t singular_step = 0;
  // host-buffer pipeline
  int64_t time_chunk = 0;
  DevBuf pf[2], pu[2], ps;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
  // overlapped 2D schedule (run_chunk_padded_overlap): launch-stream / work-ticket overrides
  // read by the DST launchers, high / low priority streams, per-chunk events
  mutable cudaStream_t run_stream = nullptr;
  mutable unsigned long long* run_ticket = nullptr;
  cudaStream_t s_hi = nullptr, s_lo = nullptr;
  std::vector<cudaEvent_t> ov_ev;
  unsigned long long* tickets = nullptr;
  int tickets_n = 0;
  // kernel-class profiling (stkg_heat_profile)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev[2];  // begin/end pairs per class
  int64_t prof_launches[2] = {0, 0};
};

