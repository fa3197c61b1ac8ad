/*
 * stk_oracle.c -- CPU restatement of the reference algorithms on the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA product path
 * (paper_1912_10082_b200/).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product never links it.
 *
 * The reference (`stk`, /root/reference/proj/include/stk) cannot be built here: it needs
 * Eigen3 and CLI11, both absent.  Each function below restates the cited
 * reference function loop-for-loop over plain arrays; sparse matrices are materialised in
 * CSR in the index order of sparse_kron (stk/types.hpp:131-145), as the reference does.
 * Parity anchors: the SPEC.md known-answer examples (tests/golden/spec_kats.json) and the
 * reference's own splines/quadrature code compiled as oracle/_ref (wave bands).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------- stk/discretize.hpp:44-57 ----- */
void or_heat_time_matrices(int nt, double T, double* d_diag, double* d_sup, double* c_diag,
                           double* c_sup) {
  const double dt = T / nt;
  for (int k = 0; k < nt; ++k) {
    d_diag[k] = 1.0;
    c_diag[k] = dt / 2.0;
    if (k + 1 < nt) {
      d_sup[k] = -1.0;
      c_sup[k] = dt / 2.0;
    }
  }
}

/* ---------------------------------------------------- stk/discretize.hpp:61-77 ----- */
void or_fem1d_matrices(double a, double b, int nh, double* m_diag, double* m_off,
                       double* a_diag, double* a_off) {
  const double h = (b - a) / (nh + 1);
  for (int i = 0; i < nh; ++i) {
    m_diag[i] = 2.0 * h / 3.0;
    a_diag[i] = 2.0 / h;
    if (i + 1 < nh) {
      m_off[i] = h / 6.0;
      a_off[i] = -1.0 / h;
    }
  }
}

/* ------------------------------------------------------------ CSR sparse matrices --- */
typedef struct {
  int64_t n;
  int64_t* rowptr;
  int64_t* col;
  double* val;
} csr_t;

static void csr_free(csr_t* m) {
  free(m->rowptr);
  free(m->col);
  free(m->val);
}

/* tridiagonal 1D factor as CSR */
static csr_t csr_tri(int64_t n, const double* diag, const double* off) {
  csr_t m;
  m.n = n;
  m.rowptr = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  m.col = (int64_t*)malloc(sizeof(int64_t) * 3 * n);
  m.val = (double*)malloc(sizeof(double) * 3 * n);
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    m.rowptr[i] = k;
    if (i > 0) { m.col[k] = i - 1; m.val[k++] = off[i - 1]; }
    m.col[k] = i; m.val[k++] = diag[i];
    if (i + 1 < n) { m.col[k] = i + 1; m.val[k++] = off[i]; }
  }
  m.rowptr[n] = k;
  return m;
}

/* sparse_kron (stk/types.hpp:131-145): entry (ia*nb + ib, ja*nb + jb) = A(ia,ja) B(ib,jb) */
static csr_t csr_kron(const csr_t* A, const csr_t* B) {
  csr_t m;
  m.n = A->n * B->n;
  const int64_t nnz = A->rowptr[A->n] * B->rowptr[B->n];
  m.rowptr = (int64_t*)malloc(sizeof(int64_t) * (m.n + 1));
  m.col = (int64_t*)malloc(sizeof(int64_t) * nnz);
  m.val = (double*)malloc(sizeof(double) * nnz);
  int64_t k = 0;
  for (int64_t ia = 0; ia < A->n; ++ia)
    for (int64_t ib = 0; ib < B->n; ++ib) {
      m.rowptr[ia * B->n + ib] = k;
      for (int64_t p = A->rowptr[ia]; p < A->rowptr[ia + 1]; ++p)
        for (int64_t q = B->rowptr[ib]; q < B->rowptr[ib + 1]; ++q) {
          m.col[k] = A->col[p] * B->n + B->col[q];
          m.val[k++] = A->val[p] * B->val[q];
        }
    }
  m.rowptr[m.n] = k;
  return m;
}

/* C = A + B, same sparsity union (both sorted by column per row) */
static csr_t csr_add(const csr_t* A, const csr_t* B) {
  csr_t m;
  m.n = A->n;
  const int64_t cap = A->rowptr[A->n] + B->rowptr[B->n];
  m.rowptr = (int64_t*)malloc(sizeof(int64_t) * (m.n + 1));
  m.col = (int64_t*)malloc(sizeof(int64_t) * cap);
  m.val = (double*)malloc(sizeof(double) * cap);
  int64_t k = 0;
  for (int64_t i = 0; i < m.n; ++i) {
    m.rowptr[i] = k;
    int64_t p = A->rowptr[i], q = B->rowptr[i];
    const int64_t pe = A->rowptr[i + 1], qe = B->rowptr[i + 1];
    while (p < pe || q < qe) {
      if (q >= qe || (p < pe && A->col[p] < B->col[q])) {
        m.col[k] = A->col[p]; m.val[k++] = A->val[p++];
      } else if (p >= pe || B->col[q] < A->col[p]) {
        m.col[k] = B->col[q]; m.val[k++] = B->val[q++];
      } else {
        m.col[k] = A->col[p]; m.val[k++] = A->val[p++] + B->val[q++];
      }
    }
  }
  m.rowptr[m.n] = k;
  return m;
}

/* fem2d_matrices (stk/discretize.hpp:81-88) and its 3D restatement:
 * M = Mx (x) My (x) Mz, A = Ax (x) My (x) Mz + Mx (x) Ay (x) Mz + Mx (x) My (x) Az. */
static void tensor_mats(int ndim, const int64_t* n, const double* const* md, const double* const* mo,
                        const double* const* ad, const double* const* ao, csr_t* M, csr_t* A) {
  csr_t m[3], a[3];
  for (int i = 0; i < ndim; ++i) {
    m[i] = csr_tri(n[i], md[i], mo[i]);
    a[i] = csr_tri(n[i], ad[i], ao[i]);
  }
  if (ndim == 1) {
    *M = m[0];
    *A = a[0];
    return;
  }
  if (ndim == 2) {
    *M = csr_kron(&m[0], &m[1]);
    csr_t t1 = csr_kron(&a[0], &m[1]), t2 = csr_kron(&m[0], &a[1]);
    *A = csr_add(&t1, &t2);
    csr_free(&t1); csr_free(&t2);
  } else {
    csr_t mxy = csr_kron(&m[0], &m[1]);
    *M = csr_kron(&mxy, &m[2]);
    csr_t axy = csr_kron(&a[0], &m[1]), may = csr_kron(&m[0], &a[1]);
    csr_t t1 = csr_kron(&axy, &m[2]), t2 = csr_kron(&may, &m[2]), t3 = csr_kron(&mxy, &a[2]);
    csr_t s12 = csr_add(&t1, &t2);
    *A = csr_add(&s12, &t3);
    csr_free(&mxy); csr_free(&axy); csr_free(&may); csr_free(&t1); csr_free(&t2);
    csr_free(&t3); csr_free(&s12);
  }
  for (int i = 0; i < ndim; ++i) { csr_free(&m[i]); csr_free(&a[i]); }
}

static void csr_mv(const csr_t* A, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A->n; ++i) {
    double s = 0.0;
    for (int64_t p = A->rowptr[i]; p < A->rowptr[i + 1]; ++p) s += A->val[p] * x[A->col[p]];
    y[i] = s;
  }
}

/* KronOp::apply (stk/sylvester.hpp:32-38) of heat_kron_op (:58-65): out = M U D + A U C
 * with D, C upper bidiagonal: (U D)[:, l] = d_l U_l + ds_{l-1} U_{l-1}.  Evaluated as the
 * reference does: (M U) first (sparse x dense), then the temporal factor. */
void or_heat_apply(int ndim, const int64_t* n, int64_t nt, const double* const* md,
                   const double* const* mo, const double* const* ad, const double* const* ao,
                   const double* d_diag, const double* d_sup, const double* c_diag,
                   const double* c_sup, const double* U, double* out) {
  csr_t M, A;
  tensor_mats(ndim, n, md, mo, ad, ao, &M, &A);
  const int64_t nx = M.n;
  double* mu = (double*)malloc(sizeof(double) * nx * 2);
  double* au = (double*)malloc(sizeof(double) * nx * 2);
  /* mu[l%2] = M U_l, au[l%2] = A U_l */
  for (int64_t l = 0; l < nt; ++l) {
    double* mc = mu + (l % 2) * nx;
    double* ac = au + (l % 2) * nx;
    csr_mv(&M, U + l * nx, mc);
    csr_mv(&A, U + l * nx, ac);
    const double* mp = mu + ((l + 1) % 2) * nx;
    const double* ap = au + ((l + 1) % 2) * nx;
    double* o = out + l * nx;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nx; ++i) {
      double s = mc[i] * d_diag[l] + ac[i] * c_diag[l];
      if (l > 0) s += mp[i] * d_sup[l - 1] + ap[i] * c_sup[l - 1];
      o[i] = s;
    }
  }
  free(mu);
  free(au);
  csr_free(&M);
  csr_free(&A);
}

/* solve_projected_heat_with (stk/sylvester.hpp:117-142) with a dense EigPair (k x k X):
 * gt = X^T G; per mode forward substitution; Y = X yt.  Returns 3 on a singular pivot. */
int or_solve_projected_heat_with(int64_t k, int64_t nt, const double* X, const double* lam,
                                 const double* d_diag, const double* d_sup, const double* c_diag,
                                 const double* c_sup, const double* G, double* Y) {
  double* gt = (double*)malloc(sizeof(double) * k * nt);
  double* yt = (double*)malloc(sizeof(double) * k * nt);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < nt; ++j)
    for (int64_t i = 0; i < k; ++i) {
      double s = 0.0;
      for (int64_t r = 0; r < k; ++r) s += X[i * k + r] * G[j * k + r];
      gt[j * k + i] = s;
    }
  int status = 0;
  for (int64_t i = 0; i < k && !status; ++i) {
    const double l = lam[i];
    for (int64_t j = 0; j < nt; ++j) {
      const double piv = d_diag[j] + l * c_diag[j];
      if (fabs(piv) < 1e-300) { status = 3; break; }
      double rhs = gt[j * k + i];
      if (j > 0) rhs -= (d_sup[j - 1] + l * c_sup[j - 1]) * yt[(j - 1) * k + i];
      yt[j * k + i] = rhs / piv;
    }
  }
  if (!status) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < nt; ++j)
      for (int64_t i = 0; i < k; ++i) {
        double s = 0.0;
        for (int64_t r = 0; r < k; ++r) s += X[r * k + i] * yt[j * k + r];
        Y[j * k + i] = s;
      }
  }
  free(gt);
  free(yt);
  return status;
}

/* crank_nicolson (stk/cn_baseline.hpp:26-48) for the tensor P1/Q1 heat system:
 * (M + dt/2 A) u^l = (M - dt/2 A) u^{l-1} + F[:, l], factor once.  SimplicialLLT is
 * replaced by a banded Cholesky (half-bandwidth = product of the faster axis sizes),
 * exact for this band structure.  Runs nsteps <= nt steps (causal prefix).
 * Returns 2 if the matrix is not s.p.d. */
int or_crank_nicolson(int ndim, const int64_t* n, int64_t nsteps, double dt,
                      const double* const* md, const double* const* mo, const double* const* ad,
                      const double* const* ao, const double* F, double* U) {
  csr_t M, A;
  tensor_mats(ndim, n, md, mo, ad, ao, &M, &A);
  const int64_t N = M.n;
  int64_t bw = 0; /* half-bandwidth of the sparsity pattern */
  for (int64_t i = 0; i < N; ++i)
    for (int64_t p = M.rowptr[i]; p < M.rowptr[i + 1]; ++p)
      if (i - M.col[p] > bw) bw = i - M.col[p];
  /* lower band of L: Lb[i*w + (i-j)] = L(i, j), j in [i-bw, i] */
  const int64_t w = bw + 1;
  double* Lb = (double*)calloc((size_t)(N * w), sizeof(double));
  for (int64_t i = 0; i < N; ++i) {
    /* lhs = M + (dt/2) A on the (shared) tensor stencil pattern, lower part */
    for (int64_t p = M.rowptr[i]; p < M.rowptr[i + 1]; ++p) {
      const int64_t j = M.col[p];
      if (j > i) continue;
      double a = 0.0;
      for (int64_t q = A.rowptr[i]; q < A.rowptr[i + 1]; ++q)
        if (A.col[q] == j) a = A.val[q];
      Lb[i * w + (i - j)] = M.val[p] + (dt / 2.0) * a;
    }
  }
  /* banded Cholesky, row-oriented */
  for (int64_t i = 0; i < N; ++i) {
    const int64_t j0 = i - bw > 0 ? i - bw : 0;
    for (int64_t j = j0; j <= i; ++j) {
      double s = Lb[i * w + (i - j)];
      for (int64_t k = j0; k < j; ++k) s -= Lb[i * w + (i - k)] * Lb[j * w + (j - k)];
      if (j == i) {
        if (!(s > 0.0)) { free(Lb); csr_free(&M); csr_free(&A); return 2; }
        Lb[i * w] = sqrt(s);
      } else {
        Lb[i * w + (i - j)] = s / Lb[j * w];
      }
    }
  }
  double* u = (double*)calloc((size_t)N, sizeof(double));
  double* b = (double*)malloc(sizeof(double) * N);
  double* mu = (double*)malloc(sizeof(double) * N);
  double* au = (double*)malloc(sizeof(double) * N);
  for (int64_t l = 0; l < nsteps; ++l) {
    csr_mv(&M, u, mu);
    csr_mv(&A, u, au);
    const double* f = F + l * N;
    for (int64_t i = 0; i < N; ++i) b[i] = (mu[i] - (dt / 2.0) * au[i]) + f[i];
    /* L y = b */
    for (int64_t i = 0; i < N; ++i) {
      double s = b[i];
      const int64_t j0 = i - bw > 0 ? i - bw : 0;
      for (int64_t j = j0; j < i; ++j) s -= Lb[i * w + (i - j)] * b[j];
      b[i] = s / Lb[i * w];
    }
    /* L^T u = y */
    for (int64_t i = N - 1; i >= 0; --i) {
      double s = b[i];
      const int64_t j1 = i + bw < N - 1 ? i + bw : N - 1;
      for (int64_t j = i + 1; j <= j1; ++j) s -= Lb[j * w + (j - i)] * u[j];
      u[i] = s / Lb[i * w];
    }
    memcpy(U + l * N, u, sizeof(double) * N);
  }
  free(u); free(b); free(mu); free(au); free(Lb);
  csr_free(&M);
  csr_free(&A);
  return 0;
}

/* --------------------------------------------------------------------- wave ------- */
/* band layout: band[d*n + i] = Mat(i, i + d - 3) */
static double band_at(const double* band, int64_t n, int64_t i, int64_t j) {
  const int64_t d = j - i + 3;
  if (d < 0 || d > 6 || i < 0 || i >= n || j < 0 || j >= n) return 0.0;
  return band[d * n + i];
}

/* WaveOperator::apply (stk/outer_krylov.hpp:178-186):
 * out = M_h U Q_t^T + A_h U E + Q_h U M_t, E = D_t + D_t^T; each term as (S U) then x T. */
void or_wave_apply(int64_t nh, int64_t nt, const double* sb /* M|A|Q */,
                   const double* tb /* Q|D|M */, const double* U, double* out) {
  const double* S[3] = {sb, sb + 7 * nh, sb + 14 * nh};
  const double* Qt = tb;
  const double* Dt = tb + 7 * nt;
  const double* Mt = tb + 14 * nt;
  double* su = (double*)malloc(sizeof(double) * nh * nt);
  memset(out, 0, sizeof(double) * nh * nt);
  for (int term = 0; term < 3; ++term) {
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < nt; ++l)
      for (int64_t i = 0; i < nh; ++i) {
        double s = 0.0;
        for (int64_t k = i - 3; k <= i + 3; ++k)
          if (k >= 0 && k < nh) s += band_at(S[term], nh, i, k) * U[l * nh + k];
        su[l * nh + i] = s;
      }
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < nt; ++j)
      for (int64_t i = 0; i < nh; ++i) {
        double s = 0.0;
        for (int64_t l = j - 3; l <= j + 3; ++l) {
          if (l < 0 || l >= nt) continue;
          double t;
          if (term == 0) t = band_at(Qt, nt, j, l);                          /* Q_t^T(l,j)=Q_t(j,l) */
          else if (term == 1) t = band_at(Dt, nt, l, j) + band_at(Dt, nt, j, l); /* E(l,j) */
          else t = band_at(Mt, nt, l, j);                                    /* M_t(l,j) */
          s += su[l * nh + i] * t;
        }
        out[j * nh + i] += s;
      }
  }
  free(su);
}

/* --------------------------------------------------------------- generator -------- */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

void or_fill_uniform(double* dst, int64_t count, uint64_t seed, uint64_t stream, int64_t off) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t x = splitmix64(seed ^ (stream << 40) ^ (uint64_t)(off + i));
    dst[i] = 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
  }
}
