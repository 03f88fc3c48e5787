/*
 * oracle/kkt_oracle.c — TEST INFRASTRUCTURE ONLY: the plain-C restatement of
 * the reference hot path (see kkt_oracle.h).  Each function cites the
 * reference source it restates (paths relative to /root/reference/proj).
 * Compiled with -ffp-contract=off (oracle/Makefile): products and sums are
 * separately rounded exactly as in the reference's x86-64 build.
 */
#define _GNU_SOURCE
#include "kkt_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- errors */
static __thread char g_err[512];
static __thread int g_err_index = -1;

static int fail(int st, int index, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
#include <stdarg.h>
static int fail(int st, int index, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_err_index = index;
  return st;
}
const char* orc_error(void) { return g_err; }
int orc_error_index(void) { return g_err_index; }

#define TRY(x)                \
  do {                        \
    int st_ = (x);            \
    if (st_) return st_;      \
  } while (0)

static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s);
  if (!p) abort();
  return p;
}

/* ---------------------------------------------- banded matrices (linalg) */
/* BandedMatrix (include/kktdd/linalg.hpp:21-42): column-compressed band,
 * entry (i,j) at data[j*(kl+ku+1) + (i-j+ku)]. */
typedef struct {
  int n, kl, ku;
  double* data;
} band_t;

static int band_in(const band_t* A, int i, int j) {
  return i >= 0 && i < A->n && j >= 0 && j < A->n && i - j <= A->kl && j - i <= A->ku;
}
static double band_at(const band_t* A, int i, int j) {
  return band_in(A, i, j) ? A->data[(size_t)j * (A->kl + A->ku + 1) + (i - j + A->ku)] : 0.0;
}
static double* band_ref(band_t* A, int i, int j) {
  return &A->data[(size_t)j * (A->kl + A->ku + 1) + (i - j + A->ku)];
}
static void band_zero(band_t* A, int n, int kl, int ku) {
  A->n = n;
  A->kl = kl;
  A->ku = ku;
  A->data = xcalloc((size_t)n * (kl + ku + 1), sizeof(double));
}
/* BandedMatrix::norm_inf (linalg.cpp:35-43) */
static double band_norm_inf(const band_t* A) {
  double best = 0.0;
  for (int i = 0; i < A->n; ++i) {
    double row = 0.0;
    int lo = i - A->kl > 0 ? i - A->kl : 0, hi = i + A->ku < A->n - 1 ? i + A->ku : A->n - 1;
    for (int j = lo; j <= hi; ++j) row += fabs(band_at(A, i, j));
    if (row > best) best = row;
  }
  return best;
}
/* band_matvec (linalg.cpp:45-54): the whole band, zeros included */
static void band_matvec(const band_t* A, const double* x, double* y) {
  for (int i = 0; i < A->n; ++i) {
    double acc = 0.0;
    int jlo = i - A->kl > 0 ? i - A->kl : 0, jhi = i + A->ku < A->n - 1 ? i + A->ku : A->n - 1;
    for (int j = jlo; j <= jhi; ++j) acc += band_at(A, i, j) * x[j];
    y[i] = acc;
  }
}
/* band_matvec_transpose (linalg.cpp:56-67) */
static void band_matvec_t(const band_t* A, const double* x, double* y) {
  for (int i = 0; i < A->n; ++i) {
    double acc = 0.0;
    int jlo = i - A->ku > 0 ? i - A->ku : 0, jhi = i + A->kl < A->n - 1 ? i + A->kl : A->n - 1;
    for (int j = jlo; j <= jhi; ++j) acc += band_at(A, j, i) * x[j];
    y[i] = acc;
  }
}

/* BandedLU (linalg.hpp:47-75, linalg.cpp:69-162) */
typedef struct {
  int n, kl, ku; /* ku = fill-extended kl + ku */
  double* ab;
  int* piv;
  double growth;
} blu_t;
#define LU_E(F, i, j) ((F)->ab[(size_t)(j) * ((F)->kl + (F)->ku + 1) + ((i) - (j) + (F)->ku)])

static int blu_factor(blu_t* F, const band_t* A) {
  const int n = A->n;
  F->n = n;
  F->kl = A->kl;
  F->ku = (n > 0 ? n - 1 : 0) < A->ku + A->kl ? (n > 0 ? n - 1 : 0) : A->ku + A->kl;
  const int ld = F->kl + F->ku + 1;
  F->ab = xcalloc((size_t)n * ld, sizeof(double));
  F->piv = xcalloc((size_t)n, sizeof(int));
  for (int j = 0; j < n; ++j) {
    int lo = j - A->ku > 0 ? j - A->ku : 0, hi = j + A->kl < n - 1 ? j + A->kl : n - 1;
    for (int i = lo; i <= hi; ++i) LU_E(F, i, j) = band_at(A, i, j);
  }
  const double tol = 1e-14 * band_norm_inf(A);
  double umax = 0.0, amax = 0.0;
  for (size_t k = 0; k < (size_t)n * ld; ++k)
    if (fabs(F->ab[k]) > amax) amax = fabs(F->ab[k]);
  for (int j = 0; j < n; ++j) {
    int p = j;
    double best = fabs(LU_E(F, j, j));
    const int imax = n - 1 < j + F->kl ? n - 1 : j + F->kl;
    const int jmax = n - 1 < j + F->ku ? n - 1 : j + F->ku;
    for (int i = j + 1; i <= imax; ++i) {
      double v = fabs(LU_E(F, i, j));
      if (v > best) {
        best = v;
        p = i;
      }
    }
    F->piv[j] = p;
    if (!(best > tol))
      return fail(KKT_ESINGULAR, j, "banded LU: pivot %g at index %d below tolerance %g", best, j, tol);
    if (p != j)
      for (int c = j; c <= jmax; ++c) {
        double t = LU_E(F, j, c);
        LU_E(F, j, c) = LU_E(F, p, c);
        LU_E(F, p, c) = t;
      }
    const double d = LU_E(F, j, j);
    if (fabs(d) > umax) umax = fabs(d);
    for (int i = j + 1; i <= imax; ++i) LU_E(F, i, j) /= d;
    for (int c = j + 1; c <= jmax; ++c) {
      const double ujc = LU_E(F, j, c);
      if (fabs(ujc) > umax) umax = fabs(ujc);
      if (ujc != 0.0) {
        double* col = &LU_E(F, j + 1, c);
        const double* mul = &LU_E(F, j + 1, j);
        for (int i = 0; i <= imax - j - 1; ++i) col[i] -= mul[i] * ujc;
      }
    }
  }
  F->growth = amax > 0.0 ? umax / amax : 0.0;
  return 0;
}

static void blu_solve(const blu_t* F, double* b) { /* linalg.cpp:127-145 */
  const int n = F->n;
  for (int j = 0; j < n; ++j) {
    if (F->piv[j] != j) {
      double t = b[j];
      b[j] = b[F->piv[j]];
      b[F->piv[j]] = t;
    }
    const double bj = b[j];
    if (bj != 0.0) {
      int hi = n - 1 < j + F->kl ? n - 1 : j + F->kl;
      for (int i = j + 1; i <= hi; ++i) b[i] -= LU_E(F, i, j) * bj;
    }
  }
  for (int j = n - 1; j >= 0; --j) {
    b[j] /= LU_E(F, j, j);
    const double bj = b[j];
    if (bj != 0.0) {
      int lo = j - F->ku > 0 ? j - F->ku : 0;
      for (int i = lo; i < j; ++i) b[i] -= LU_E(F, i, j) * bj;
    }
  }
}

static void blu_solve_t(const blu_t* F, double* b) { /* linalg.cpp:147-162 */
  const int n = F->n;
  for (int j = 0; j < n; ++j) {
    double acc = b[j];
    int lo = j - F->ku > 0 ? j - F->ku : 0;
    for (int i = lo; i < j; ++i) acc -= LU_E(F, i, j) * b[i];
    b[j] = acc / LU_E(F, j, j);
  }
  for (int j = n - 1; j >= 0; --j) {
    double acc = b[j];
    int hi = n - 1 < j + F->kl ? n - 1 : j + F->kl;
    for (int i = j + 1; i <= hi; ++i) acc -= LU_E(F, i, j) * b[i];
    b[j] = acc;
    if (F->piv[j] != j) {
      double t = b[j];
      b[j] = b[F->piv[j]];
      b[F->piv[j]] = t;
    }
  }
}

/* DenseLU (linalg.cpp:199-249), row-major */
typedef struct {
  int n;
  double* lu;
  int* piv;
} dlu_t;

static int dlu_factor(dlu_t* F, const double* A, int n) {
  F->n = n;
  F->lu = xcalloc((size_t)n * n, sizeof(double));
  memcpy(F->lu, A, sizeof(double) * (size_t)n * n);
  F->piv = xcalloc((size_t)n, sizeof(int));
  double anorm = 0.0;
  for (int i = 0; i < n; ++i) {
    double row = 0.0;
    for (int j = 0; j < n; ++j) row += fabs(A[(size_t)i * n + j]);
    if (row > anorm) anorm = row;
  }
  const double tol = 1e-14 * anorm;
#define DA(i, j) F->lu[(size_t)(i) * n + (j)]
  for (int j = 0; j < n; ++j) {
    int p = j;
    double best = fabs(DA(j, j));
    for (int i = j + 1; i < n; ++i)
      if (fabs(DA(i, j)) > best) {
        best = fabs(DA(i, j));
        p = i;
      }
    F->piv[j] = p;
    if (!(best > tol)) return fail(KKT_ESINGULAR, j, "dense LU: pivot below tolerance at index %d", j);
    if (p != j)
      for (int c = 0; c < n; ++c) {
        double t = DA(j, c);
        DA(j, c) = DA(p, c);
        DA(p, c) = t;
      }
    const double d = DA(j, j);
    for (int i = j + 1; i < n; ++i) {
      const double l = DA(i, j) / d;
      DA(i, j) = l;
      for (int c = j + 1; c < n; ++c) DA(i, c) -= l * DA(j, c);
    }
  }
  return 0;
}

static void dlu_solve(const dlu_t* F, double* b) {
  const int n = F->n;
  for (int j = 0; j < n; ++j) {
    if (F->piv[j] != j) {
      double t = b[j];
      b[j] = b[F->piv[j]];
      b[F->piv[j]] = t;
    }
    const double bj = b[j];
    for (int i = j + 1; i < n; ++i) b[i] -= DA(i, j) * bj;
  }
  for (int j = n - 1; j >= 0; --j) {
    b[j] /= DA(j, j);
    const double bj = b[j];
    for (int i = 0; i < j; ++i) b[i] -= DA(i, j) * bj;
  }
}
#undef DA

static double dot(const double* a, const double* b, size_t n) { /* linalg.cpp:372-378 */
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}
static double norm2(const double* a, size_t n) { return sqrt(dot(a, a, n)); }
static void axpy(double alpha, const double* x, double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

/* ------------------------------------------------------------- context */
typedef struct {
  kkt_problem_desc d;
  int nx, ny, nsp, Nt, Nd, m;
  size_t B;
  double dt, ms, shift;
  band_t A, Ahat;
  blu_t F; /* Ahat factors */
  /* TimePartition (time_partition.cpp:61-86) */
  int *nfirst, *nlast, *ofirst, *olast, *efirst, *elast, *owner;
  /* CoarseSpace (schur.hpp:244-285) */
  int has_coarse, variant, ncols;
  int *col_s, *col_kind, *col_dof;
  double **phi_c, **phi_l;
  int* phi_len;
  double* S0;       /* dense (scalar) or densified (per-dof, for coarse_matrix) */
  int sparse;       /* per-dof: banded LU of the CSR envelope */
  dlu_t S0d;
  blu_t S0s;
} orc_t;

/* ProblemConfig::validate (config.cpp:5-22) */
static int validate(const kkt_problem_desc* d) {
  if (d->Nx < 2 || d->Ny < 2) return fail(KKT_ECONFIG, -1, "mesh needs Nx, Ny >= 2, got Nx=%d Ny=%d", d->Nx, d->Ny);
  if (d->Lx <= 0 || d->Ly <= 0 || d->T <= 0) return fail(KKT_ECONFIG, -1, "domain extents and T must be positive");
  if (d->Nt < 1) return fail(KKT_ECONFIG, -1, "Nt must be >= 1, got %d", d->Nt);
  if (d->Nd < 1) return fail(KKT_ECONFIG, -1, "Nd must be >= 1, got %d", d->Nd);
  if (d->Nt % d->Nd) return fail(KKT_ECONFIG, -1, "Nt=%d is not divisible by Nd=%d", d->Nt, d->Nd);
  if (d->nu < 0) return fail(KKT_ECONFIG, -1, "conductivity nu must be >= 0");
  if (!(d->omega > 0)) return fail(KKT_ECONFIG, -1, "regularization omega must be > 0");
  if (!(d->tol > 0)) return fail(KKT_ECONFIG, -1, "gmres tol must be > 0");
  if (d->max_iters < 1) return fail(KKT_ECONFIG, -1, "gmres max_iters must be >= 1");
  if (d->restart != KKT_NO_RESTART && d->restart < 1) return fail(KKT_ECONFIG, -1, "gmres restart must be >= 1");
  return 0;
}

/* assemble_spatial_operator (heat_operators.cpp:24-44) */
static void assemble_A(const orc_t* c, band_t* A) {
  const int nx = c->nx, ny = c->ny;
  const double dx = c->d.Lx / c->d.Nx, dy = c->d.Ly / c->d.Ny;
  const double cx = c->dt * c->d.nu / (dx * dx);
  const double cy = c->dt * c->d.nu / (dy * dy);
  const int bw = ny > 1 ? nx : (nx > 1 ? 1 : 0);
  band_zero(A, nx * ny, bw, bw);
  for (int j = 1; j <= ny; ++j)
    for (int i = 1; i <= nx; ++i) {
      const int p = (j - 1) * nx + (i - 1);
      *band_ref(A, p, p) = 1.0 + 2.0 * cx + 2.0 * cy;
      if (i > 1) *band_ref(A, p, p - 1) = -cx;
      if (i < nx) *band_ref(A, p, p + 1) = -cx;
      if (j > 1) *band_ref(A, p, p - nx) = -cy;
      if (j < ny) *band_ref(A, p, p + nx) = -cy;
    }
}

static int build_coarse(orc_t* c);

int orc_create(const kkt_problem_desc* d, void** out) {
  TRY(validate(d));
  if (d->precond == KKT_PRECOND_DENSE_SCHUR || d->precond == KKT_PRECOND_TRUE_SCHUR)
    return fail(KKT_EUNSUPPORTED, -1, "dense Schur kinds are not restated");
  orc_t* c = xcalloc(1, sizeof(orc_t));
  c->d = *d;
  c->nx = d->Nx - 1;
  c->ny = d->Ny - 1;
  c->nsp = c->nx * c->ny;
  c->Nt = d->Nt;
  c->Nd = d->Nd;
  c->m = d->Nt / d->Nd;
  c->B = (size_t)c->Nt * c->nsp;
  c->dt = d->T / d->Nt;
  c->ms = c->dt * (d->Lx / d->Nx) * (d->Ly / d->Ny); /* mass_scale (config.hpp:58) */
  c->shift = (d->jhat_sign == KKT_SIGN_PLUS ? 1.0 : -1.0) / sqrt(d->omega);
  assemble_A(c, &c->A);
  /* make_ahat (heat_operators.cpp:16-20) */
  band_zero(&c->Ahat, c->A.n, c->A.kl, c->A.ku);
  memcpy(c->Ahat.data, c->A.data, sizeof(double) * (size_t)c->A.n * (c->A.kl + c->A.ku + 1));
  for (int i = 0; i < c->Ahat.n; ++i) *band_ref(&c->Ahat, i, i) -= c->shift * c->dt;
  int st = blu_factor(&c->F, &c->Ahat);
  if (st) {
    orc_destroy(c);
    return st;
  }
  /* partition */
  c->nfirst = xcalloc(c->Nd, sizeof(int));
  c->nlast = xcalloc(c->Nd, sizeof(int));
  c->ofirst = xcalloc(c->Nd, sizeof(int));
  c->olast = xcalloc(c->Nd, sizeof(int));
  c->efirst = xcalloc(c->Nd, sizeof(int));
  c->elast = xcalloc(c->Nd, sizeof(int));
  c->owner = xcalloc(c->Nt + 1, sizeof(int));
  for (int n = 1; n <= c->Nt; ++n) c->owner[n] = (n - 1) / c->m;
  for (int s = 0; s < c->Nd; ++s) {
    c->nlast[s] = (s + 1) * c->m;
    c->nfirst[s] = s == 0 ? 1 : s * c->m;
    c->ofirst[s] = s == 0 ? 1 : s * c->m + 1;
    c->olast[s] = c->nlast[s];
    const int wf = c->nfirst[s] - 1;
    c->efirst[s] = wf >= 1 ? wf : c->nfirst[s];
    c->elast[s] = c->nlast[s];
  }
  if (d->precond == KKT_PRECOND_TWO_LEVEL) {
    st = build_coarse(c);
    if (st) {
      orc_destroy(c);
      return st == KKT_ESINGULAR ? KKT_ECONFIG : st;
    }
  }
  *out = c;
  return 0;
}

static void blu_free(blu_t* F) {
  free(F->ab);
  free(F->piv);
}

void orc_destroy(void* vc) {
  orc_t* c = vc;
  if (!c) return;
  free(c->A.data);
  free(c->Ahat.data);
  blu_free(&c->F);
  free(c->nfirst); free(c->nlast); free(c->ofirst); free(c->olast);
  free(c->efirst); free(c->elast); free(c->owner);
  if (c->phi_c) {
    for (int s = 0; s < c->Nd; ++s) {
      free(c->phi_c[s]);
      free(c->phi_l[s]);
    }
  }
  free(c->phi_c); free(c->phi_l); free(c->phi_len);
  free(c->col_s); free(c->col_kind); free(c->col_dof);
  free(c->S0);
  free(c->S0d.lu); free(c->S0d.piv);
  blu_free(&c->S0s);
  free(c);
}

int64_t orc_block(void* vc) { return (int64_t)((orc_t*)vc)->B; }

/* ------------------------------------------------------ heat operators */
#define NODE(n) ((size_t)((n)-1) * nsp)

/* apply_J / apply_Jhat (heat_operators.cpp:57-69, 111-123) */
static void time_lower(const orc_t* c, const band_t* A, const double* u, double* out) {
  const int nsp = c->nsp;
  for (int n = 1; n <= c->Nt; ++n) {
    band_matvec(A, u + NODE(n), out + NODE(n));
    if (n > 1)
      for (int p = 0; p < nsp; ++p) out[NODE(n) + p] -= u[NODE(n - 1) + p];
  }
}
/* apply_JT / apply_JhatT (:71-83, 125-137) */
static void time_upper(const orc_t* c, const band_t* A, const double* w, double* out) {
  const int nsp = c->nsp;
  for (int n = 1; n <= c->Nt; ++n) {
    band_matvec_t(A, w + NODE(n), out + NODE(n));
    if (n < c->Nt)
      for (int p = 0; p < nsp; ++p) out[NODE(n) + p] -= w[NODE(n + 1) + p];
  }
}

int orc_apply_J(void* vc, const double* in, double* out) { orc_t* c = vc; time_lower(c, &c->A, in, out); return 0; }
int orc_apply_JT(void* vc, const double* in, double* out) { orc_t* c = vc; time_upper(c, &c->A, in, out); return 0; }
int orc_apply_Jhat(void* vc, const double* in, double* out) { orc_t* c = vc; time_lower(c, &c->Ahat, in, out); return 0; }
int orc_apply_JhatT(void* vc, const double* in, double* out) { orc_t* c = vc; time_upper(c, &c->Ahat, in, out); return 0; }
int orc_apply_L(void* vc, const double* in, double* out) { /* :85-89 */
  orc_t* c = vc;
  for (size_t k = 0; k < c->B; ++k) out[k] = -c->dt * in[k];
  return 0;
}
int orc_apply_LT(void* vc, const double* in, double* out) { return orc_apply_L(vc, in, out); }
int orc_apply_Mu(void* vc, const double* in, double* out) { /* :95-99 */
  orc_t* c = vc;
  for (size_t k = 0; k < c->B; ++k) out[k] = c->ms * in[k];
  return 0;
}
int orc_apply_Mz(void* vc, const double* in, double* out) { return orc_apply_Mu(vc, in, out); }
int orc_apply_Mu_inv(void* vc, const double* in, double* out) { /* :101-105 */
  orc_t* c = vc;
  for (size_t k = 0; k < c->B; ++k) out[k] = in[k] / c->ms;
  return 0;
}

/* apply_shat (schur.cpp:71-78) */
int orc_apply_shat(void* vc, const double* v, double* out) {
  orc_t* c = vc;
  double* t = xcalloc(c->B, sizeof(double));
  time_upper(c, &c->Ahat, v, t);
  for (size_t k = 0; k < c->B; ++k) t[k] /= c->ms;
  time_lower(c, &c->Ahat, t, out);
  free(t);
  return 0;
}

/* apply_K (kkt.cpp:50-65) */
int orc_apply_K(void* vc, const double* v, double* out) {
  orc_t* c = vc;
  const size_t nb = c->B;
  const double omega = c->d.omega;
  const double *u = v, *z = v + nb, *w = v + 2 * nb;
  double *ou = out, *oz = out + nb, *ow = out + 2 * nb;
  time_upper(c, &c->A, w, ou);
  for (size_t k = 0; k < nb; ++k) ou[k] += c->ms * u[k];
  for (size_t k = 0; k < nb; ++k) oz[k] = omega * c->ms * z[k] - c->dt * w[k];
  time_lower(c, &c->A, u, ow);
  for (size_t k = 0; k < nb; ++k) ow[k] -= c->dt * z[k];
  return 0;
}

/* forward_solve_window / adjoint_solve_window (heat_operators.cpp:139-169) */
static void fwd_window(const orc_t* c, double* b, int len) {
  const int nsp = c->nsp;
  for (int k = 0; k < len; ++k) {
    double* xk = b + (size_t)k * nsp;
    if (k > 0)
      for (int p = 0; p < nsp; ++p) xk[p] += b[(size_t)(k - 1) * nsp + p];
    blu_solve(&c->F, xk);
  }
}
static void adj_window(const orc_t* c, double* b, int len) {
  const int nsp = c->nsp;
  for (int k = len - 1; k >= 0; --k) {
    double* xk = b + (size_t)k * nsp;
    if (k < len - 1)
      for (int p = 0; p < nsp; ++p) xk[p] += b[(size_t)(k + 1) * nsp + p];
    blu_solve_t(&c->F, xk);
  }
}
int orc_forward_solve_window(void* vc, double* b, int len) { fwd_window(vc, b, len); return 0; }
int orc_adjoint_solve_window(void* vc, double* b, int len) { adj_window(vc, b, len); return 0; }
int orc_band_solve(void* vc, double* b, int nrhs, int transpose) {
  orc_t* c = vc;
  for (int k = 0; k < nrhs; ++k) {
    if (transpose)
      blu_solve_t(&c->F, b + (size_t)k * c->nsp);
    else
      blu_solve(&c->F, b + (size_t)k * c->nsp);
  }
  return 0;
}
int orc_ahat_factor(void* vc, int* kl, int* ku, double* ab, int* piv, double* growth) {
  orc_t* c = vc;
  *kl = c->F.kl;
  *ku = c->F.ku;
  if (ab) memcpy(ab, c->F.ab, sizeof(double) * (size_t)c->F.n * (c->F.kl + c->F.ku + 1));
  if (piv) memcpy(piv, c->F.piv, sizeof(int) * (size_t)c->F.n);
  if (growth) *growth = c->F.growth;
  return 0;
}

/* apply_rasq (schur.cpp:103-130), W-node included as in the reference */
int orc_apply_rasq(void* vc, const double* r, double* out) {
  orc_t* c = vc;
  const int nsp = c->nsp;
  memset(out, 0, sizeof(double) * c->B);
  for (int s = 0; s < c->Nd; ++s) {
    const int ns = c->nlast[s] - c->nfirst[s] + 1;
    const int wlen = c->elast[s] - c->efirst[s] + 1;
    const int off = c->nfirst[s] - c->efirst[s];
    double* win = xcalloc((size_t)wlen * nsp, sizeof(double));
    memcpy(win + (size_t)off * nsp, r + NODE(c->nfirst[s]), sizeof(double) * (size_t)ns * nsp);
    fwd_window(c, win, wlen);
    for (size_t k = 0; k < (size_t)wlen * nsp; ++k) win[k] *= c->ms;
    adj_window(c, win, wlen);
    double* sub = win + (size_t)off * nsp;
    for (int k = 0; k < ns; ++k)
      if (c->owner[c->nfirst[s] + k] != s) memset(sub + (size_t)k * nsp, 0, sizeof(double) * nsp);
    const size_t base = NODE(c->nfirst[s]);
    for (size_t k = 0; k < (size_t)ns * nsp; ++k) out[base + k] += sub[k];
    free(win);
  }
  return 0;
}

/* ------------------------------------------------------- coarse space */
/* build_coarse_space (schur.cpp:266-413), scalar and per-dof */
typedef struct {
  int i, j;
  double v;
} trip_t;
static int trip_cmp(const void* a, const void* b) {
  const trip_t *x = a, *y = b;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return 0;
}

static int build_coarse(orc_t* c) {
  const int Nd = c->Nd, nsp = c->nsp, Nt = c->Nt;
  const int scalar = c->d.coarse_variant == KKT_COARSE_SCALAR;
  c->variant = c->d.coarse_variant;
  c->phi_c = xcalloc(Nd, sizeof(double*));
  c->phi_l = xcalloc(Nd, sizeof(double*));
  c->phi_len = xcalloc(Nd, sizeof(int));
  for (int s = 0; s < Nd; ++s) {
    const int ns = c->nlast[s] - c->nfirst[s] + 1;
    const int skip = c->ofirst[s] - c->nfirst[s];
    c->phi_len[s] = ns - skip;
    c->phi_c[s] = xcalloc(ns, sizeof(double));
    c->phi_l[s] = xcalloc(ns, sizeof(double));
    for (int k = 0; k < ns - skip; ++k) c->phi_c[s][k] = 1.0;
    for (int k = skip; k < ns; ++k) c->phi_l[s][k - skip] = ns > 1 ? -1.0 + 2.0 * k / (ns - 1) : 0.0;
  }
  const int ndof = scalar ? 1 : nsp;
  int* cstart = xcalloc(2 * (size_t)Nd, sizeof(int));
  int ncols = 0;
  c->col_s = xcalloc(2 * (size_t)Nd * ndof, sizeof(int));
  c->col_kind = xcalloc(2 * (size_t)Nd * ndof, sizeof(int));
  c->col_dof = xcalloc(2 * (size_t)Nd * ndof, sizeof(int));
  for (int s = 0; s < Nd; ++s)
    for (int kind = 0; kind < 2; ++kind) {
      cstart[2 * s + kind] = -1;
      const double* phi = kind == 0 ? c->phi_c[s] : c->phi_l[s];
      int allz = 1;
      for (int k = 0; k < c->phi_len[s]; ++k) allz &= phi[k] == 0.0;
      if (allz) continue;
      if (kind == 1 && c->olast[s] - c->ofirst[s] + 1 < 2) continue;
      cstart[2 * s + kind] = ncols;
      for (int dof = 0; dof < ndof; ++dof) {
        c->col_s[ncols] = s;
        c->col_kind[ncols] = kind;
        c->col_dof[ncols] = scalar ? -1 : dof;
        ++ncols;
      }
    }
  c->ncols = ncols;
  if (ncols == 0) {
    free(cstart);
    return fail(KKT_ECONFIG, -1, "coarse space is empty");
  }
  double* S0 = scalar ? xcalloc((size_t)ncols * ncols, sizeof(double)) : NULL;
  size_t ntrip = 0, captrip = 1024;
  trip_t* trips = scalar ? NULL : xcalloc(captrip, sizeof(trip_t));
  int wmax = 0;
  for (int s = 0; s < Nd; ++s) {
    int e0 = c->ofirst[s] - 1 > 1 ? c->ofirst[s] - 1 : 1;
    int e1 = c->olast[s] + 1 < Nt ? c->olast[s] + 1 : Nt;
    if (e1 - e0 + 1 > wmax) wmax = e1 - e0 + 1;
  }
  double* zwin = xcalloc((size_t)wmax * nsp, sizeof(double));
  double* twin = xcalloc((size_t)wmax * nsp, sizeof(double));
  double* ywin = xcalloc((size_t)wmax * nsp, sizeof(double));
  double* nsums = xcalloc(wmax, sizeof(double));
  for (int s = 0; s < Nd; ++s) {
    const int of = c->ofirst[s], oc = c->olast[s] - c->ofirst[s] + 1;
    const int e0 = of - 1 > 1 ? of - 1 : 1;
    const int e1 = c->olast[s] + 1 < Nt ? c->olast[s] + 1 : Nt;
    const int wlen = e1 - e0 + 1, off = of - e0;
    for (int kind = 0; kind < 2; ++kind) {
      if (cstart[2 * s + kind] < 0) continue;
      const double* phi = kind == 0 ? c->phi_c[s] : c->phi_l[s];
      for (int dof = 0; dof < ndof; ++dof) {
        const int ci = cstart[2 * s + kind] + (scalar ? 0 : dof);
        memset(zwin, 0, sizeof(double) * (size_t)wlen * nsp);
        for (int k = 0; k < oc; ++k) {
          double* node = zwin + (size_t)(off + k) * nsp;
          if (scalar)
            for (int p = 0; p < nsp; ++p) node[p] = phi[k];
          else
            node[dof] = phi[k];
        }
        for (int k = 0; k < wlen; ++k) {
          double* tk = twin + (size_t)k * nsp;
          band_matvec_t(&c->Ahat, zwin + (size_t)k * nsp, tk);
          if (k + 1 < wlen)
            for (int p = 0; p < nsp; ++p) tk[p] -= zwin[(size_t)(k + 1) * nsp + p];
        }
        for (size_t k = 0; k < (size_t)wlen * nsp; ++k) twin[k] /= c->ms;
        for (int k = 0; k < wlen; ++k) {
          double* yk = ywin + (size_t)k * nsp;
          band_matvec(&c->Ahat, twin + (size_t)k * nsp, yk);
          if (k > 0)
            for (int p = 0; p < nsp; ++p) yk[p] -= twin[(size_t)(k - 1) * nsp + p];
        }
        if (scalar)
          for (int k = 0; k < wlen; ++k) {
            double acc = 0.0;
            for (int p = 0; p < nsp; ++p) acc += ywin[(size_t)k * nsp + p];
            nsums[k] = acc;
          }
        for (int s2 = s - 1 > 0 ? s - 1 : 0; s2 <= (s + 1 < Nd - 1 ? s + 1 : Nd - 1); ++s2) {
          const int of2 = c->ofirst[s2], oc2 = c->olast[s2] - c->ofirst[s2] + 1;
          for (int kind2 = 0; kind2 < 2; ++kind2) {
            if (cstart[2 * s2 + kind2] < 0) continue;
            const double* phi2 = kind2 == 0 ? c->phi_c[s2] : c->phi_l[s2];
            for (int dof2 = 0; dof2 < ndof; ++dof2) {
              const int ri = cstart[2 * s2 + kind2] + (scalar ? 0 : dof2);
              double acc = 0.0;
              for (int k2 = 0; k2 < oc2; ++k2) {
                const int n2 = of2 + k2;
                if (n2 < e0 || n2 > e1) continue;
                const int pos = n2 - e0;
                if (scalar)
                  acc += phi2[k2] * nsums[pos];
                else
                  acc += phi2[k2] * ywin[(size_t)pos * nsp + dof2];
              }
              if (scalar) {
                S0[(size_t)ri * ncols + ci] = acc;
              } else if (acc != 0.0) {
                if (ntrip == captrip) {
                  captrip *= 2;
                  trips = realloc(trips, captrip * sizeof(trip_t));
                }
                trips[ntrip++] = (trip_t){ri, ci, acc};
              }
            }
          }
        }
      }
    }
  }
  free(zwin); free(twin); free(ywin); free(nsums); free(cstart);
  int st;
  if (scalar) {
    c->S0 = S0;
    st = dlu_factor(&c->S0d, S0, ncols);
  } else {
    /* sparse_from_triplets (linalg.cpp:267-296) + SparseLU::to_banded (:312-331) */
    qsort(trips, ntrip, sizeof(trip_t), trip_cmp);
    size_t w = 0;
    for (size_t k = 0; k < ntrip;) {
      trip_t t = trips[k];
      double sum = t.v;
      size_t k2 = k + 1;
      while (k2 < ntrip && trips[k2].i == t.i && trips[k2].j == t.j) sum += trips[k2++].v;
      trips[w++] = (trip_t){t.i, t.j, sum};
      k = k2;
    }
    ntrip = w;
    int kl = 0, ku = 0;
    for (size_t k = 0; k < ntrip; ++k) {
      if (trips[k].i - trips[k].j > kl) kl = trips[k].i - trips[k].j;
      if (trips[k].j - trips[k].i > ku) ku = trips[k].j - trips[k].i;
    }
    band_t Bm;
    band_zero(&Bm, ncols, kl, ku);
    for (size_t k = 0; k < ntrip; ++k) *band_ref(&Bm, trips[k].i, trips[k].j) = trips[k].v;
    c->S0 = xcalloc((size_t)ncols * ncols < (size_t)4096 * 4096 ? (size_t)ncols * ncols : 1, sizeof(double));
    if ((size_t)ncols <= 4096)
      for (size_t k = 0; k < ntrip; ++k) c->S0[(size_t)trips[k].i * ncols + trips[k].j] = trips[k].v;
    c->sparse = 1;
    st = blu_factor(&c->S0s, &Bm);
    free(Bm.data);
    free(trips);
  }
  if (st)
    return fail(KKT_ECONFIG, g_err_index, "coarse operator (%s variant) is rank deficient: %s",
                scalar ? "scalar" : "per-dof", g_err);
  c->has_coarse = 1;
  return 0;
}

int orc_coarse_dim(void* vc) { orc_t* c = vc; return c->has_coarse ? c->ncols : -1; }

/* restrict_to_coarse (schur.cpp:181-204) */
int orc_coarse_restrict(void* vc, const double* r, double* cv) {
  orc_t* c = vc;
  const int nsp = c->nsp;
  for (int ci = 0; ci < c->ncols; ++ci) {
    const int s = c->col_s[ci];
    const double* phi = c->col_kind[ci] == 0 ? c->phi_c[s] : c->phi_l[s];
    const int of = c->ofirst[s], oc = c->olast[s] - of + 1;
    double acc = 0.0;
    for (int k = 0; k < oc; ++k) {
      const size_t base = NODE(of + k);
      if (c->col_dof[ci] < 0) {
        double ns = 0.0;
        for (int p = 0; p < nsp; ++p) ns += r[base + p];
        acc += phi[k] * ns;
      } else {
        acc += phi[k] * r[base + c->col_dof[ci]];
      }
    }
    cv[ci] = acc;
  }
  return 0;
}

/* prolong_add (schur.cpp:206-226) */
int orc_coarse_prolong_add(void* vc, const double* cv, double* out) {
  orc_t* c = vc;
  const int nsp = c->nsp;
  for (int ci = 0; ci < c->ncols; ++ci) {
    const int s = c->col_s[ci];
    const double* phi = c->col_kind[ci] == 0 ? c->phi_c[s] : c->phi_l[s];
    const int of = c->ofirst[s], oc = c->olast[s] - of + 1;
    for (int k = 0; k < oc; ++k) {
      const size_t base = NODE(of + k);
      const double v = phi[k] * cv[ci];
      if (c->col_dof[ci] < 0)
        for (int p = 0; p < nsp; ++p) out[base + p] += v;
      else
        out[base + c->col_dof[ci]] += v;
    }
  }
  return 0;
}

int orc_coarse_solve(void* vc, double* cv) { /* solve_in_place (schur.cpp:228-234) */
  orc_t* c = vc;
  if (c->sparse)
    blu_solve(&c->S0s, cv);
  else
    dlu_solve(&c->S0d, cv);
  return 0;
}

int orc_coarse_matrix(void* vc, double* out) {
  orc_t* c = vc;
  if (c->ncols > 4096) return fail(KKT_ECONFIG, -1, "coarse_matrix_dense: beyond the dense limit");
  memcpy(out, c->S0, sizeof(double) * (size_t)c->ncols * c->ncols);
  return 0;
}

/* apply_two_level (schur.cpp:415-444) */
int orc_apply_two_level(void* vc, const double* r, double* out, int form) {
  orc_t* c = vc;
  if (!c->has_coarse) return fail(KKT_ECONFIG, -1, "two-level apply without a coarse space");
  double* cv = xcalloc(c->ncols, sizeof(double));
  orc_coarse_restrict(c, r, cv);
  orc_coarse_solve(c, cv);
  double* yc = xcalloc(c->B, sizeof(double));
  orc_coarse_prolong_add(c, cv, yc);
  if (form == KKT_FORM_LITERAL) {
    orc_apply_rasq(c, yc, out);
  } else if (form == KKT_FORM_ADDITIVE) {
    orc_apply_rasq(c, r, out);
    for (size_t k = 0; k < c->B; ++k) out[k] += yc[k];
  } else {
    double* res = xcalloc(c->B, sizeof(double));
    orc_apply_shat(c, yc, res);
    for (size_t k = 0; k < c->B; ++k) res[k] = r[k] - res[k];
    orc_apply_rasq(c, res, out);
    for (size_t k = 0; k < c->B; ++k) out[k] += yc[k];
    free(res);
  }
  free(cv);
  free(yc);
  return 0;
}

/* SchurSolver::apply (schur.cpp:494-533) */
int orc_schur_apply(void* vc, const double* r, double* out) {
  orc_t* c = vc;
  switch (c->d.precond) {
    case KKT_PRECOND_NONE: memcpy(out, r, sizeof(double) * c->B); return 0;
    case KKT_PRECOND_ONE_LEVEL: return orc_apply_rasq(c, r, out);
    case KKT_PRECOND_TWO_LEVEL: return orc_apply_two_level(c, r, out, c->d.two_level_form);
  }
  return fail(KKT_EUNSUPPORTED, -1, "unsupported preconditioner kind");
}

/* apply_P_inv (kkt.cpp:71-81) */
int orc_apply_P_inv(void* vc, const double* r, double* out) {
  orc_t* c = vc;
  const size_t nb = c->B;
  for (size_t k = 0; k < nb; ++k) out[k] = r[k] / c->ms;
  for (size_t k = 0; k < nb; ++k) out[nb + k] = r[nb + k] / (c->d.omega * c->ms);
  return orc_schur_apply(c, r + 2 * nb, out + 2 * nb);
}

int orc_kkt_residual(void* vc, const double* v, const double* rhs, double* out) { /* kkt.cpp:110-124 */
  orc_t* c = vc;
  const size_t n = 3 * c->B;
  double* kv = xcalloc(n, sizeof(double));
  orc_apply_K(c, v, kv);
  double rn = 0.0, bn = 0.0;
  for (size_t k = 0; k < n; ++k) {
    const double d = rhs[k] - kv[k];
    rn += d * d;
    bn += rhs[k] * rhs[k];
  }
  free(kv);
  const double r = sqrt(rn);
  *out = bn > 0.0 ? r / sqrt(bn) : r;
  return 0;
}

/* ---------------------------------------------------------------- GMRES */
typedef int (*map_fn)(void* ctx, const double* in, double* out);

/* gmres_solve (gmres.cpp:21-155) */
static int gmres(map_fn op, void* opc, map_fn prec, void* pc, const double* b, size_t n,
                 double tol, int max_iters, int restart, double happy_tol, double* xout,
                 kkt_gmres_result* res, double* hist, int cap) {
  if (!(tol > 0) || max_iters < 1) return fail(KKT_EINVAL, -1, "gmres: tol must be > 0 and max_iters >= 1");
  memset(xout, 0, sizeof(double) * n);
  res->converged = 0;
  res->iterations = 0;
  res->true_final_relres = 0.0;
  res->history_len = 0;
  const double bnorm = norm2(b, n);
  if (bnorm == 0.0) {
    res->converged = 1;
    return 0;
  }
  double* x = xout;
  double* scratch = xcalloc(n, sizeof(double));
  double* r = xcalloc(n, sizeof(double));
  double* w = xcalloc(n, sizeof(double));
  double* z = xcalloc(n, sizeof(double));
  int total = 0, converged = 0, first = 1, nh = 0;
  double* histall = xcalloc((size_t)max_iters + 1, sizeof(double));
  int st = 0;
  while (total < max_iters && !converged) {
    if (first) {
      memcpy(r, b, sizeof(double) * n);
      first = 0;
    } else {
      op(opc, x, scratch);
      for (size_t k = 0; k < n; ++k) r[k] = b[k] - scratch[k];
    }
    const double beta = norm2(r, n);
    if (beta / bnorm <= tol) {
      converged = 1;
      break;
    }
    const int cycle = restart > 0 ? (restart < max_iters - total ? restart : max_iters - total)
                                  : max_iters - total;
    double** V = xcalloc((size_t)cycle + 1, sizeof(double*));
    V[0] = xcalloc(n, sizeof(double));
    for (size_t k = 0; k < n; ++k) V[0][k] = r[k] / beta;
    double** H = xcalloc((size_t)cycle, sizeof(double*));
    double* g = xcalloc((size_t)cycle + 1, sizeof(double));
    double* cs = xcalloc((size_t)cycle, sizeof(double));
    double* sn = xcalloc((size_t)cycle, sizeof(double));
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < cycle; ++j) {
      if (prec) {
        prec(pc, V[j], z);
        op(opc, z, w);
      } else {
        op(opc, V[j], w);
      }
      for (size_t e = 0; e < n; ++e)
        if (!isfinite(w[e])) {
          st = fail(KKT_EDIVERGED, total + 1, "gmres: non-finite values in Krylov vector at iteration %d", total + 1);
          break;
        }
      if (st) break;
      H[j] = xcalloc((size_t)j + 2, sizeof(double));
      double* h = H[j];
      for (int i = 0; i <= j; ++i) {
        h[i] = dot(w, V[i], n);
        axpy(-h[i], V[i], w, n);
      }
      h[j + 1] = norm2(w, n);
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t;
      }
      const double denom = hypot(h[j], h[j + 1]);
      cs[j] = h[j] / denom;
      sn[j] = h[j + 1] / denom;
      h[j] = denom;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      ++k;
      const double relest = fabs(g[j + 1]) / bnorm;
      histall[nh++] = relest;
      const int happy = h[j + 1] <= happy_tol;
      if (relest <= tol || happy) {
        converged = 1;
        break;
      }
      if (j + 1 < cycle) {
        V[j + 1] = xcalloc(n, sizeof(double));
        for (size_t e = 0; e < n; ++e) V[j + 1][e] = w[e] / h[j + 1];
      }
    }
    if (!st) {
      double* y = xcalloc((size_t)k + 1, sizeof(double));
      for (int i = k - 1; i >= 0; --i) {
        double acc = g[i];
        for (int j2 = i + 1; j2 < k; ++j2) acc -= H[j2][i] * y[j2];
        y[i] = acc / H[i][i];
      }
      memset(scratch, 0, sizeof(double) * n);
      for (int i = 0; i < k; ++i) axpy(y[i], V[i], scratch, n);
      if (prec) {
        prec(pc, scratch, z);
        axpy(1.0, z, x, n);
      } else {
        axpy(1.0, scratch, x, n);
      }
      free(y);
    }
    for (int i = 0; i <= cycle; ++i) free(V[i]);
    for (int i = 0; i < cycle; ++i) free(H[i]);
    free(V); free(H); free(g); free(cs); free(sn);
    if (st) break;
  }
  if (!st) {
    res->converged = converged;
    res->iterations = nh;
    op(opc, x, scratch);
    double rn2 = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double d = b[i] - scratch[i];
      rn2 += d * d;
    }
    res->true_final_relres = sqrt(rn2) / bnorm;
    const int m = cap < nh ? cap : nh;
    res->history_len = hist ? m : 0;
    if (hist) memcpy(hist, histall, sizeof(double) * m);
  }
  free(histall); free(scratch); free(r); free(w); free(z);
  return st;
}

int orc_gmres_solve(void* vc, const double* b, double* x, kkt_gmres_result* res, double* hist, int cap) {
  orc_t* c = vc;
  const kkt_problem_desc* d = &c->d;
  return gmres((map_fn)orc_apply_K, c, d->precond != KKT_PRECOND_NONE ? (map_fn)orc_apply_P_inv : NULL, c, b,
               3 * c->B, d->tol, d->max_iters, d->restart, d->happy_breakdown_tol, x, res, hist, cap);
}

typedef struct {
  int n;
  const double* M;
} dense_map;
static int dense_apply(void* vc, const double* v, double* o) {
  const dense_map* m = vc;
  for (int i = 0; i < m->n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < m->n; ++j) acc += m->M[(size_t)i * m->n + j] * v[j];
    o[i] = acc;
  }
  return 0;
}

int orc_gmres_dense(int n, const double* A, const double* M, const double* b, double tol, int max_iters,
                    int restart, double* x, kkt_gmres_result* res, double* hist, int cap) {
  dense_map a = {n, A}, m = {n, M};
  return gmres(dense_apply, &a, M ? dense_apply : NULL, &m, b, (size_t)n, tol, max_iters, restart, 1e-14, x,
               res, hist, cap);
}
