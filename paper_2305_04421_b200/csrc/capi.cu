// capi.cu — the extern "C" boundary (include/kktdd_b200.h) and context setup.
//
// kkt_ctx_create does what the reference's run_single does before the solve
// (experiments.cpp:39-45): ProblemConfig::validate (config.cpp:5-22),
// HeatOperators (heat_operators.cpp:46-55: derived constants with the
// reference's expressions, Ahat factorisation), build_time_partition
// (time_partition.cpp:61-86) and make_schur_solver (schur.cpp:543-558).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "sweep.cuh"

namespace kkt {

Ctx::~Ctx() {
  if (stream) cudaStreamSynchronize(stream);
  v4_unregister(this);
  delete comm;
  for (auto& g : graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  basis.clear();
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (auto& iv : ev_pending) { cudaEventDestroy(iv.a); cudaEventDestroy(iv.b); }
  for (auto e : ev_open) if (e) cudaEventDestroy(e);
  for (auto e : e2e_ev) if (e) cudaEventDestroy(e);
  for (auto e : e2e_chunk_ev) cudaEventDestroy(e);
  for (auto st : {e2e_in, e2e_out, e2e_aux, e2e_trail}) if (st) cudaStreamDestroy(st);
  if (e2e_step_ev) cudaEventDestroy(e2e_step_ev);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

static cudaEvent_t pool_get(Ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  KKT_CUDA(cudaEventCreate(&e));
  return e;
}

void Ctx::tbegin(int slot) {
  if (!phase_timing) return;
  if (!ev_open[slot]) ev_open[slot] = pool_get(this);
  KKT_CUDA(cudaEventRecord(ev_open[slot], stream));
}

void Ctx::tend(int slot) {
  if (!phase_timing || !ev_open[slot]) return;
  cudaEvent_t b = pool_get(this);
  KKT_CUDA(cudaEventRecord(b, stream));
  ev_pending.push_back({slot, ev_open[slot], b});
  ev_open[slot] = nullptr;
}

void Ctx::tcollect() {
  for (auto& iv : ev_pending) {
    float ms = 0.f;
    KKT_CUDA(cudaEventSynchronize(iv.b));
    KKT_CUDA(cudaEventElapsedTime(&ms, iv.a, iv.b));
    phase_ms[iv.slot] += ms;
    phase_cnt[iv.slot] += 1;
    ev_pool.push_back(iv.a);
    ev_pool.push_back(iv.b);
  }
  ev_pending.clear();
}

namespace {

thread_local std::string g_create_err;
thread_local int g_create_err_index = -1;

void validate(const kkt_problem_desc& d) {
  auto fail = [](const std::string& m) { throw Error(KKT_ECONFIG, m); };
  if (d.Nx < 2 || d.Ny < 2)
    fail("mesh needs Nx, Ny >= 2, got Nx=" + std::to_string(d.Nx) + " Ny=" + std::to_string(d.Ny));
  if (d.Lx <= 0 || d.Ly <= 0 || d.T <= 0) fail("domain extents and T must be positive");
  if (d.Nt < 1) fail("Nt must be >= 1, got " + std::to_string(d.Nt));
  if (d.Nd < 1) fail("Nd must be >= 1, got " + std::to_string(d.Nd));
  if (d.Nt % d.Nd != 0)
    fail("Nt=" + std::to_string(d.Nt) + " is not divisible by Nd=" + std::to_string(d.Nd));
  if (d.nu < 0) fail("conductivity nu must be >= 0");
  if (!(d.omega > 0)) fail("regularization omega must be > 0");
  if (!(d.tol > 0)) fail("gmres tol must be > 0");
  if (d.max_iters < 1) fail("gmres max_iters must be >= 1");
  if (d.restart != KKT_NO_RESTART && d.restart < 1) fail("gmres restart must be >= 1");
  if (d.precond < KKT_PRECOND_NONE || d.precond > KKT_PRECOND_TRUE_SCHUR) fail("unknown preconditioner kind");
  if (d.two_level_form < KKT_FORM_LITERAL || d.two_level_form > KKT_FORM_ADDITIVE) fail("unknown two-level form");
  if (d.coarse_variant != KKT_COARSE_SCALAR && d.coarse_variant != KKT_COARSE_PER_DOF) fail("unknown coarse variant");
  if (d.jhat_sign != KKT_SIGN_PLUS && d.jhat_sign != KKT_SIGN_MINUS) fail("unknown jhat sign");
}

void setup(Ctx* c, const kkt_problem_desc& d, const kkt_runtime_opts* o) {
  validate(d);
  c->desc = d;
  c->mode = o ? o->mode : KKT_MODE_FAST;
  if (c->mode == KKT_MODE_SPECTRAL) {  // FAST arithmetic + eigenbasis spatial solves
    c->mode = KKT_MODE_FAST;
    c->spectral = true;
  }
  if (c->mode != KKT_MODE_FAST && c->mode != KKT_MODE_STRICT) throw Error(KKT_EINVAL, "unknown mode");
  if (const char* e = std::getenv("KKT_BISECT")) c->bisect = c->mode == KKT_MODE_FAST ? std::atoi(e) : 0;
  c->rank = o ? o->rank : 0;
  c->nranks = o ? o->nranks : 1;
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks)
    throw Error(KKT_EINVAL, "bad rank / nranks");
  if (c->nranks > 1) {
    if (c->mode == KKT_MODE_STRICT)
      throw Error(KKT_EUNSUPPORTED,
                  "strict (bitwise) mode is single-rank: the reference's left-to-right sums cross slabs");
    if (d.Nd % c->nranks != 0)
      throw Error(KKT_ECONFIG, "time-slab sharding needs nranks to divide Nd (Nd=" +
                                   std::to_string(d.Nd) + ", nranks=" + std::to_string(c->nranks) + ")");
  }
  int dev = (o && o->device >= 0) ? o->device : -1;
  if (dev < 0) KKT_CUDA(cudaGetDevice(&dev));
  KKT_CUDA(cudaSetDevice(dev));
  c->device = dev;
  if (o && o->stream) {
    c->stream = static_cast<cudaStream_t>(o->stream);
  } else {
    KKT_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  if (c->nranks > 1) {
    if (o->local_group)
      c->comm = make_local_comm(o->local_group, c->rank);
    else if (o->nccl_unique_id)
      c->comm = make_nccl_comm(o->nccl_unique_id, c->rank, c->nranks);
    else
      throw Error(KKT_EINVAL, "nranks > 1 needs an NCCL unique id or a local group");
  }
  if (d.precond == KKT_PRECOND_DENSE_SCHUR || d.precond == KKT_PRECOND_TRUE_SCHUR)
    throw Error(KKT_EUNSUPPORTED,
                "dense-schur / true-schur are desk-scale dense oracles (schur.cpp:13-21), not on the device path");

  // ---- derived constants, reference expressions (config.hpp:52-65, heat_operators.cpp:16-37)
  c->nx = d.Nx - 1;
  c->ny = d.Ny - 1;
  c->nsp = c->nx * c->ny;
  c->Nt = d.Nt;
  c->Nd = d.Nd;
  c->m = d.Nt / d.Nd;
  c->Bg = int64_t(c->Nt) * c->nsp;
  // time slab of this rank: whole subdomains [s0, s0+ndl), nodes [n0, n0+ntl)
  c->ndl = c->Nd / c->nranks;
  c->s0 = c->rank * c->ndl;
  c->ntl = c->ndl * c->m;
  c->n0 = c->s0 * c->m + 1;
  c->B = int64_t(c->ntl) * c->nsp;
  c->halo.alloc(size_t(4) * c->nsp);
  c->dx = d.Lx / d.Nx;
  c->dy = d.Ly / d.Ny;
  c->dt = d.T / d.Nt;
  c->ms = c->dt * c->dx * c->dy;
  {
    const double s = (d.jhat_sign == KKT_SIGN_PLUS) ? 1.0 : -1.0;
    c->sigma = s / std::sqrt(d.omega);
  }
  c->omega = d.omega;
  c->oms = d.omega * c->ms;
  c->cx = c->dt * d.nu / (c->dx * c->dx);
  c->cy = c->dt * d.nu / (c->dy * c->dy);
  const double diag = 1.0 + 2.0 * c->cx + 2.0 * c->cy;
  c->A = Stencil{c->nx, c->ny, diag, -c->cx, -c->cy};
  c->Ahat = Stencil{c->nx, c->ny, diag - c->sigma * c->dt, -c->cx, -c->cy};

  // ---- time partition
  c->nodes.clear();
  c->owned.clear();
  c->owner.assign(c->Nt + 1, 0);
  for (int n = 1; n <= c->Nt; ++n) c->owner[n] = (n - 1) / c->m;
  for (int s = 0; s < c->Nd; ++s) {
    const int last = (s + 1) * c->m;
    const int first = s == 0 ? 1 : s * c->m;
    c->nodes.push_back({first, last});
    c->owned.push_back({s == 0 ? 1 : s * c->m + 1, last});
  }

  // ---- factor + preconditioner setup: the reference's banded LU (bitwise) for
  // STRICT mode and small grids; the block recursion for FAST mode on large
  // grids (nx > 128), where the band's rank-1 updates do not scale
  static const bool force_rec = getenv("KKT_FORCE_BLOCK_RECURSION") != nullptr;  // testing
  if (c->mode == KKT_MODE_FAST && (c->nx > 128 || force_rec)) {
    // The block recursion is an UNPIVOTED LU.  BandedLU (linalg.cpp:69-125) pivots, and the two
    // agree only where no row interchange happens: a (weakly) diagonally dominant Ahat, which
    // the minus sign always gives.  With jhat_sign = plus the diagonal 1 + 2cx + 2cy - dt/sqrt(omega)
    // can lose dominance; there is no scalable pivoting factor for these grids, so refuse
    // instead of silently using a different (possibly unstable) factorisation.
    if (!(std::abs(c->Ahat.diag) >= 2.0 * std::abs(c->cx) + 2.0 * std::abs(c->cy)))
      throw Error(KKT_EUNSUPPORTED,
                  "FAST mode on grids with nx > 128 needs a diagonally dominant Ahat (unpivoted block LU); "
                  "Ahat diagonal " + std::to_string(c->Ahat.diag) + " vs off-diagonal sum " +
                      std::to_string(2.0 * std::abs(c->cx) + 2.0 * std::abs(c->cy)) +
                      " (jhat_sign = plus with dt > sqrt(omega)): use STRICT mode");
    build_block_recursion(c);
    if (v6_supported(c))
      build_v6(c);
    else if (v5_supported(c))
      build_v5(c);
  } else {
    build_factor(c);
    if (c->mode == KKT_MODE_FAST) build_block_inverses(c);
  }
  // SPECTRAL mode only: RASQ in Ahat's eigenbasis (spectral.cu).  FAST keeps
  // the reference's LU method (sweep_group.cu / sweep_tma.cu / sweep_fast.cu).
  if (c->spectral) build_spectral(c);
  if (d.precond == KKT_PRECOND_TWO_LEVEL) build_coarse(c);
  KKT_CUDA(cudaStreamSynchronize(c->stream));
}

template <class F>
int guard(kkt_ctx* ctx, F&& f) {
  if (!ctx) return KKT_EINVAL;
  Ctx* c = &ctx->impl;
  try {
    KKT_CUDA(cudaSetDevice(c->device));
    f(c);
    c->err.clear();
    c->err_index = -1;
    return KKT_OK;
  } catch (const Error& e) {
    c->err = e.what();
    c->err_index = e.index;
    return e.status;
  } catch (const std::exception& e) {
    c->err = e.what();
    return KKT_EINVAL;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw Error(KKT_EINVAL, what);
}

}  // namespace
}  // namespace kkt

using kkt::Ctx;
using kkt::Error;

extern "C" {

void kkt_problem_desc_default(kkt_problem_desc* d) {
  if (!d) return;
  std::memset(d, 0, sizeof(*d));
  d->Lx = 1.0;
  d->Ly = 2.0;
  d->T = 1.0;
  d->Nx = 16;
  d->Ny = 16;
  d->Nt = 100;
  d->nu = 1.0;
  d->omega = 1e-3;
  d->Nd = 5;
  d->precond = KKT_PRECOND_TWO_LEVEL;
  d->coarse_variant = KKT_COARSE_PER_DOF;
  d->two_level_form = KKT_FORM_MULTIPLICATIVE;
  d->jhat_sign = KKT_SIGN_MINUS;
  d->tol = 1e-6;
  d->max_iters = 420;
  d->restart = KKT_NO_RESTART;
  d->happy_breakdown_tol = 1e-14;
}

const char* kkt_status_string(int s) {
  switch (s) {
    case KKT_OK: return "ok";
    case KKT_EINVAL: return "invalid argument";
    case KKT_ECONFIG: return "configuration error";
    case KKT_ESINGULAR: return "singular matrix";
    case KKT_EDIVERGED: return "gmres diverged";
    case KKT_ECUDA: return "cuda error";
    case KKT_ENCCL: return "nccl error";
    case KKT_EUNSUPPORTED: return "unsupported";
  }
  return "unknown";
}

const char* kkt_create_error(void) { return kkt::g_create_err.c_str(); }
int kkt_create_error_index(void) { return kkt::g_create_err_index; }

int kkt_ctx_create(const kkt_problem_desc* desc, const kkt_runtime_opts* opts, kkt_ctx** out) {
  if (!desc || !out) return KKT_EINVAL;
  *out = nullptr;
  kkt_ctx* h = new kkt_ctx();
  try {
    kkt::setup(&h->impl, *desc, opts);
  } catch (const Error& e) {
    kkt::g_create_err = e.what();
    kkt::g_create_err_index = e.index;
    const int st = e.status;
    delete h;
    return st;
  } catch (const std::exception& e) {
    kkt::g_create_err = e.what();
    kkt::g_create_err_index = -1;
    delete h;
    return KKT_EINVAL;
  }
  kkt::g_create_err.clear();
  kkt::g_create_err_index = -1;
  *out = h;
  return KKT_OK;
}

int kkt_ctx_destroy(kkt_ctx* ctx) {
  delete ctx;
  return KKT_OK;
}

const char* kkt_last_error(const kkt_ctx* ctx) { return ctx ? ctx->impl.err.c_str() : ""; }
int kkt_last_error_index(const kkt_ctx* ctx) { return ctx ? ctx->impl.err_index : -1; }

int kkt_layout(const kkt_ctx* ctx, int64_t* block, int32_t* n_sp, int32_t* node_first,
               int32_t* node_last, int64_t* local_block) {
  if (!ctx) return KKT_EINVAL;
  const Ctx& c = ctx->impl;
  if (n_sp) *n_sp = c.nsp;
  if (block) *block = c.Bg;
  if (node_first) *node_first = c.n0;
  if (node_last) *node_last = c.n0 + c.ntl - 1;
  if (local_block) *local_block = c.B;
  return KKT_OK;
}

int kkt_stream(const kkt_ctx* ctx, void** stream) {
  if (!ctx || !stream) return KKT_EINVAL;
  *stream = ctx->impl.stream;
  return KKT_OK;
}

int kkt_synchronize(kkt_ctx* ctx) {
  return kkt::guard(ctx, [](Ctx* c) { KKT_CUDA(cudaStreamSynchronize(c->stream)); });
}

int kkt_device_alloc(kkt_ctx* ctx, size_t count, double** out) {
  return kkt::guard(ctx, [&](Ctx*) {
    kkt::need(out != nullptr, "kkt_device_alloc: null out");
    *out = nullptr;
    if (count) KKT_CUDA(cudaMalloc(out, count * sizeof(double)));
  });
}

int kkt_device_free(kkt_ctx* ctx, double* p) {
  return kkt::guard(ctx, [&](Ctx* c) {
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    if (p) KKT_CUDA(cudaFree(p));
  });
}

int kkt_copy_to_device(kkt_ctx* ctx, double* dst, const double* src_host, size_t count) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(count == 0 || (dst && src_host), "kkt_copy_to_device: null pointer");
    KKT_CUDA(cudaMemcpyAsync(dst, src_host, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int kkt_copy_to_host(kkt_ctx* ctx, double* dst_host, const double* src, size_t count) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(count == 0 || (dst_host && src), "kkt_copy_to_host: null pointer");
    KKT_CUDA(cudaMemcpyAsync(dst_host, src, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

#define KKT_OP(name, body)                                                   \
  int name(kkt_ctx* ctx, const double* in, double* out) {                    \
    return kkt::guard(ctx, [&](Ctx* c) {                                     \
      kkt::need(in && out, #name ": null vector");                           \
      kkt::need(in != out, #name ": in and out must not alias");             \
      body;                                                                  \
    });                                                                      \
  }
KKT_OP(kkt_apply_J, kkt::op_time_stencil(c, kkt::OpKind::J, in, out))
KKT_OP(kkt_apply_JT, kkt::op_time_stencil(c, kkt::OpKind::JT, in, out))
KKT_OP(kkt_apply_Jhat, kkt::op_time_stencil(c, kkt::OpKind::Jhat, in, out))
KKT_OP(kkt_apply_JhatT, kkt::op_time_stencil(c, kkt::OpKind::JhatT, in, out))
KKT_OP(kkt_apply_L, kkt::op_scale(c, in, out, -c->dt, false))
KKT_OP(kkt_apply_LT, kkt::op_scale(c, in, out, -c->dt, false))
KKT_OP(kkt_apply_Mu, kkt::op_scale(c, in, out, c->ms, false))
KKT_OP(kkt_apply_Mu_inv, kkt::op_scale(c, in, out, c->ms, true))
KKT_OP(kkt_apply_Mz, kkt::op_scale(c, in, out, c->ms, false))
KKT_OP(kkt_apply_K, kkt::op_apply_K(c, in, out, nullptr))
KKT_OP(kkt_apply_P_inv, kkt::pinv_apply(c, in, out))
KKT_OP(kkt_apply_rasq, kkt::rasq_apply(c, in, out, false))
KKT_OP(kkt_schur_apply, kkt::schur_apply(c, in, out))
KKT_OP(kkt_apply_shat, {
  if (c->tmpB1.n < size_t(c->B)) c->tmpB1.alloc(c->B);
  kkt::op_shat(c, in, out, c->tmpB1.p);
})
#undef KKT_OP

int kkt_apply_two_level(kkt_ctx* ctx, const double* r, double* out, int32_t form) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(r && out && r != out, "kkt_apply_two_level: bad vectors");
    kkt::two_level_apply(c, r, out, form);
  });
}

int kkt_forward_solve_window(kkt_ctx* ctx, double* b, int32_t len) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(len >= 0 && (len == 0 || b), "forward_solve_window: bad window");
    kkt::window_solve(c, b, len, false);
  });
}

int kkt_adjoint_solve_window(kkt_ctx* ctx, double* b, int32_t len) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(len >= 0 && (len == 0 || b), "adjoint_solve_window: bad window");
    kkt::window_solve(c, b, len, true);
  });
}

int kkt_band_solve(kkt_ctx* ctx, double* b, int32_t nrhs) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(nrhs >= 0 && (nrhs == 0 || b), "band_solve: bad rhs");
    if (nrhs) kkt::band_solve(c, b, nrhs, false);
  });
}

int kkt_band_solve_transpose(kkt_ctx* ctx, double* b, int32_t nrhs) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(nrhs >= 0 && (nrhs == 0 || b), "band_solve_transpose: bad rhs");
    if (nrhs) kkt::band_solve(c, b, nrhs, true);
  });
}

int kkt_residual(kkt_ctx* ctx, const double* v, const double* rhs, double* relres) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(v && rhs && relres, "kkt_residual: null argument");
    *relres = kkt::kkt_relres(c, v, rhs);
  });
}

int kkt_coarse_dim(const kkt_ctx* ctx, int32_t* dim) {
  if (!ctx || !dim) return KKT_EINVAL;
  *dim = ctx->impl.has_coarse ? ctx->impl.cdim : -1;
  return ctx->impl.has_coarse ? KKT_OK : KKT_ECONFIG;
}

int kkt_coarse_restrict(kkt_ctx* ctx, const double* r, double* cvec) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(c->has_coarse, "no coarse space");
    kkt::coarse_restrict(c, r, cvec);
  });
}

int kkt_coarse_solve(kkt_ctx* ctx, double* cvec) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(c->has_coarse, "no coarse space");
    kkt::coarse_solve(c, cvec);
  });
}

int kkt_coarse_prolong_add(kkt_ctx* ctx, const double* cvec, double* out) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(c->has_coarse, "no coarse space");
    kkt::coarse_prolong_add(c, cvec, out);
  });
}

int kkt_coarse_matrix(kkt_ctx* ctx, double* host_out) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(c->has_coarse && host_out, "no coarse space");
    if (c->h_S0.empty() || (c->cdim > 4096 && !std::getenv("KKT_KEEP_S0")))
      throw kkt::Error(KKT_ECONFIG, "coarse_matrix_dense: dimension " + std::to_string(c->cdim) +
                                        " exceeds the dense limit 4096");
    std::memcpy(host_out, c->h_S0.data(), sizeof(double) * c->h_S0.size());
  });
}

int kkt_gmres_solve(kkt_ctx* ctx, const double* b, double* x, kkt_gmres_result* res,
                    double* history, int32_t history_cap) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(b && x && res && b != x, "kkt_gmres_solve: bad arguments");
    kkt::gmres(c, b, x, res, history, history_cap);
  });
}

int kkt_gmres_solve_host(kkt_ctx* ctx, const double* b_host, double* x_host,
                         kkt_gmres_result* res, double* history, int32_t history_cap) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(b_host && x_host && res, "kkt_gmres_solve_host: bad arguments");
    const size_t n = size_t(3 * c->B);
    if (c->e2e_b.n < n) c->e2e_b.alloc(n);
    if (c->e2e_x.n < n) c->e2e_x.alloc(n);
    KKT_CUDA(cudaMemcpyAsync(c->e2e_b.p, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    kkt::gmres(c, c->e2e_b.p, c->e2e_x.p, res, history, history_cap);
    KKT_CUDA(cudaMemcpyAsync(x_host, c->e2e_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// apply_P_inv from host buffers, with the copies overlapped with the compute: P^-1 is block
// diagonal (kkt.cpp:71-81), so the Schur block's sweep needs only r_w.  r_w goes up first and the
// sweep starts.  r_u and r_z follow in chunks on the copy-in stream while it runs; each chunk is
// divided on a side stream as soon as it has landed and goes straight back down (PCIe is full
// duplex), so the u/z download runs one chunk behind the upload instead of after it.  Where the
// sweep's output is the final w block its finished planes trail the adjoint sweep on a third copy
// stream.  The kernels of the sweep must not touch a copy engine (a cudaMemsetAsync queued behind
// the bulk upload stalled the sweep until the upload was over: dev_fill is a kernel).  With pinned
// host memory the end-to-end time approaches one block up plus the larger of the sweep and three
// blocks down, instead of the sweep plus three blocks each way.
int kkt_apply_P_inv_host(kkt_ctx* ctx, const double* r_host, double* out_host) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(r_host && out_host, "kkt_apply_P_inv_host: bad arguments");
    const size_t B = size_t(c->B), n = 3 * B;
    if (c->e2e_b.n < n) c->e2e_b.alloc(n);
    if (c->e2e_x.n < n) c->e2e_x.alloc(n);
    if (!c->e2e_in) {
      KKT_CUDA(cudaStreamCreateWithFlags(&c->e2e_in, cudaStreamNonBlocking));
      KKT_CUDA(cudaStreamCreateWithFlags(&c->e2e_out, cudaStreamNonBlocking));
      KKT_CUDA(cudaStreamCreateWithFlags(&c->e2e_aux, cudaStreamNonBlocking));
      for (auto& e : c->e2e_ev) KKT_CUDA(cudaEventCreate(&e));
    }
    double* in = c->e2e_b.p;
    double* out = c->e2e_x.p;
    const size_t bytes = sizeof(double) * B;
    cudaEvent_t* ev = c->e2e_ev;  // 0: start, 1: r_w up, 2: r_u r_z up, 3: u z computed, 4: w done
    // KKT_E2E_CHUNK_KB: KB of each block per chunk of the u/z pipeline (default 64 MB; 0: the blocks whole)
    static const long chunk_kb = std::getenv("KKT_E2E_CHUNK_KB") ? std::atol(std::getenv("KKT_E2E_CHUNK_KB")) : 65536;
    const size_t chunk = chunk_kb > 0 ? std::min(B, size_t(chunk_kb) << 7) : B;  // doubles per block per chunk
    const size_t nchunks = (B + chunk - 1) / chunk;
    while (c->e2e_chunk_ev.size() < nchunks) {
      cudaEvent_t e;
      KKT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->e2e_chunk_ev.push_back(e);
    }
    // the staging vectors may still be read by earlier work on the context stream
    KKT_CUDA(cudaEventRecord(ev[0], c->stream));
    KKT_CUDA(cudaStreamWaitEvent(c->e2e_in, ev[0], 0));
    KKT_CUDA(cudaStreamWaitEvent(c->e2e_aux, ev[0], 0));
    KKT_CUDA(cudaMemcpyAsync(in + 2 * B, r_host + 2 * B, bytes, cudaMemcpyHostToDevice, c->e2e_in));
    KKT_CUDA(cudaEventRecord(ev[1], c->e2e_in));
    // u and z blocks, chunk by chunk: up on the copy-in stream, divided and sent down on the side
    // stream (the kernels launch on c->stream: swap it for the calls).  Enqueued before the sweep
    // so that none of it queues behind the sweep's launches.
    for (size_t q = 0; q < nchunks; ++q) {
      const size_t o = q * chunk, len = std::min(chunk, B - o);
      KKT_CUDA(cudaMemcpyAsync(in + o, r_host + o, sizeof(double) * len, cudaMemcpyHostToDevice, c->e2e_in));
      KKT_CUDA(cudaMemcpyAsync(in + B + o, r_host + B + o, sizeof(double) * len, cudaMemcpyHostToDevice, c->e2e_in));
      KKT_CUDA(cudaEventRecord(c->e2e_chunk_ev[q], c->e2e_in));
      KKT_CUDA(cudaStreamWaitEvent(c->e2e_aux, c->e2e_chunk_ev[q], 0));
      cudaStream_t keep = c->stream;
      c->stream = c->e2e_aux;
      try {
        kkt::op_pinv_uz_range(c, in, out, int64_t(o), int64_t(o + len));
      } catch (...) {
        c->stream = keep;
        throw;
      }
      c->stream = keep;
      if (q + 1 == nchunks) KKT_CUDA(cudaEventRecord(ev[3], c->e2e_aux));
      KKT_CUDA(cudaMemcpyAsync(out_host + o, out + o, sizeof(double) * len, cudaMemcpyDeviceToHost, c->e2e_aux));
      KKT_CUDA(cudaMemcpyAsync(out_host + B + o, out + B + o, sizeof(double) * len, cudaMemcpyDeviceToHost, c->e2e_aux));
    }
    KKT_CUDA(cudaEventRecord(ev[2], c->e2e_in));
    // Schur block on the context stream.  Where the RASQ sweep's output is the final w block
    // (one-level; two-level literal; the fused multiplicative form) and the host buffer is pinned,
    // the sweep sends each adjoint step's finished planes to the host behind the step
    // (rasq_apply's step hook, on its own copy stream), so the w download overlaps the sweep
    // instead of following it.
    KKT_CUDA(cudaStreamWaitEvent(c->stream, ev[1], 0));
    {
      static const bool trail_off = std::getenv("KKT_E2E_TRAIL_OFF") != nullptr;  // testing: one copy at the end
      const auto& d = c->desc;
      const bool fused = d.precond == KKT_PRECOND_TWO_LEVEL && d.two_level_form == KKT_FORM_MULTIPLICATIVE &&
                         !c->perdof && c->mode == KKT_MODE_FAST && c->has_fast() && !(c->bisect & 5);
      const bool final_rasq = d.precond == KKT_PRECOND_ONE_LEVEL || fused ||
                              (d.precond == KKT_PRECOND_TWO_LEVEL && d.two_level_form == KKT_FORM_LITERAL);
      cudaPointerAttributes pa{};
      const bool pinned = cudaPointerGetAttributes(&pa, out_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
      (void)cudaGetLastError();
      c->e2e_trailed = false;
      if (final_rasq && pinned && !trail_off) {
        if (!c->e2e_step_ev) {
          KKT_CUDA(cudaEventCreateWithFlags(&c->e2e_step_ev, cudaEventDisableTiming));
          KKT_CUDA(cudaStreamCreateWithFlags(&c->e2e_trail, cudaStreamNonBlocking));
        }
        c->e2e_w_host = out_host + 2 * B;
      }
      try {
        kkt::schur_apply(c, in + 2 * B, out + 2 * B);
      } catch (...) {
        c->e2e_w_host = nullptr;
        throw;
      }
      c->e2e_w_host = nullptr;
    }
    KKT_CUDA(cudaEventRecord(ev[4], c->stream));
    if (!c->e2e_trailed) {
      KKT_CUDA(cudaStreamWaitEvent(c->e2e_out, ev[4], 0));
      KKT_CUDA(cudaMemcpyAsync(out_host + 2 * B, out + 2 * B, bytes, cudaMemcpyDeviceToHost, c->e2e_out));
    } else {
      KKT_CUDA(cudaStreamSynchronize(c->e2e_trail));
    }
    KKT_CUDA(cudaStreamSynchronize(c->e2e_out));
    KKT_CUDA(cudaStreamSynchronize(c->e2e_aux));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    static const bool tim = std::getenv("KKT_E2E_TIM") != nullptr;  // stage completion times since the start
    if (tim) {
      cudaEvent_t done;
      KKT_CUDA(cudaEventCreate(&done));
      KKT_CUDA(cudaEventRecord(done, c->stream));  // everything has been synchronised: the end of the call
      KKT_CUDA(cudaEventSynchronize(done));
      float t[5] = {0, 0, 0, 0, 0};
      for (int i = 1; i < 5; ++i) KKT_CUDA(cudaEventElapsedTime(&t[i], ev[0], ev[i]));
      KKT_CUDA(cudaEventElapsedTime(&t[0], ev[0], done));
      std::fprintf(stderr, "P_inv_host ms since start: r_w up %.1f, r_u r_z up %.1f, u z computed %.1f, sweep done %.1f, all down %.1f (%zu u/z chunks%s)\n",
                   t[1], t[2], t[3], t[4], t[0], nchunks, c->e2e_trailed ? "; w planes trailed the adjoint sweep" : "");
      cudaEventDestroy(done);
    }
  });
}

namespace kkt {
namespace {
// assemble_rhs (kkt.cpp:29-48) with model_initial_condition / model_target
// (model_problem.hpp:11-18), for the local slab; same expressions and order.
void model_rhs(const Ctx* c, double* b, double* target) {
  const double two_pi = 2.0 * 3.141592653589793;  // 2 * std::numbers::pi
  const int64_t B = c->B;
  for (int nl = 0; nl < c->ntl; ++nl) {
    const int n = c->n0 + nl;
    const double t = n * c->dt;
    for (int j = 1; j <= c->ny; ++j) {
      for (int i = 1; i <= c->nx; ++i) {
        const double x = i * c->dx, y = j * c->dy;
        const int64_t k = (int64_t(nl) * c->ny + (j - 1)) * c->nx + (i - 1);
        const double tv = std::sin(two_pi * t) * std::sin(two_pi * x) * std::sin(two_pi * y);
        b[k] = c->ms * tv;
        b[B + k] = 0.0;
        b[2 * B + k] = n == 1 ? -x * y * (x - 1.0) * (y - 2.0) : 0.0;
        if (target) target[k] = tv;
      }
    }
  }
}
}  // namespace
}  // namespace kkt

int kkt_evaluate_objective(kkt_ctx* ctx, const double* u, const double* z, const double* target,
                           double* objective) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(u && z && target && objective, "evaluate_objective: bad arguments");
    *objective = kkt::kkt_objective(c, u, z, target);
  });
}

int kkt_model_rhs(kkt_ctx* ctx, double* b_host, double* target_host) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(b_host != nullptr, "model_rhs: bad arguments");
    kkt::model_rhs(c, b_host, target_host);
  });
}

int kkt_run_single(const kkt_problem_desc* desc, const kkt_runtime_opts* opts, kkt_run_record* rec,
                   double* x_host) {
  if (!desc || !rec) return KKT_EINVAL;
  using clock = std::chrono::steady_clock;
  auto secs = [](clock::time_point a) { return std::chrono::duration<double>(clock::now() - a).count(); };
  const auto t_setup = clock::now();
  kkt_ctx* ctx = nullptr;
  int st = kkt_ctx_create(desc, opts, &ctx);
  if (st != KKT_OK) return st;
  st = kkt::guard(ctx, [&](Ctx* c) {
    const size_t B = size_t(c->B);
    std::vector<double> b(3 * B), tgt(B);
    kkt::model_rhs(c, b.data(), tgt.data());
    kkt::DBuf<double> db{3 * B}, dx{3 * B}, dt{B};
    KKT_CUDA(cudaMemcpyAsync(db.p, b.data(), sizeof(double) * 3 * B, cudaMemcpyHostToDevice, c->stream));
    KKT_CUDA(cudaMemcpyAsync(dt.p, tgt.data(), sizeof(double) * B, cudaMemcpyHostToDevice, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    rec->setup_seconds = secs(t_setup);
    const auto t_solve = clock::now();
    kkt_gmres_result res{};
    kkt::gmres(c, db.p, dx.p, &res, nullptr, 0);
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    rec->solve_seconds = secs(t_solve);
    rec->iterations = res.iterations;
    rec->converged = res.converged;
    rec->true_final_relres = res.true_final_relres;
    rec->objective = kkt::kkt_objective(c, dx.p, dx.p + B, dt.p);
    if (x_host) {
      KKT_CUDA(cudaMemcpyAsync(x_host, dx.p, sizeof(double) * 3 * B, cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
  if (st != KKT_OK) {
    kkt::g_create_err = kkt_last_error(ctx);
    kkt::g_create_err_index = kkt_last_error_index(ctx);
  }
  kkt_ctx_destroy(ctx);
  return st;
}

int kkt_launch_count(const kkt_ctx* ctx, int64_t* count) {
  if (!ctx || !count) return KKT_EINVAL;
  *count = ctx->impl.launches;
  return KKT_OK;
}

int kkt_reset_launch_count(kkt_ctx* ctx) {
  if (!ctx) return KKT_EINVAL;
  ctx->impl.launches = 0;
  return KKT_OK;
}

int kkt_set_phase_timing(kkt_ctx* ctx, int32_t on) {
  if (!ctx) return KKT_EINVAL;
  Ctx& c = ctx->impl;
  c.phase_timing = on != 0;
  for (int i = 0; i < 4; ++i) { c.phase_ms[i] = 0; c.phase_cnt[i] = 0; }
  return KKT_OK;
}

int kkt_phase_times(const kkt_ctx* ctx, double* ms4, int64_t* counts4) {
  if (!ctx) return KKT_EINVAL;
  const_cast<kkt_ctx*>(ctx)->impl.tcollect();
  for (int i = 0; i < 4; ++i) {
    if (ms4) ms4[i] = ctx->impl.phase_ms[i];
    if (counts4) counts4[i] = ctx->impl.phase_cnt[i];
  }
  return KKT_OK;
}

int kkt_debug_ahat_factor(kkt_ctx* ctx, int32_t* kl, int32_t* ku, double* ab_host,
                          int32_t* piv_host) {
  return kkt::guard(ctx, [&](Ctx* c) {
    if (kl) *kl = c->kl;
    if (ku) *ku = c->kuf;
    if (ab_host) {
      KKT_CUDA(cudaMemcpyAsync(ab_host, c->ab.p, sizeof(double) * c->ab.n, cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (piv_host) {
      KKT_CUDA(cudaMemcpyAsync(piv_host, c->piv.p, sizeof(int) * c->piv.n, cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
}

int kkt_debug_coarse_factor(kkt_ctx* ctx, int32_t* kl, int32_t* ku, double* ab_host,
                            int32_t* piv_host) {
  return kkt::guard(ctx, [&](Ctx* c) {
    kkt::need(c->has_coarse && c->perdof, "no per-dof coarse space");
    if (kl) *kl = c->cb_kl;
    if (ku) *ku = c->cb_kuf;
    if (ab_host) {
      KKT_CUDA(cudaMemcpyAsync(ab_host, c->cb_ab.p, sizeof(double) * c->cb_ab.n, cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (piv_host) {
      KKT_CUDA(cudaMemcpyAsync(piv_host, c->cb_piv.p, sizeof(int) * c->cb_piv.n, cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
}

int kkt_nccl_unique_id(void* out128) {
  if (!out128) return KKT_EINVAL;
  try {
    return kkt::nccl_unique_id(out128);
  } catch (const Error& e) {
    kkt::g_create_err = e.what();
    return e.status;
  }
}

int kkt_local_group_create(int32_t nranks, void** out) {
  if (!out || nranks < 1) return KKT_EINVAL;
  *out = kkt::local_group_create(nranks);
  return KKT_OK;
}

int kkt_local_group_destroy(void* group) {
  kkt::local_group_destroy(group);
  return KKT_OK;
}

}  // extern "C"
