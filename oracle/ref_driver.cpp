// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the
// product).  A thin extern "C" driver around the UNMODIFIED reference library
// compiled from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libkktdd_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference / cpu_baseline legs may load it.
//
// It wires the reference exactly like run_single does
// (proj/src/experiments.cpp:33-57): HeatOperators, build_time_partition,
// make_schur_solver, then gmres_solve with the apply_K / apply_P_inv lambdas —
// except that the right-hand side is supplied by the caller (the harness's
// seeded generator) instead of model_problem.hpp.
#include <cstdio>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

// Read-only access to BandedLU's private factor storage for the factor-parity
// test (linalg.hpp:45-75).  Nothing is modified.
#define private public
#include "kktdd/linalg.hpp"
#undef private
#include "kktdd/config.hpp"
#include "kktdd/experiments.hpp"
#include "kktdd/model_problem.hpp"
#include "kktdd/gmres.hpp"
#include "kktdd/heat_operators.hpp"
#include "kktdd/kkt.hpp"
#include "kktdd/schur.hpp"
#include "kktdd/time_partition.hpp"

#include "../include/kktdd_b200.h"

using namespace kktdd;

namespace {

thread_local std::string g_err;
thread_local int g_err_index = -1;

struct RefCtx {
  ProblemConfig cfg;
  std::unique_ptr<HeatOperators> ops;
  std::unique_ptr<TimePartition> part;
  std::unique_ptr<SchurSolver> schur;
};

ProblemConfig to_cfg(const kkt_problem_desc* d) {
  ProblemConfig c;
  c.Lx = d->Lx;
  c.Ly = d->Ly;
  c.T = d->T;
  c.Nx = d->Nx;
  c.Ny = d->Ny;
  c.Nt = d->Nt;
  c.nu = d->nu;
  c.omega = d->omega;
  c.Nd = d->Nd;
  c.precond = static_cast<PrecondKind>(d->precond);
  c.coarse_variant = static_cast<CoarseVariant>(d->coarse_variant);
  c.two_level_form = static_cast<TwoLevelForm>(d->two_level_form);
  c.jhat_sign = d->jhat_sign == KKT_SIGN_PLUS ? JhatSign::plus : JhatSign::minus;
  c.gmres.tol = d->tol;
  c.gmres.max_iters = d->max_iters;
  if (d->restart != KKT_NO_RESTART) c.gmres.restart = d->restart;  // < 1 -> validate() throws
  c.gmres.happy_breakdown_tol = d->happy_breakdown_tol;
  return c;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    g_err_index = -1;
    return KKT_OK;
  } catch (const SingularMatrixError& e) {
    g_err = e.what();
    g_err_index = e.pivot_index;
    return KKT_ESINGULAR;
  } catch (const GmresDivergenceError& e) {
    g_err = e.what();
    g_err_index = e.iteration;
    return KKT_EDIVERGED;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return KKT_ECONFIG;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return KKT_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

std::size_t nb(const RefCtx* c) { return c->ops->layout.size(); }

std::span<const double> cin(const double* p, std::size_t n) { return {p, n}; }
std::span<double> cout_(double* p, std::size_t n) { return {p, n}; }

}  // namespace

extern "C" {

const char* ref_error(void) { return g_err.c_str(); }
int ref_error_index(void) { return g_err_index; }

int ref_create(const kkt_problem_desc* d, void** out) {
  return guarded([&] {
    auto c = std::make_unique<RefCtx>();
    c->cfg = to_cfg(d);
    c->cfg.validate();
    c->ops = std::make_unique<HeatOperators>(c->cfg);
    c->part = std::make_unique<TimePartition>(build_time_partition(c->cfg.Nt, c->cfg.Nd));
    c->schur = std::make_unique<SchurSolver>(make_schur_solver(*c->ops, *c->part, c->cfg));
    *out = c.release();
  });
}

void ref_destroy(void* c) { delete static_cast<RefCtx*>(c); }

int64_t ref_block(void* c) { return static_cast<int64_t>(nb(static_cast<RefCtx*>(c))); }

#define REF_UNARY(name, fn)                                                     \
  int name(void* vc, const double* in, double* out) {                          \
    auto* c = static_cast<RefCtx*>(vc);                                         \
    return guarded([&] { fn(*c->ops, cin(in, nb(c)), cout_(out, nb(c))); }); \
  }
REF_UNARY(ref_apply_J, apply_J)
REF_UNARY(ref_apply_JT, apply_JT)
REF_UNARY(ref_apply_L, apply_L)
REF_UNARY(ref_apply_LT, apply_LT)
REF_UNARY(ref_apply_Mu, apply_Mu)
REF_UNARY(ref_apply_Mu_inv, apply_Mu_inv)
REF_UNARY(ref_apply_Mz, apply_Mz)
REF_UNARY(ref_apply_Jhat, apply_Jhat)
REF_UNARY(ref_apply_JhatT, apply_JhatT)
REF_UNARY(ref_apply_shat, apply_shat)
#undef REF_UNARY

int ref_apply_K(void* vc, const double* v, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] { apply_K(*c->ops, cin(v, 3 * nb(c)), cout_(out, 3 * nb(c))); });
}

int ref_apply_P_inv(void* vc, const double* r, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded(
      [&] { apply_P_inv(*c->ops, *c->schur, cin(r, 3 * nb(c)), cout_(out, 3 * nb(c))); });
}

int ref_schur_apply(void* vc, const double* r, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] { c->schur->apply(cin(r, nb(c)), cout_(out, nb(c))); });
}

int ref_apply_rasq(void* vc, const double* r, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    SpaceTimeVector rv(r, r + nb(c));
    SpaceTimeVector o = apply_rasq(*c->ops, *c->part, rv);
    std::memcpy(out, o.data(), sizeof(double) * o.size());
  });
}

int ref_apply_two_level(void* vc, const double* r, double* out, int form) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const CoarseSpace* cs = c->schur->coarse();
    if (!cs) throw ConfigError("ref_apply_two_level: solver has no coarse space");
    SpaceTimeVector rv(r, r + nb(c));
    SpaceTimeVector o =
        apply_two_level(*c->ops, *c->part, *cs, rv, static_cast<TwoLevelForm>(form));
    std::memcpy(out, o.data(), sizeof(double) * o.size());
  });
}

int ref_forward_solve_window(void* vc, double* b, int len) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    forward_solve_window(*c->ops, cout_(b, static_cast<std::size_t>(len) * c->ops->layout.n_sp()));
  });
}

int ref_adjoint_solve_window(void* vc, double* b, int len) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    adjoint_solve_window(*c->ops, cout_(b, static_cast<std::size_t>(len) * c->ops->layout.n_sp()));
  });
}

int ref_band_solve(void* vc, double* b, int nrhs, int transpose) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const std::size_t nsp = c->ops->layout.n_sp();
    for (int k = 0; k < nrhs; ++k) {
      auto s = cout_(b + k * nsp, nsp);
      if (transpose)
        c->ops->Ahat_factors.solve_transpose_in_place(s);
      else
        c->ops->Ahat_factors.solve_in_place(s);
    }
  });
}

// Band storage of the Ahat factor: (kl + ku_ + 1) rows per column, col-major
// (linalg.hpp:65-74).  Returns kl, ku_ and the pivot vector.
int ref_ahat_factor(void* vc, int* kl, int* ku, double* ab, int* piv, double* pivot_growth) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const BandedLU& F = c->ops->Ahat_factors;
    *kl = F.kl_;
    *ku = F.ku_;
    if (ab) std::memcpy(ab, F.ab_.data(), sizeof(double) * F.ab_.size());
    if (piv) std::memcpy(piv, F.piv_.data(), sizeof(int) * F.piv_.size());
    if (pivot_growth) *pivot_growth = F.pivot_growth_;
  });
}

int ref_coarse_dim(void* vc) {
  auto* c = static_cast<RefCtx*>(vc);
  const CoarseSpace* cs = c->schur->coarse();
  return cs ? cs->dim() : -1;
}

int ref_coarse_restrict(void* vc, const double* r, double* cvec) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const CoarseSpace* cs = c->schur->coarse();
    cs->restrict_to_coarse(c->ops->layout, *c->part, cin(r, nb(c)), cout_(cvec, cs->dim()));
  });
}

int ref_coarse_solve(void* vc, double* cvec) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const CoarseSpace* cs = c->schur->coarse();
    cs->solve_in_place(cout_(cvec, cs->dim()));
  });
}

int ref_coarse_prolong_add(void* vc, const double* cvec, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const CoarseSpace* cs = c->schur->coarse();
    cs->prolong_add(c->ops->layout, *c->part, cin(cvec, cs->dim()), cout_(out, nb(c)));
  });
}

int ref_coarse_matrix(void* vc, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const CoarseSpace* cs = c->schur->coarse();
    DenseMatrix m = cs->coarse_matrix_dense();
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
  });
}

// run_single's solve (experiments.cpp:46-57) on a caller-supplied rhs.
int ref_gmres_solve(void* vc, const double* b, double* x, kkt_gmres_result* res,
                    double* history, int history_cap) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const HeatOperators& ops = *c->ops;
    const SchurSolver& schur = *c->schur;
    const LinearMap op = [&](std::span<const double> v, std::span<double> o) {
      apply_K(ops, v, o);
    };
    LinearMap prec;
    if (c->cfg.precond != PrecondKind::none) {
      prec = [&](std::span<const double> v, std::span<double> o) {
        apply_P_inv(ops, schur, v, o);
      };
    }
    GmresResult r = gmres_solve(op, prec, cin(b, 3 * nb(c)), c->cfg.gmres);
    std::memcpy(x, r.solution.data(), sizeof(double) * r.solution.size());
    res->converged = r.converged ? 1 : 0;
    res->iterations = r.iterations;
    res->true_final_relres = r.true_final_relres;
    const int nh = std::min<int>(history_cap, static_cast<int>(r.residual_history.size()));
    res->history_len = nh;
    if (history) std::memcpy(history, r.residual_history.data(), sizeof(double) * nh);
  });
}

int ref_kkt_residual(void* vc, const double* v, const double* rhs, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    KKTVector kv(nb(c));
    std::memcpy(kv.data.data(), v, sizeof(double) * 3 * nb(c));
    RhsBundle b;
    b.f_u.assign(rhs, rhs + nb(c));
    b.f_z.assign(rhs + nb(c), rhs + 2 * nb(c));
    b.f.assign(rhs + 2 * nb(c), rhs + 3 * nb(c));
    *out = kkt_residual(*c->ops, kv, b);
  });
}

// gmres_solve on a dense row-major operator (and optional dense right
// preconditioner), for the reference's own GMRES unit cases (test_gmres.cpp).
int ref_gmres_dense(int n, const double* A, const double* M, const double* b, double tol,
                    int max_iters, int restart, double* x, kkt_gmres_result* res,
                    double* history, int history_cap) {
  return guarded([&] {
    auto dense = [n](const double* m) {
      return [n, m](std::span<const double> v, std::span<double> o) {
        for (int i = 0; i < n; ++i) {
          double acc = 0.0;
          for (int j = 0; j < n; ++j) acc += m[static_cast<std::size_t>(i) * n + j] * v[j];
          o[i] = acc;
        }
      };
    };
    GmresParams p;
    p.tol = tol;
    p.max_iters = max_iters;
    if (restart > 0) p.restart = restart;
    LinearMap prec;
    if (M) prec = dense(M);
    GmresResult r = gmres_solve(dense(A), prec, cin(b, n), p);
    std::memcpy(x, r.solution.data(), sizeof(double) * n);
    res->converged = r.converged;
    res->iterations = r.iterations;
    res->true_final_relres = r.true_final_relres;
    const int nh = std::min<int>(history_cap, static_cast<int>(r.residual_history.size()));
    res->history_len = nh;
    if (history) std::memcpy(history, r.residual_history.data(), sizeof(double) * nh);
  });
}

// run_single itself (experiments.cpp:33-69) and its JSON record
// (experiments.cpp:179-208): the f1 record the device's kkt_run_single mirrors.
int ref_run_single(const kkt_problem_desc* d, kkt_run_record* rec, double* x, char* json,
                   int json_cap) {
  return guarded([&] {
    ProblemConfig cfg = to_cfg(d);
    GmresResult res;
    RunRecord r = run_single(cfg, &res);
    rec->iterations = r.iterations;
    rec->converged = r.converged ? 1 : 0;
    rec->true_final_relres = r.true_final_relres;
    rec->objective = r.objective;
    rec->setup_seconds = r.setup_seconds;
    rec->solve_seconds = r.solve_seconds;
    if (x) std::memcpy(x, res.solution.data(), sizeof(double) * res.solution.size());
    if (json && json_cap > 0) {
      const std::string js = to_json_string(r);
      std::snprintf(json, static_cast<std::size_t>(json_cap), "%s", js.c_str());
    }
  });
}

// The reference's own sweeps (experiments.cpp:97-142) and their CSV
// (experiments.cpp:144-177): the f3 records the device sweeps mirror.
// kind 0: weak_scaling_sweep(base, steps, nts, omegas, preconds)
// kind 1: omega_sweep(base, nt, nd, omegas, preconds)
int ref_sweep_csv(int kind, const kkt_problem_desc* d, int steps, int nt, int nd, const int* nts,
                  int n_nts, const double* omegas, int n_omegas, const int* preconds, int n_preconds,
                  char* csv, int csv_cap) {
  return guarded([&] {
    ProblemConfig base = to_cfg(d);
    std::vector<int> ntl(nts, nts + n_nts);
    std::vector<double> oml(omegas, omegas + n_omegas);
    std::vector<PrecondKind> pl;
    for (int i = 0; i < n_preconds; ++i) pl.push_back(static_cast<PrecondKind>(preconds[i]));
    const SweepResult sw = kind == 0 ? weak_scaling_sweep(base, steps, ntl, oml, pl)
                                     : omega_sweep(base, nt, nd, oml, pl);
    const std::string text = to_csv(sw);
    std::snprintf(csv, static_cast<std::size_t>(csv_cap), "%s", text.c_str());
  });
}

// assemble_rhs(ops, model_initial_condition, model_target).to_kkt() and the
// target samples evaluate_objective uses (kkt.cpp:88-108).
int ref_model_rhs(void* vc, double* b, double* target) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const HeatOperators& ops = *c->ops;
    const KKTVector kb = assemble_rhs(ops, model_initial_condition, model_target).to_kkt();
    std::memcpy(b, kb.data.data(), sizeof(double) * kb.data.size());
    const auto& L = ops.layout;
    for (int n = 1; n <= L.nt; ++n)
      for (int j = 1; j <= L.ny_int; ++j)
        for (int i = 1; i <= L.nx_int; ++i)
          target[L.index(n, i, j)] = model_target(i * c->cfg.dx(), j * c->cfg.dy(), n * ops.dt);
  });
}

int ref_evaluate_objective(void* vc, const double* u, const double* z, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] { *out = evaluate_objective(*c->ops, cin(u, nb(c)), cin(z, nb(c)), model_target); });
}

// The acceptance suite's zero-control comparison (acceptance_main.cpp:70-84,
// :443-448): objective of the state driven by f alone, z = 0.
int ref_zero_control_objective(void* vc, double* out) {
  auto* c = static_cast<RefCtx*>(vc);
  return guarded([&] {
    const HeatOperators& ops = *c->ops;
    const RhsBundle rhs = assemble_rhs(ops, model_initial_condition, model_target);
    const int nsp = ops.layout.n_sp();
    SpaceTimeVector u = ops.layout.zeros();
    std::vector<double> step(nsp);
    for (int n = 1; n <= ops.layout.nt; ++n) {
      const std::size_t off = ops.layout.node_offset(n);
      for (int p = 0; p < nsp; ++p) {
        step[p] = rhs.f[off + p];
        if (n > 1) step[p] += u[ops.layout.node_offset(n - 1) + p];
      }
      ops.A_factors.solve_in_place(step);
      std::copy(step.begin(), step.end(), u.begin() + off);
    }
    *out = evaluate_objective(ops, u, ops.layout.zeros(), model_target);
  });
}

}  // extern "C"
