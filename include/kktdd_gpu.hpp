// kktdd_gpu.hpp — the reference-side C++ binding over libkktdd_b200.so.
//
// Header-only, C++20, no CUDA headers needed: it talks to the device only
// through the C-ABI of include/kktdd_b200.h.  It re-exports the hot path of the
// reference library `kktdd` (/root/reference/proj/include/kktdd/*.hpp) under the
// reference's own names, argument meaning and error behaviour:
//
//   ProblemConfig, GmresParams, enums, ConfigError      config.hpp:12-85
//   SpaceTimeLayout, SpaceTimeVector                    layout.hpp:13-44
//   TimePartition, NodeRange, build_time_partition      time_partition.hpp:11-45
//   HeatOperators, apply_J/JT/L/LT/Mu/Mu_inv/Mz/Jhat/JhatT,
//   forward_solve_window, adjoint_solve_window          heat_operators.hpp:26-61
//   KKTVector, RhsBundle, assemble_rhs, apply_K, apply_P_inv,
//   evaluate_objective, kkt_residual                    kkt.hpp:15-65
//   apply_shat, apply_rasq, CoarseSpace, build_coarse_space, apply_two_level,
//   SchurSolver, make_schur_solver                      schur.hpp:22-143
//   GmresResult, GmresDivergenceError, gmres_solve      gmres.hpp:13-36
//   RunRecord, run_single                               experiments.hpp:14-31
//   model_initial_condition, model_target               model_problem.hpp:11-18
//
// Differences from the reference, all forced by the device:
//   * HeatOperators owns a device context (kkt_ctx) instead of CPU band
//     factors; it is movable, not copyable.  Its constructor takes the
//     arithmetic mode (Arithmetic::fast, the performance path, or ::strict,
//     bitwise the reference).
//   * std::span / std::vector arguments are HOST memory, as in the reference;
//     every call copies in and out through kkt_copy_to_device / _to_host.  Code
//     that keeps its vectors on the device calls the C-ABI entry points with
//     ops.ctx() directly (that is what gmres_solve does internally: the whole
//     Krylov solve runs on the device, only b and x cross).
//   * gmres_solve takes the operators and the Schur solver instead of two
//     std::function maps: a host callback per Krylov step would put the host
//     back on the hot path.  It is run_single's wiring (experiments.cpp:46-57).
//   * The dense-oracle Schur kinds (dense_shat, dense_ras, dense_true;
//     schur.cpp:13-21) are desk-scale test oracles and are not offered.
//
// Link: -L paper_2305_04421_b200/_lib -lkktdd_b200 (static cudart inside).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstring>
#include <functional>
#include <memory>
#include <numbers>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kktdd_b200.h"

namespace kktdd_gpu {

// ---------------------------------------------------------------- config.hpp
enum class PrecondKind { none, one_level, two_level, dense_schur, true_schur };
enum class CoarseVariant { scalar, per_dof };
enum class TwoLevelForm { literal, multiplicative, additive };
enum class JhatSign { plus, minus };
enum class Arithmetic { fast = KKT_MODE_FAST, strict = KKT_MODE_STRICT };

struct GmresParams {
  double tol = 1e-6;
  int max_iters = 420;
  std::optional<int> restart;  // no value = full (non-restarted) GMRES
  double happy_breakdown_tol = 1e-14;
};

struct ProblemConfig {
  double Lx = 1.0, Ly = 2.0, T = 1.0;
  int Nx = 16, Ny = 16, Nt = 100;
  double nu = 1.0, omega = 1e-3;
  int Nd = 5;
  PrecondKind precond = PrecondKind::two_level;
  CoarseVariant coarse_variant = CoarseVariant::per_dof;
  TwoLevelForm two_level_form = TwoLevelForm::multiplicative;
  JhatSign jhat_sign = JhatSign::minus;
  GmresParams gmres;

  double dx() const { return Lx / Nx; }
  double dy() const { return Ly / Ny; }
  double dt() const { return T / Nt; }
  int nx_interior() const { return Nx - 1; }
  int ny_interior() const { return Ny - 1; }
  int n_sp() const { return nx_interior() * ny_interior(); }
  double mass_scale() const { return dt() * dx() * dy(); }
  double sigma() const { return ((jhat_sign == JhatSign::plus) ? 1.0 : -1.0) / std::sqrt(omega); }
};

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};
class SingularMatrixError : public std::runtime_error {  // linalg.hpp:14-19
 public:
  SingularMatrixError(const std::string& what, int pivot) : std::runtime_error(what), pivot_index(pivot) {}
  int pivot_index;
};
class GmresDivergenceError : public std::runtime_error {  // gmres.hpp:22-27
 public:
  GmresDivergenceError(const std::string& what, int it) : std::runtime_error(what), iteration(it) {}
  int iteration;
};

// ---------------------------------------------------------------- layout.hpp
using SpaceTimeVector = std::vector<double>;

struct SpaceTimeLayout {
  int nt = 0, nx_int = 0, ny_int = 0;
  int n_sp() const { return nx_int * ny_int; }
  std::size_t size() const { return static_cast<std::size_t>(nt) * n_sp(); }
  int spatial_index(int i, int j) const { return (j - 1) * nx_int + (i - 1); }
  std::size_t index(int n, int p) const { return static_cast<std::size_t>(n - 1) * n_sp() + p; }
  std::size_t index(int n, int i, int j) const { return index(n, spatial_index(i, j)); }
  std::size_t node_offset(int n) const { return static_cast<std::size_t>(n - 1) * n_sp(); }
  SpaceTimeVector zeros() const { return SpaceTimeVector(size(), 0.0); }
};
inline SpaceTimeLayout make_layout(const ProblemConfig& c) {
  return SpaceTimeLayout{c.Nt, c.nx_interior(), c.ny_interior()};
}

// -------------------------------------------------------- time_partition.hpp
struct NodeRange {
  int first = 0, last = -1;
  int count() const { return last - first + 1; }
  bool contains(int n) const { return n >= first && n <= last; }
};

struct TimePartition {
  int nt = 0, nd = 0, m = 0;
  std::vector<NodeRange> nodes, owned, extended;
  std::vector<int> owner;  // owner[n], n = 1..nt
  std::optional<int> w_node(int s) const {
    return extended[s].first < nodes[s].first ? std::optional<int>(extended[s].first) : std::nullopt;
  }
};

// Pure index arithmetic (time_partition.cpp:61-86); the device context builds
// the same partition for itself from Nt and Nd.
inline TimePartition build_time_partition(int nt, int nd) {
  if (nt < 1 || nd < 1) throw ConfigError("time partition needs Nt, Nd >= 1");
  if (nt % nd != 0)
    throw ConfigError("Nt=" + std::to_string(nt) + " is not divisible by Nd=" + std::to_string(nd));
  TimePartition p;
  p.nt = nt;
  p.nd = nd;
  p.m = nt / nd;
  p.owner.assign(nt + 1, 0);
  for (int n = 1; n <= nt; ++n) p.owner[n] = (n - 1) / p.m;
  for (int s = 0; s < nd; ++s) {
    const int last = (s + 1) * p.m, first = s == 0 ? 1 : s * p.m;
    p.nodes.push_back({first, last});
    p.owned.push_back({s == 0 ? 1 : s * p.m + 1, last});
    p.extended.push_back({first > 1 ? first - 1 : 1, last});
  }
  return p;
}

// -------------------------------------------------------------------- detail
namespace detail {

inline kkt_problem_desc to_desc(const ProblemConfig& c) {
  kkt_problem_desc d;
  kkt_problem_desc_default(&d);
  d.Lx = c.Lx; d.Ly = c.Ly; d.T = c.T;
  d.Nx = c.Nx; d.Ny = c.Ny; d.Nt = c.Nt;
  d.nu = c.nu; d.omega = c.omega; d.Nd = c.Nd;
  d.precond = static_cast<int>(c.precond);
  d.coarse_variant = static_cast<int>(c.coarse_variant);
  d.two_level_form = static_cast<int>(c.two_level_form);
  d.jhat_sign = c.jhat_sign == JhatSign::plus ? KKT_SIGN_PLUS : KKT_SIGN_MINUS;
  d.tol = c.gmres.tol;
  d.max_iters = c.gmres.max_iters;
  d.restart = c.gmres.restart ? *c.gmres.restart : KKT_NO_RESTART;
  d.happy_breakdown_tol = c.gmres.happy_breakdown_tol;
  return d;
}

// status -> the reference's exception types
[[noreturn]] inline void raise(int st, const std::string& what, int index) {
  switch (st) {
    case KKT_ECONFIG: throw ConfigError(what);
    case KKT_ESINGULAR: throw SingularMatrixError(what, index);
    case KKT_EDIVERGED: throw GmresDivergenceError(what, index);
    case KKT_EINVAL: throw std::invalid_argument(what);
    default: throw std::runtime_error(std::string(kkt_status_string(st)) + ": " + what);
  }
}

// One device context plus two reusable staging vectors for the host adapters.
class Device {
 public:
  Device(const ProblemConfig& cfg, Arithmetic mode) : config(cfg), mode(mode) {
    kkt_problem_desc d = to_desc(cfg);
    kkt_runtime_opts o{};
    o.mode = static_cast<int>(mode);
    o.device = -1;
    o.rank = 0;
    o.nranks = 1;
    const int st = kkt_ctx_create(&d, &o, &ctx_);
    if (st != KKT_OK) raise(st, kkt_create_error(), kkt_create_error_index());
  }
  ~Device() {
    if (ctx_) {
      for (auto& s : slot_) kkt_device_free(ctx_, s.p);
      kkt_ctx_destroy(ctx_);
    }
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  kkt_ctx* ctx() const { return ctx_; }
  void check(int st) const {
    if (st != KKT_OK) raise(st, kkt_last_error(ctx_), kkt_last_error_index(ctx_));
  }
  // staging vector `i` (0..2) with room for n doubles
  double* stage(int i, std::size_t n) {
    Slot& s = slot_[i];
    if (s.n < n) {
      check(kkt_device_free(ctx_, s.p));
      s.p = nullptr;
      check(kkt_device_alloc(ctx_, n, &s.p));
      s.n = n;
    }
    return s.p;
  }
  double* upload(int i, std::span<const double> v) {
    double* d = stage(i, v.size());
    check(kkt_copy_to_device(ctx_, d, v.data(), v.size()));
    return d;
  }
  void download(std::span<double> out, const double* d) { check(kkt_copy_to_host(ctx_, out.data(), d, out.size())); }

  ProblemConfig config;
  Arithmetic mode;

 private:
  struct Slot {
    double* p = nullptr;
    std::size_t n = 0;
  };
  kkt_ctx* ctx_ = nullptr;
  Slot slot_[3];
};

inline void need_size(std::size_t got, std::size_t want, const char* what) {
  if (got != want)
    throw std::invalid_argument(std::string(what) + ": length " + std::to_string(got) + ", expected " +
                                std::to_string(want));
}

}  // namespace detail

// --------------------------------------------------------- heat_operators.hpp
struct HeatOperators {
  explicit HeatOperators(const ProblemConfig& cfg, Arithmetic mode = Arithmetic::fast)
      : config(cfg), layout(make_layout(cfg)), dt(cfg.dt()), mass_scale(cfg.mass_scale()), shift(cfg.sigma()),
        dev(std::make_shared<detail::Device>(cfg, mode)) {}

  ProblemConfig config;
  SpaceTimeLayout layout;
  double dt;
  double mass_scale;
  double shift;  // sigma = sign * omega^{-1/2}
  std::shared_ptr<detail::Device> dev;

  kkt_ctx* ctx() const { return dev->ctx(); }
  Arithmetic mode() const { return dev->mode; }
  /// Entries of A and Ahat (the reference exposes them as BandedMatrix::at):
  /// assemble_spatial_operator (heat_operators.cpp:24-44) and make_ahat (:16-20).
  double A_at(int p, int q) const { return entry(p, q, 0.0); }
  double Ahat_at(int p, int q) const { return entry(p, q, shift * dt); }

 private:
  double entry(int p, int q, double sub) const {
    const int nx = layout.nx_int;
    const double cx = dt * config.nu / (config.dx() * config.dx());
    const double cy = dt * config.nu / (config.dy() * config.dy());
    if (p == q) return 1.0 + 2.0 * cx + 2.0 * cy - sub;
    if ((q == p + 1 || q == p - 1) && p / nx == q / nx) return -cx;
    if (q == p + nx || q == p - nx) return -cy;
    return 0.0;
  }
};

namespace detail {
using BlockOp = int (*)(kkt_ctx*, const double*, double*);
inline void block_op(const HeatOperators& ops, BlockOp f, std::span<const double> in, std::span<double> out,
                     std::size_t n, const char* what) {
  need_size(in.size(), n, what);
  need_size(out.size(), n, what);
  Device& d = *ops.dev;
  const double* din = d.upload(0, in);
  double* dout = d.stage(1, n);
  d.check(f(d.ctx(), din, dout));
  d.download(out, dout);
}
}  // namespace detail

#define KKTDD_GPU_BLOCK_OP(name)                                                                         \
  inline void name(const HeatOperators& ops, std::span<const double> in, std::span<double> out) {        \
    detail::block_op(ops, &kkt_##name, in, out, ops.layout.size(), #name);                               \
  }
KKTDD_GPU_BLOCK_OP(apply_J)
KKTDD_GPU_BLOCK_OP(apply_JT)
KKTDD_GPU_BLOCK_OP(apply_L)
KKTDD_GPU_BLOCK_OP(apply_LT)
KKTDD_GPU_BLOCK_OP(apply_Mu)
KKTDD_GPU_BLOCK_OP(apply_Mu_inv)
KKTDD_GPU_BLOCK_OP(apply_Mz)
KKTDD_GPU_BLOCK_OP(apply_Jhat)
KKTDD_GPU_BLOCK_OP(apply_JhatT)
KKTDD_GPU_BLOCK_OP(apply_shat)  // schur.hpp:22-23
#undef KKTDD_GPU_BLOCK_OP

namespace detail {
inline void window(const HeatOperators& ops, std::span<double> w, bool adjoint) {
  const std::size_t nsp = ops.layout.n_sp();
  if (nsp == 0 || w.size() % nsp != 0) throw std::invalid_argument("window length is not a multiple of n_sp");
  Device& d = *ops.dev;
  double* dw = d.upload(0, w);
  const int len = static_cast<int>(w.size() / nsp);
  d.check(adjoint ? kkt_adjoint_solve_window(d.ctx(), dw, len) : kkt_forward_solve_window(d.ctx(), dw, len));
  d.download(w, dw);
}
}  // namespace detail
inline void forward_solve_window(const HeatOperators& ops, std::span<double> window) { detail::window(ops, window, false); }
inline void adjoint_solve_window(const HeatOperators& ops, std::span<double> window) { detail::window(ops, window, true); }

// -------------------------------------------------------------------- kkt.hpp
struct KKTVector {
  std::size_t block = 0;
  std::vector<double> data;
  explicit KKTVector(std::size_t block_size = 0) : block(block_size), data(3 * block_size, 0.0) {}
  std::span<double> u() { return {data.data(), block}; }
  std::span<double> z() { return {data.data() + block, block}; }
  std::span<double> w() { return {data.data() + 2 * block, block}; }
  std::span<const double> u() const { return {data.data(), block}; }
  std::span<const double> z() const { return {data.data() + block, block}; }
  std::span<const double> w() const { return {data.data() + 2 * block, block}; }
};

struct RhsBundle {
  SpaceTimeVector f_u, f_z, f;
  KKTVector to_kkt() const {
    KKTVector b(f_u.size());
    std::copy(f_u.begin(), f_u.end(), b.u().begin());
    std::copy(f_z.begin(), f_z.end(), b.z().begin());
    std::copy(f.begin(), f.end(), b.w().begin());
    return b;
  }
};

using SpatialFn = std::function<double(double, double)>;
using SpaceTimeFn = std::function<double(double, double, double)>;

// Host-side sampling, the input boundary (kkt.cpp:29-48): f_u^n = ms * target, f_z = 0, f^1 = u0.
inline RhsBundle assemble_rhs(const HeatOperators& ops, const SpatialFn& u0, const SpaceTimeFn& target) {
  const SpaceTimeLayout& L = ops.layout;
  RhsBundle r{L.zeros(), L.zeros(), L.zeros()};
  const double dx = ops.config.dx(), dy = ops.config.dy();
  for (int n = 1; n <= L.nt; ++n) {
    const double t = n * ops.dt;
    for (int j = 1; j <= L.ny_int; ++j)
      for (int i = 1; i <= L.nx_int; ++i) {
        const double x = i * dx, y = j * dy;
        const std::size_t k = L.index(n, i, j);
        r.f_u[k] = ops.mass_scale * target(x, y, t);
        if (n == 1) r.f[k] = u0(x, y);
      }
  }
  return r;
}

inline void apply_K(const HeatOperators& ops, std::span<const double> v, std::span<double> out) {
  detail::block_op(ops, &kkt_apply_K, v, out, 3 * ops.layout.size(), "apply_K");
}
inline void apply_K(const HeatOperators& ops, const KKTVector& v, KKTVector& out) { apply_K(ops, v.data, out.data); }

// ------------------------------------------------------------------ schur.hpp
inline SpaceTimeVector apply_rasq(const HeatOperators& ops, const TimePartition& part, const SpaceTimeVector& r) {
  if (part.nt != ops.config.Nt || part.nd != ops.config.Nd)
    throw std::invalid_argument("apply_rasq: the partition differs from the operators' Nt / Nd");
  SpaceTimeVector out(ops.layout.size());
  detail::block_op(ops, &kkt_apply_rasq, r, out, ops.layout.size(), "apply_rasq");
  return out;
}

namespace detail {
// A context whose preconditioner is the requested one: the operators' own
// context when it matches, else a second one built for the changed config.
inline std::shared_ptr<Device> context_for(const HeatOperators& ops, PrecondKind kind, CoarseVariant variant,
                                           TwoLevelForm form) {
  const ProblemConfig& c = ops.config;
  const bool same = c.precond == kind &&
                    (kind != PrecondKind::two_level || (c.coarse_variant == variant && c.two_level_form == form));
  if (same) return ops.dev;
  ProblemConfig cfg = c;
  cfg.precond = kind;
  cfg.coarse_variant = variant;
  cfg.two_level_form = form;
  return std::make_shared<Device>(cfg, ops.dev->mode);
}
}  // namespace detail

class CoarseSpace {
 public:
  CoarseVariant variant() const { return variant_; }
  int dim() const { return dim_; }
  void restrict_to_coarse(const SpaceTimeLayout& layout, const TimePartition&, std::span<const double> r,
                          std::span<double> c) const {
    detail::need_size(r.size(), layout.size(), "restrict_to_coarse r");
    detail::need_size(c.size(), static_cast<std::size_t>(dim_), "restrict_to_coarse c");
    double* dr = dev_->upload(0, r);
    double* dc = dev_->stage(1, c.size());
    dev_->check(kkt_coarse_restrict(dev_->ctx(), dr, dc));
    dev_->download(c, dc);
  }
  void prolong_add(const SpaceTimeLayout& layout, const TimePartition&, std::span<const double> c,
                   std::span<double> out) const {
    detail::need_size(out.size(), layout.size(), "prolong_add out");
    detail::need_size(c.size(), static_cast<std::size_t>(dim_), "prolong_add c");
    double* dc = dev_->upload(0, c);
    double* dout = dev_->upload(1, out);
    dev_->check(kkt_coarse_prolong_add(dev_->ctx(), dc, dout));
    dev_->download(out, dout);
  }
  void solve_in_place(std::span<double> c) const {
    detail::need_size(c.size(), static_cast<std::size_t>(dim_), "solve_in_place c");
    double* dc = dev_->upload(0, c);
    dev_->check(kkt_coarse_solve(dev_->ctx(), dc));
    dev_->download(c, dc);
  }
  /// Row-major dim x dim (the reference returns a DenseMatrix).
  std::vector<double> coarse_matrix_dense() const {
    std::vector<double> m(static_cast<std::size_t>(dim_) * dim_);
    dev_->check(kkt_coarse_matrix(dev_->ctx(), m.data()));
    return m;
  }
  const std::shared_ptr<detail::Device>& device() const { return dev_; }

 private:
  friend CoarseSpace build_coarse_space(const HeatOperators&, const TimePartition&, CoarseVariant);
  CoarseSpace() = default;
  CoarseVariant variant_ = CoarseVariant::scalar;
  int dim_ = 0;
  std::shared_ptr<detail::Device> dev_;
};

inline CoarseSpace build_coarse_space(const HeatOperators& ops, const TimePartition&, CoarseVariant variant) {
  CoarseSpace cs;
  cs.variant_ = variant;
  cs.dev_ = detail::context_for(ops, PrecondKind::two_level, variant, ops.config.two_level_form);
  int32_t d = 0;
  cs.dev_->check(kkt_coarse_dim(cs.dev_->ctx(), &d));
  cs.dim_ = d;
  return cs;
}

inline SpaceTimeVector apply_two_level(const HeatOperators& ops, const TimePartition&, const CoarseSpace& coarse,
                                       const SpaceTimeVector& r, TwoLevelForm form) {
  detail::need_size(r.size(), ops.layout.size(), "apply_two_level r");
  detail::Device& d = *coarse.device();
  SpaceTimeVector out(r.size());
  const double* dr = d.upload(0, r);
  double* dout = d.stage(1, r.size());
  d.check(kkt_apply_two_level(d.ctx(), dr, dout, static_cast<int>(form)));
  d.download(out, dout);
  return out;
}

class SchurSolver {
 public:
  enum class Kind { identity, one_level, two_level };

  static SchurSolver make_identity(const HeatOperators& ops) {
    return SchurSolver(Kind::identity, detail::context_for(ops, PrecondKind::none, ops.config.coarse_variant,
                                                           ops.config.two_level_form));
  }
  static SchurSolver make_one_level(const HeatOperators& ops, const TimePartition&) {
    return SchurSolver(Kind::one_level, detail::context_for(ops, PrecondKind::one_level, ops.config.coarse_variant,
                                                            ops.config.two_level_form));
  }
  static SchurSolver make_two_level(const HeatOperators& ops, const TimePartition&, CoarseVariant variant,
                                    TwoLevelForm form) {
    return SchurSolver(Kind::two_level, detail::context_for(ops, PrecondKind::two_level, variant, form));
  }
  Kind kind() const { return kind_; }
  void apply(std::span<const double> r, std::span<double> out) const {
    const std::size_t n = dev_->config.Nt * static_cast<std::size_t>(dev_->config.n_sp());
    detail::need_size(r.size(), n, "SchurSolver::apply r");
    detail::need_size(out.size(), n, "SchurSolver::apply out");
    const double* dr = dev_->upload(0, r);
    double* dout = dev_->stage(1, n);
    dev_->check(kkt_schur_apply(dev_->ctx(), dr, dout));
    dev_->download(out, dout);
  }
  const std::shared_ptr<detail::Device>& device() const { return dev_; }

 private:
  SchurSolver(Kind k, std::shared_ptr<detail::Device> d) : kind_(k), dev_(std::move(d)) {}
  Kind kind_;
  std::shared_ptr<detail::Device> dev_;
};

inline SchurSolver make_schur_solver(const HeatOperators& ops, const TimePartition& part, const ProblemConfig& cfg) {
  switch (cfg.precond) {
    case PrecondKind::none: return SchurSolver::make_identity(ops);
    case PrecondKind::one_level: return SchurSolver::make_one_level(ops, part);
    case PrecondKind::two_level:
      return SchurSolver::make_two_level(ops, part, cfg.coarse_variant, cfg.two_level_form);
    default:
      throw ConfigError("dense-schur / true-schur are desk-scale dense oracles (schur.cpp:13-21), not on the device path");
  }
}

// ------------------------------------------------------- kkt.hpp (continued)
inline void apply_P_inv(const HeatOperators& ops, const SchurSolver& schur, std::span<const double> r,
                        std::span<double> out) {
  const std::size_t n = 3 * ops.layout.size();
  detail::need_size(r.size(), n, "apply_P_inv r");
  detail::need_size(out.size(), n, "apply_P_inv out");
  detail::Device& d = *schur.device();
  const double* dr = d.upload(0, r);
  double* dout = d.stage(1, n);
  d.check(kkt_apply_P_inv(d.ctx(), dr, dout));
  d.download(out, dout);
}
inline void apply_P_inv(const HeatOperators& ops, const SchurSolver& schur, const KKTVector& r, KKTVector& out) {
  apply_P_inv(ops, schur, r.data, out.data);
}

inline double kkt_residual(const HeatOperators& ops, const KKTVector& v, const RhsBundle& rhs) {
  const KKTVector b = rhs.to_kkt();
  detail::need_size(v.data.size(), b.data.size(), "kkt_residual v");
  detail::Device& d = *ops.dev;
  const double* dv = d.upload(0, v.data);
  const double* db = d.upload(1, b.data);
  double rel = 0.0;
  d.check(::kkt_residual(d.ctx(), dv, db, &rel));
  return rel;
}

inline double evaluate_objective(const HeatOperators& ops, std::span<const double> u, std::span<const double> z,
                                 const SpaceTimeFn& target) {
  const SpaceTimeLayout& L = ops.layout;
  detail::need_size(u.size(), L.size(), "evaluate_objective u");
  detail::need_size(z.size(), L.size(), "evaluate_objective z");
  SpaceTimeVector t(L.size());
  const double dx = ops.config.dx(), dy = ops.config.dy();
  for (int n = 1; n <= L.nt; ++n)
    for (int j = 1; j <= L.ny_int; ++j)
      for (int i = 1; i <= L.nx_int; ++i) t[L.index(n, i, j)] = target(i * dx, j * dy, n * ops.dt);
  detail::Device& d = *ops.dev;
  const double* du = d.upload(0, u);
  const double* dz = d.upload(1, z);
  const double* dtg = d.upload(2, t);
  double obj = 0.0;
  d.check(kkt_evaluate_objective(d.ctx(), du, dz, dtg, &obj));
  return obj;
}

// ------------------------------------------------------------------ gmres.hpp
struct GmresResult {
  std::vector<double> solution;
  bool converged = false;
  int iterations = 0;
  std::vector<double> residual_history;
  double true_final_relres = 0.0;
};

/// Right-preconditioned GMRES on the device with apply_K and apply_P_inv(schur)
/// as its maps (run_single's wiring, experiments.cpp:46-57); the parameters are
/// the GmresParams of the configuration the solver's context was built with.
/// b is a host [u; z; w] vector; the solution comes back to the host.
inline GmresResult gmres_solve(const HeatOperators& ops, const SchurSolver& schur, std::span<const double> b) {
  detail::need_size(b.size(), 3 * ops.layout.size(), "gmres_solve b");
  detail::Device& d = *schur.device();
  GmresResult r;
  r.solution.resize(b.size());
  std::vector<double> hist(static_cast<std::size_t>(d.config.gmres.max_iters));
  kkt_gmres_result res{};
  d.check(kkt_gmres_solve_host(d.ctx(), b.data(), r.solution.data(), &res, hist.data(), static_cast<int>(hist.size())));
  r.converged = res.converged != 0;
  r.iterations = res.iterations;
  r.true_final_relres = res.true_final_relres;
  r.residual_history.assign(hist.begin(), hist.begin() + res.history_len);
  return r;
}

// ---------------------------------------------------------- model_problem.hpp
inline double model_initial_condition(double x, double y) { return -x * y * (x - 1.0) * (y - 2.0); }
inline double model_target(double x, double y, double t) {
  constexpr double two_pi = 2.0 * std::numbers::pi;
  return std::sin(two_pi * t) * std::sin(two_pi * x) * std::sin(two_pi * y);
}

// ------------------------------------------------------------ experiments.hpp
struct RunRecord {
  ProblemConfig config;
  int iterations = 0;
  bool converged = false;
  double true_final_relres = 0.0;
  double objective = 0.0;
  double setup_seconds = 0.0;
  double solve_seconds = 0.0;
};

/// run_single (experiments.cpp:33-69) entirely behind the C-ABI: setup, the
/// model right-hand side, the solve and the objective run in kkt_run_single.
inline RunRecord run_single(const ProblemConfig& cfg, GmresResult* out_result = nullptr,
                            Arithmetic mode = Arithmetic::fast) {
  kkt_problem_desc d = detail::to_desc(cfg);
  kkt_runtime_opts o{};
  o.mode = static_cast<int>(mode);
  o.device = -1;
  o.nranks = 1;
  kkt_run_record rec{};
  std::vector<double> x;
  if (out_result) x.resize(3 * static_cast<std::size_t>(cfg.Nt) * cfg.n_sp());
  const int st = kkt_run_single(&d, &o, &rec, out_result ? x.data() : nullptr);
  if (st != KKT_OK) detail::raise(st, kkt_create_error(), kkt_create_error_index());
  RunRecord r;
  r.config = cfg;
  r.iterations = rec.iterations;
  r.converged = rec.converged != 0;
  r.true_final_relres = rec.true_final_relres;
  r.objective = rec.objective;
  r.setup_seconds = rec.setup_seconds;
  r.solve_seconds = rec.solve_seconds;
  if (out_result) {
    out_result->solution = std::move(x);
    out_result->converged = r.converged;
    out_result->iterations = r.iterations;
    out_result->true_final_relres = r.true_final_relres;
  }
  return r;
}

}  // namespace kktdd_gpu
