// test_reference_cases.cpp — a subset of the reference's own unit tests
// (/root/reference/proj/tests/test_{heat_operators,kkt,schur,gmres,experiments}.cpp),
// restated against the reference-side binding include/kktdd_gpu.hpp, so they run
// through the C++ shim -> C-ABI -> libkktdd_b200.so on the device.  Each case
// keeps the reference test's name, sizes, seeds' role and tolerance and cites
// the case it restates.  Cases that need the reference's std::function GMRES or
// its dense-oracle Schur kinds are restated with the device GMRES / a dense
// matrix assembled from unit vectors, as the reference's own dense_from_operator
// does (schur.cpp:57-69).
//
// Built by tests/cpp/Makefile (g++ -std=c++20, links libkktdd_b200.so); run by
// tests/test_gpu_cpp_shim.py under `-m gpu`.  KKTDD_ARITH=strict selects the
// bitwise mode.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <random>

#include "kktdd_gpu.hpp"

using namespace kktdd_gpu;

namespace {

using Mat = std::vector<std::vector<double>>;

Arithmetic arith() {
  const char* e = std::getenv("KKTDD_ARITH");
  return e && std::string(e) == "strict" ? Arithmetic::strict : Arithmetic::fast;
}

// ---- a small independent dense oracle (the role of tests/oracles.hpp)
Mat zeros(int r, int c) { return Mat(r, std::vector<double>(c, 0.0)); }
std::vector<double> matvec(const Mat& m, const std::vector<double>& v) {
  std::vector<double> y(m.size(), 0.0);
  for (std::size_t i = 0; i < m.size(); ++i)
    for (std::size_t j = 0; j < v.size(); ++j) y[i] += m[i][j] * v[j];
  return y;
}
Mat transpose(const Mat& a) {
  Mat t = zeros(int(a[0].size()), int(a.size()));
  for (std::size_t i = 0; i < a.size(); ++i)
    for (std::size_t j = 0; j < a[0].size(); ++j) t[j][i] = a[i][j];
  return t;
}
Mat matmul(const Mat& a, const Mat& b) {
  Mat c = zeros(int(a.size()), int(b[0].size()));
  for (std::size_t i = 0; i < a.size(); ++i)
    for (std::size_t k = 0; k < b.size(); ++k)
      for (std::size_t j = 0; j < b[0].size(); ++j) c[i][j] += a[i][k] * b[k][j];
  return c;
}
// Gaussian elimination with partial pivoting on [A | B]
Mat solve_many(Mat a, Mat b) {
  const int n = int(a.size()), m = int(b[0].size());
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[i][k]) > std::abs(a[p][k])) p = i;
    std::swap(a[k], a[p]);
    std::swap(b[k], b[p]);
    for (int i = k + 1; i < n; ++i) {
      const double f = a[i][k] / a[k][k];
      if (f == 0.0) continue;
      for (int j = k; j < n; ++j) a[i][j] -= f * a[k][j];
      for (int j = 0; j < m; ++j) b[i][j] -= f * b[k][j];
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < m; ++j) {
      double acc = b[k][j];
      for (int i = k + 1; i < n; ++i) acc -= a[k][i] * b[i][j];
      b[k][j] = acc / a[k][k];
    }
  return b;
}
std::vector<double> gauss_solve(const Mat& a, const std::vector<double>& rhs) {
  Mat b = zeros(int(rhs.size()), 1);
  for (std::size_t i = 0; i < rhs.size(); ++i) b[i][0] = rhs[i];
  Mat x = solve_many(a, b);
  std::vector<double> out(rhs.size());
  for (std::size_t i = 0; i < rhs.size(); ++i) out[i] = x[i][0];
  return out;
}
Mat inverse(const Mat& a) {
  Mat e = zeros(int(a.size()), int(a.size()));
  for (std::size_t i = 0; i < a.size(); ++i) e[i][i] = 1.0;
  return solve_many(a, e);
}
double rel_err(const std::vector<double>& got, const std::vector<double>& want) {
  double d = 0.0, n = 0.0;
  for (std::size_t i = 0; i < got.size(); ++i) {
    d += (got[i] - want[i]) * (got[i] - want[i]);
    n += want[i] * want[i];
  }
  return n > 0.0 ? std::sqrt(d / n) : std::sqrt(d);
}
std::vector<double> random_vector(std::size_t n, std::mt19937& rng) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> v(n);
  for (double& x : v) x = u(rng);
  return v;
}
double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double norm2(const std::vector<double>& a) { return std::sqrt(dot(a, a)); }

ProblemConfig desk_config(int nt, int nd, int nx, int ny, double omega = 1e-2) {
  ProblemConfig cfg;  // reference defaults: Lx = 1, Ly = 2, T = 1, nu = 1, two-level per-dof
  cfg.Nt = nt;
  cfg.Nd = nd;
  cfg.Nx = nx;
  cfg.Ny = ny;
  cfg.omega = omega;
  return cfg;
}

// dense matrix of a block operator from unit vectors (schur.cpp:57-69)
template <class F>
Mat dense_from_operator(int n, F&& op) {
  Mat m = zeros(n, n);
  std::vector<double> e(n, 0.0), col(n);
  for (int j = 0; j < n; ++j) {
    e[j] = 1.0;
    op(e, col);
    for (int i = 0; i < n; ++i) m[i][j] = col[i];
    e[j] = 0.0;
  }
  return m;
}

}  // namespace

// ------------------------------------------------ test_heat_operators.cpp
TEST_CASE("single interior unknown evaluates the stencil coefficients") {  // :34-41
  ProblemConfig cfg = desk_config(3, 1, 2, 2);
  cfg.T = 0.3;  // dt = 0.1, dx = 0.5, dy = 1: A = [1 + 2*0.4 + 2*0.1] = [2]
  cfg.precond = PrecondKind::none;
  HeatOperators ops(cfg, arith());
  REQUIRE(ops.layout.n_sp() == 1);
  CHECK(ops.A_at(0, 0) == doctest::Approx(2.0).epsilon(1e-15));
  std::vector<double> u = {1.5, -2.0, 0.25}, out(3);
  apply_J(ops, u, out);
  CHECK(out[0] == doctest::Approx(2.0 * 1.5).epsilon(1e-15));
  CHECK(out[1] == doctest::Approx(2.0 * -2.0 - 1.5).epsilon(1e-15));
  CHECK(out[2] == doctest::Approx(2.0 * 0.25 + 2.0).epsilon(1e-15));
}

TEST_CASE("adjoint pairing for J, L, Jhat") {  // :84-110
  std::mt19937 rng(31);
  HeatOperators ops(desk_config(5, 1, 4, 3, 1e-3), arith());
  const std::size_t n = ops.layout.size();
  for (int trial = 0; trial < 20; ++trial) {
    auto x = random_vector(n, rng);
    auto y = random_vector(n, rng);
    std::vector<double> ax(n), aty(n);
    apply_J(ops, x, ax);
    apply_JT(ops, y, aty);
    double lhs = dot(ax, y), rhs = dot(x, aty);
    CHECK(std::abs(lhs - rhs) <= 1e-13 * (std::abs(lhs) + std::abs(rhs) + 1.0));
    apply_L(ops, x, ax);
    apply_LT(ops, y, aty);
    lhs = dot(ax, y);
    rhs = dot(x, aty);
    CHECK(std::abs(lhs - rhs) <= 1e-13 * (std::abs(lhs) + std::abs(rhs) + 1.0));
    apply_Jhat(ops, x, ax);
    apply_JhatT(ops, y, aty);
    lhs = dot(ax, y);
    rhs = dot(x, aty);
    CHECK(std::abs(lhs - rhs) <= 1e-13 * (std::abs(lhs) + std::abs(rhs) + 1.0));
  }
}

TEST_CASE("Jhat equals J plus the scaled control coupling") {  // :112-129
  std::mt19937 rng(8);
  for (JhatSign sign : {JhatSign::plus, JhatSign::minus}) {
    ProblemConfig cfg = desk_config(4, 1, 3, 4, 1e-3);
    cfg.jhat_sign = sign;
    HeatOperators ops(cfg, arith());
    const std::size_t n = ops.layout.size();
    auto x = random_vector(n, rng);
    std::vector<double> jh(n), j(n), l(n);
    apply_Jhat(ops, x, jh);
    apply_J(ops, x, j);
    apply_L(ops, x, l);
    for (std::size_t k = 0; k < n; ++k) CHECK(jh[k] == doctest::Approx(j[k] + ops.shift * l[k]).epsilon(1e-14));
  }
}

TEST_CASE("forward window solve: zero input, and the round trip through Jhat") {  // :140-167
  HeatOperators ops(desk_config(4, 1, 3, 3, 1e-2), arith());
  const int nsp = ops.layout.n_sp();
  std::vector<double> z(3 * nsp, 0.0);
  forward_solve_window(ops, z);
  for (double v : z) CHECK(v == 0.0);
  std::mt19937 rng(13);
  auto b = random_vector(ops.layout.size(), rng);
  auto x = b;
  forward_solve_window(ops, x);
  std::vector<double> back(x.size());
  apply_Jhat(ops, x, back);
  CHECK(rel_err(back, b) <= 1e-10);
}

TEST_CASE("forward and adjoint window solves are mutual adjoints") {  // :169-183
  std::mt19937 rng(17);
  HeatOperators ops(desk_config(5, 1, 3, 4, 1e-2), arith());
  const std::size_t n = ops.layout.size();
  for (int trial = 0; trial < 10; ++trial) {
    auto a = random_vector(n, rng);
    auto b = random_vector(n, rng);
    auto fa = a, gb = b;
    forward_solve_window(ops, fa);
    adjoint_solve_window(ops, gb);
    const double lhs = dot(fa, b), rhs = dot(a, gb);
    CHECK(std::abs(lhs - rhs) <= 1e-12 * (std::abs(lhs) + std::abs(rhs) + 1.0));
  }
}

TEST_CASE("adjoint window solve matches the dense transpose solve") {  // :185-200
  HeatOperators ops(desk_config(3, 1, 3, 3, 1e-2), arith());
  const int nsp = ops.layout.n_sp(), N = int(ops.layout.size());
  Mat jm = zeros(N, N);  // Jhat: block lower bidiagonal, diag Ahat, subdiag -I
  for (int k = 0; k < ops.layout.nt; ++k)
    for (int p = 0; p < nsp; ++p) {
      for (int q = 0; q < nsp; ++q) jm[k * nsp + p][k * nsp + q] = ops.Ahat_at(p, q);
      if (k > 0) jm[k * nsp + p][(k - 1) * nsp + p] = -1.0;
    }
  std::mt19937 rng(5);
  auto b = random_vector(N, rng);
  auto got = b;
  adjoint_solve_window(ops, got);
  CHECK(rel_err(got, gauss_solve(transpose(jm), b)) <= 1e-10);
  got = b;
  forward_solve_window(ops, got);  // :202-218
  CHECK(rel_err(got, gauss_solve(jm, b)) <= 1e-10);
}

TEST_CASE("singular Ahat from the literal shift is reported") {  // :220-232
  ProblemConfig cfg = desk_config(10, 1, 2, 2, 0.0025);
  cfg.jhat_sign = JhatSign::plus;
  CHECK_THROWS_AS(HeatOperators(cfg, arith()), SingularMatrixError);
  try {
    HeatOperators ops(cfg, arith());
  } catch (const SingularMatrixError& e) {
    CHECK(e.pivot_index == 0);  // test_linalg.cpp:97-108 pins the index payload
  }
}

TEST_CASE("layout mismatches are shape errors") {  // :234-240
  HeatOperators ops(desk_config(3, 1, 3, 3), arith());
  std::vector<double> shortv(ops.layout.size() - 1), out(ops.layout.size());
  CHECK_THROWS_AS(apply_J(ops, shortv, out), std::invalid_argument);
  std::vector<double> bad(ops.layout.n_sp() + 1);
  CHECK_THROWS_AS(forward_solve_window(ops, bad), std::invalid_argument);
}

TEST_CASE("invalid configurations raise ConfigError") {  // config.cpp:5-22, test_experiments.cpp
  ProblemConfig cfg = desk_config(7, 3, 3, 3);  // 7 % 3 != 0
  CHECK_THROWS_AS(HeatOperators(cfg, arith()), ConfigError);
  cfg = desk_config(6, 3, 3, 3);
  cfg.gmres.restart = 0;  // config.cpp:21
  CHECK_THROWS_AS(HeatOperators(cfg, arith()), ConfigError);
  CHECK_THROWS_AS(build_time_partition(7, 3), ConfigError);
}

// ------------------------------------------------------------ test_kkt.cpp
TEST_CASE("K is symmetric in the inner-product pairing") {  // :136-149
  std::mt19937 rng(3);
  HeatOperators ops(desk_config(4, 1, 3, 4, 1e-3), arith());
  const std::size_t n3 = 3 * ops.layout.size();
  for (int trial = 0; trial < 10; ++trial) {
    auto x = random_vector(n3, rng);
    auto y = random_vector(n3, rng);
    std::vector<double> kx(n3), ky(n3);
    apply_K(ops, x, kx);
    apply_K(ops, y, ky);
    const double lhs = dot(kx, y), rhs = dot(x, ky);
    CHECK(std::abs(lhs - rhs) <= 1e-12 * (std::abs(lhs) + std::abs(rhs) + 1.0));
  }
}

TEST_CASE("apply_K matches the dense assembly at desk scale") {  // :151-162, dense K as :29-63
  std::mt19937 rng(19);
  HeatOperators ops(desk_config(4, 1, 3, 3, 1e-2), arith());
  REQUIRE(ops.layout.n_sp() == 4);
  const int nb = int(ops.layout.size()), nsp = ops.layout.n_sp();
  const double ms = ops.mass_scale, omega = ops.config.omega, dt = ops.dt;
  Mat K = zeros(3 * nb, 3 * nb);
  for (int k = 0; k < nb; ++k) {
    K[k][k] = ms;
    K[nb + k][nb + k] = omega * ms;
  }
  for (int n = 1; n <= ops.layout.nt; ++n)
    for (int p = 0; p < nsp; ++p) {
      const int row = 2 * nb + int(ops.layout.index(n, p));
      for (int q = 0; q < nsp; ++q) {
        const double a = ops.A_at(p, q);
        if (a != 0.0) {
          const int col = int(ops.layout.index(n, q));
          K[row][col] += a;
          K[col][row] += a;
        }
      }
      if (n > 1) {
        const int col = int(ops.layout.index(n - 1, p));
        K[row][col] -= 1.0;
        K[col][row] -= 1.0;
      }
      const int zcol = nb + int(ops.layout.index(n, p));
      K[row][zcol] -= dt;
      K[zcol][row] -= dt;
    }
  auto v = random_vector(3 * nb, rng);
  std::vector<double> got(3 * nb);
  apply_K(ops, v, got);
  CHECK(rel_err(got, matvec(K, v)) <= 1e-12);
}

TEST_CASE("preconditioner diagonal blocks scale as expected") {  // :164-182
  HeatOperators ops(desk_config(3, 1, 3, 3, 1e-3), arith());
  const auto part = build_time_partition(3, 1);
  const auto schur = SchurSolver::make_one_level(ops, part);
  std::mt19937 rng(8);
  KKTVector r(ops.layout.size()), out(ops.layout.size());
  auto ru = random_vector(ops.layout.size(), rng);
  auto rz = random_vector(ops.layout.size(), rng);
  std::copy(ru.begin(), ru.end(), r.u().begin());
  std::copy(rz.begin(), rz.end(), r.z().begin());
  apply_P_inv(ops, schur, r, out);
  for (std::size_t k = 0; k < ops.layout.size(); ++k) {
    CHECK(out.u()[k] == doctest::Approx(ru[k] / ops.mass_scale).epsilon(1e-14));
    CHECK(out.z()[k] == doctest::Approx(rz[k] / (ops.config.omega * ops.mass_scale)).epsilon(1e-14));
    CHECK(out.w()[k] == 0.0);
  }
}

TEST_CASE("constraint residual of a converged solve stays within the slack") {  // :316-345
  ProblemConfig cfg = desk_config(6, 2, 3, 3, 1e-3);
  HeatOperators ops(cfg, arith());
  const auto part = build_time_partition(cfg.Nt, cfg.Nd);
  const auto schur = SchurSolver::make_two_level(ops, part, CoarseVariant::per_dof, TwoLevelForm::multiplicative);
  auto rhs = assemble_rhs(ops, model_initial_condition, model_target);
  auto b = rhs.to_kkt();
  auto res = gmres_solve(ops, schur, b.data);  // GmresParams{}: tol 1e-6
  REQUIRE(res.converged);
  const std::size_t nb = ops.layout.size();
  const std::span<const double> sol(res.solution);
  std::vector<double> cons(nb), lz(nb);
  apply_J(ops, sol.subspan(0, nb), cons);
  apply_L(ops, sol.subspan(nb, nb), lz);
  double rn = 0.0;
  for (std::size_t k = 0; k < nb; ++k) {
    const double d = cons[k] + lz[k] - rhs.f[k];
    rn += d * d;
  }
  CHECK(std::sqrt(rn) / norm2(rhs.f) <= 10.0 * cfg.gmres.tol);
  // kkt_residual (:277-314) of the same solve
  KKTVector x(nb);
  x.data = res.solution;
  CHECK(kkt_residual(ops, x, rhs) == doctest::Approx(res.true_final_relres).epsilon(1e-9));
}

TEST_CASE("objective of the solved problem does not exceed the zero-control objective") {  // :221-275, acceptance 10
  ProblemConfig cfg = desk_config(6, 2, 4, 4, 1e-3);
  cfg.gmres.tol = 1e-10;
  HeatOperators ops(cfg, arith());
  const auto part = build_time_partition(cfg.Nt, cfg.Nd);
  const auto schur = make_schur_solver(ops, part, cfg);
  auto rhs = assemble_rhs(ops, model_initial_condition, model_target);
  auto res = gmres_solve(ops, schur, rhs.to_kkt().data);
  REQUIRE(res.converged);
  const std::size_t nb = ops.layout.size();
  const std::span<const double> sol(res.solution);
  const double obj = evaluate_objective(ops, sol.subspan(0, nb), sol.subspan(nb, nb), model_target);
  // zero control: integrate the constraint forward with z = 0 (window solve with A needs sigma = 0;
  // use the dense route instead)
  const int nsp = ops.layout.n_sp();
  Mat A = zeros(nsp, nsp);
  for (int p = 0; p < nsp; ++p)
    for (int q = 0; q < nsp; ++q) A[p][q] = ops.A_at(p, q);
  std::vector<double> u0(nb, 0.0), prev(nsp, 0.0), zero(nb, 0.0);
  for (int n = 1; n <= ops.layout.nt; ++n) {
    std::vector<double> step(nsp);
    for (int p = 0; p < nsp; ++p) step[p] = rhs.f[ops.layout.index(n, p)] + prev[p];
    prev = gauss_solve(A, step);
    std::copy(prev.begin(), prev.end(), u0.begin() + ops.layout.node_offset(n));
  }
  const double obj0 = evaluate_objective(ops, u0, zero, model_target);
  CHECK(obj > 0.0);
  CHECK(obj <= obj0 * (1.0 + 1e-9));
}

// ---------------------------------------------------------- test_schur.cpp
TEST_CASE("apply_rasq on zero input is zero") {  // :56-61
  HeatOperators ops(desk_config(6, 3, 3, 3), arith());
  auto part = build_time_partition(6, 3);
  auto out = apply_rasq(ops, part, ops.layout.zeros());
  for (double v : out) CHECK(v == 0.0);
}

TEST_CASE("single-subdomain sweep inverts Shat exactly") {  // :63-73
  HeatOperators ops(desk_config(6, 1, 4, 4, 1e-2), arith());
  REQUIRE(ops.layout.n_sp() == 9);
  auto part = build_time_partition(6, 1);
  std::mt19937 rng(2);
  auto r = random_vector(ops.layout.size(), rng);
  auto got = apply_rasq(ops, part, r);
  const Mat shat = dense_from_operator(int(ops.layout.size()), [&](const std::vector<double>& v, std::vector<double>& o) {
    apply_shat(ops, v, o);
  });
  CHECK(rel_err(got, gauss_solve(shat, r)) <= 1e-10);
}

TEST_CASE("apply_rasq equals the explicitly assembled windowed sweep") {  // :75-123
  HeatOperators ops(desk_config(9, 3, 3, 3, 1e-2), arith());
  REQUIRE(ops.layout.n_sp() == 4);
  auto part = build_time_partition(9, 3);
  const auto& layout = ops.layout;
  const int nsp = layout.n_sp(), N = int(layout.size());
  Mat total = zeros(N, N);
  for (int s = 0; s < part.nd; ++s) {
    const int wlen = part.extended[s].count();
    Mat wj = zeros(wlen * nsp, wlen * nsp);
    for (int k = 0; k < wlen; ++k)
      for (int p = 0; p < nsp; ++p) {
        for (int q = 0; q < nsp; ++q) wj[k * nsp + p][k * nsp + q] = ops.Ahat_at(p, q);
        if (k > 0) wj[k * nsp + p][(k - 1) * nsp + p] = -1.0;
      }
    const Mat wj_inv = inverse(wj);
    Mat inner = matmul(transpose(wj_inv), wj_inv);
    for (auto& row : inner)
      for (double& v : row) v *= ops.mass_scale;
    const auto wpos = [&](int n, int p) { return (n - part.extended[s].first) * nsp + p; };
    for (int n = part.nodes[s].first; n <= part.nodes[s].last; ++n) {
      if (part.owner[n] != s) continue;
      for (int n2 = part.nodes[s].first; n2 <= part.nodes[s].last; ++n2)
        for (int p = 0; p < nsp; ++p)
          for (int q = 0; q < nsp; ++q) total[layout.index(n, p)][layout.index(n2, q)] += inner[wpos(n, p)][wpos(n2, q)];
    }
  }
  std::mt19937 rng(77);
  for (int trial = 0; trial < 5; ++trial) {
    auto r = random_vector(N, rng);
    CHECK(rel_err(apply_rasq(ops, part, r), matvec(total, r)) <= 1e-12);
  }
}

TEST_CASE("apply_rasq is linear and deterministic") {  // :125-143
  HeatOperators ops(desk_config(8, 4, 3, 3, 1e-3), arith());
  auto part = build_time_partition(8, 4);
  std::mt19937 rng(11);
  auto a = random_vector(ops.layout.size(), rng);
  auto b = random_vector(ops.layout.size(), rng);
  const double alpha = 0.37, beta = -2.25;
  SpaceTimeVector combo(ops.layout.size());
  for (std::size_t k = 0; k < combo.size(); ++k) combo[k] = alpha * a[k] + beta * b[k];
  auto lhs = apply_rasq(ops, part, combo);
  auto ya = apply_rasq(ops, part, a);
  auto yb = apply_rasq(ops, part, b);
  std::vector<double> rhs(combo.size());
  for (std::size_t k = 0; k < rhs.size(); ++k) rhs[k] = alpha * ya[k] + beta * yb[k];
  CHECK(rel_err(lhs, rhs) <= 1e-12);
  auto again = apply_rasq(ops, part, a);
  CHECK(std::memcmp(again.data(), ya.data(), ya.size() * sizeof(double)) == 0);
}

TEST_CASE("coarse space: scalar variant is Galerkin and SPD at desk scale") {  // :221-299
  HeatOperators ops(desk_config(6, 2, 3, 3, 1e-2), arith());
  auto part = build_time_partition(6, 2);
  auto cs = build_coarse_space(ops, part, CoarseVariant::scalar);
  REQUIRE(cs.dim() == 4);  // constant + ramp per subdomain
  const auto S0 = cs.coarse_matrix_dense();
  const int d = cs.dim();
  // Galerkin: S0 = Z^T Shat Z, column by column through prolong_add / apply_shat / restrict
  for (int j = 0; j < d; ++j) {
    std::vector<double> e(d, 0.0), col(d);
    e[j] = 1.0;
    SpaceTimeVector z = ops.layout.zeros(), sz(ops.layout.size());
    cs.prolong_add(ops.layout, part, e, z);
    apply_shat(ops, z, sz);
    cs.restrict_to_coarse(ops.layout, part, sz, col);
    for (int i = 0; i < d; ++i) CHECK(std::abs(col[i] - S0[std::size_t(i) * d + j]) <= 1e-11 * std::abs(S0[std::size_t(j) * d + j]));
  }
  for (int i = 0; i < d; ++i) {
    CHECK(S0[std::size_t(i) * d + i] > 0.0);
    for (int j = 0; j < d; ++j) CHECK(std::abs(S0[std::size_t(i) * d + j] - S0[std::size_t(j) * d + i]) <= 1e-12 * S0[std::size_t(i) * d + i]);
  }
}

TEST_CASE("two-level application: zero stays zero in every form") {  // :301-313
  HeatOperators ops(desk_config(6, 2, 3, 3, 1e-2), arith());
  auto part = build_time_partition(6, 2);
  auto cs = build_coarse_space(ops, part, CoarseVariant::scalar);
  for (auto form : {TwoLevelForm::literal, TwoLevelForm::multiplicative, TwoLevelForm::additive}) {
    auto out = apply_two_level(ops, part, cs, ops.layout.zeros(), form);
    for (double v : out) CHECK(v == 0.0);
  }
}

TEST_CASE("two-level application: coarse-range residuals are solved by the coarse step alone") {  // :315-326
  HeatOperators ops(desk_config(6, 2, 3, 3, 1e-2), arith());
  auto part = build_time_partition(6, 2);
  auto cs = build_coarse_space(ops, part, CoarseVariant::scalar);
  std::mt19937 rng(21);
  std::vector<double> c = random_vector(cs.dim(), rng);
  SpaceTimeVector zc = ops.layout.zeros();
  cs.prolong_add(ops.layout, part, c, zc);
  SpaceTimeVector r(ops.layout.size());
  apply_shat(ops, zc, r);
  auto y = apply_two_level(ops, part, cs, r, TwoLevelForm::multiplicative);
  SpaceTimeVector sy(ops.layout.size());
  apply_shat(ops, y, sy);
  CHECK(rel_err(sy, r) <= 1e-10);
}

TEST_CASE("two-level application: additive form sums the two corrections") {  // :352-363
  HeatOperators ops(desk_config(6, 2, 3, 3, 1e-2), arith());
  auto part = build_time_partition(6, 2);
  auto cs = build_coarse_space(ops, part, CoarseVariant::scalar);
  std::mt19937 rng(31);
  auto r = random_vector(ops.layout.size(), rng);
  auto add = apply_two_level(ops, part, cs, r, TwoLevelForm::additive);
  auto fine = apply_rasq(ops, part, r);
  std::vector<double> c(cs.dim());
  cs.restrict_to_coarse(ops.layout, part, r, c);
  cs.solve_in_place(c);
  SpaceTimeVector want(fine);
  cs.prolong_add(ops.layout, part, c, want);
  CHECK(rel_err(add, want) <= 1e-13);
}

TEST_CASE("schur solver dispatch follows the configured kind") {  // :366-397
  ProblemConfig cfg = desk_config(6, 2, 3, 3, 1e-2);
  cfg.coarse_variant = CoarseVariant::scalar;
  HeatOperators ops(cfg, arith());
  auto part = build_time_partition(6, 2);
  std::mt19937 rng(9);
  auto r = random_vector(ops.layout.size(), rng);
  std::vector<double> out(r.size());
  cfg.precond = PrecondKind::none;
  auto id = make_schur_solver(ops, part, cfg);
  CHECK(id.kind() == SchurSolver::Kind::identity);
  id.apply(r, out);
  CHECK(out == r);
  cfg.precond = PrecondKind::one_level;
  auto one = make_schur_solver(ops, part, cfg);
  CHECK(one.kind() == SchurSolver::Kind::one_level);
  one.apply(r, out);
  CHECK(rel_err(out, apply_rasq(ops, part, r)) <= 1e-14);
  cfg.precond = PrecondKind::two_level;
  auto two = make_schur_solver(ops, part, cfg);
  CHECK(two.kind() == SchurSolver::Kind::two_level);
  two.apply(r, out);
  auto cs = build_coarse_space(ops, part, CoarseVariant::scalar);
  CHECK(rel_err(out, apply_two_level(ops, part, cs, r, TwoLevelForm::multiplicative)) <= 1e-14);
  cfg.precond = PrecondKind::dense_schur;
  CHECK_THROWS_AS(make_schur_solver(ops, part, cfg), ConfigError);
}

// ---------------------------------------------------------- test_gmres.cpp
TEST_CASE("residual history is nonincreasing and tracks the true residual") {  // :88-101
  ProblemConfig cfg = desk_config(8, 2, 4, 4, 1e-2);
  cfg.coarse_variant = CoarseVariant::scalar;
  HeatOperators ops(cfg, arith());
  auto part = build_time_partition(8, 2);
  auto schur = make_schur_solver(ops, part, cfg);
  auto rhs = assemble_rhs(ops, model_initial_condition, model_target);
  auto res = gmres_solve(ops, schur, rhs.to_kkt().data);
  REQUIRE(res.converged);
  for (std::size_t k = 1; k < res.residual_history.size(); ++k)
    CHECK(res.residual_history[k] <= res.residual_history[k - 1] * (1.0 + 1e-12) + 1e-15);
  const double est = res.residual_history.back();
  CHECK(res.true_final_relres <= 10.0 * est + 1e-15);
  CHECK(est <= 10.0 * res.true_final_relres + 1e-15);
  CHECK(int(res.residual_history.size()) == res.iterations);
}

TEST_CASE("zero rhs returns the zero solution, converged") {  // :103-110
  ProblemConfig cfg = desk_config(4, 2, 3, 3);
  HeatOperators ops(cfg, arith());
  auto part = build_time_partition(4, 2);
  auto schur = make_schur_solver(ops, part, cfg);
  auto res = gmres_solve(ops, schur, std::vector<double>(3 * ops.layout.size(), 0.0));
  CHECK(res.converged);
  CHECK(res.iterations == 0);
  for (double v : res.solution) CHECK(v == 0.0);
}

TEST_CASE("restarted cycles still converge") {  // :112-122
  ProblemConfig cfg = desk_config(8, 2, 4, 4, 1e-2);
  cfg.coarse_variant = CoarseVariant::scalar;
  cfg.gmres.restart = 5;
  cfg.gmres.max_iters = 200;
  HeatOperators ops(cfg, arith());
  auto part = build_time_partition(8, 2);
  auto schur = make_schur_solver(ops, part, cfg);
  auto rhs = assemble_rhs(ops, model_initial_condition, model_target);
  auto res = gmres_solve(ops, schur, rhs.to_kkt().data);
  CHECK(res.converged);
  CHECK(res.true_final_relres <= 10.0 * cfg.gmres.tol);
}

TEST_CASE("non-finite Krylov vectors raise a divergence error naming the iteration") {  // :141-153
  ProblemConfig cfg = desk_config(4, 2, 3, 3);
  HeatOperators ops(cfg, arith());
  auto part = build_time_partition(4, 2);
  auto schur = make_schur_solver(ops, part, cfg);
  std::vector<double> b(3 * ops.layout.size(), 1.0);
  b[1] = std::numeric_limits<double>::quiet_NaN();
  CHECK_THROWS_AS(gmres_solve(ops, schur, b), GmresDivergenceError);
  try {
    gmres_solve(ops, schur, b);
  } catch (const GmresDivergenceError& e) {
    CHECK(e.iteration == 1);
    CHECK(std::string(e.what()).find("1") != std::string::npos);
  }
}

TEST_CASE("non-converged runs still report the least-squares iterate") {  // :155-167
  ProblemConfig cfg = desk_config(8, 2, 4, 4, 1e-2);
  cfg.precond = PrecondKind::none;
  cfg.gmres.tol = 1e-14;
  cfg.gmres.max_iters = 5;
  HeatOperators ops(cfg, arith());
  auto part = build_time_partition(8, 2);
  auto schur = make_schur_solver(ops, part, cfg);
  auto rhs = assemble_rhs(ops, model_initial_condition, model_target);
  auto res = gmres_solve(ops, schur, rhs.to_kkt().data);
  CHECK_FALSE(res.converged);
  CHECK(res.iterations == 5);
  CHECK(res.true_final_relres < 1.0);
  CHECK(res.true_final_relres == doctest::Approx(res.residual_history.back()).epsilon(1e-6));
}

// ----------------------------------------------------- test_experiments.cpp
namespace {
ProblemConfig tiny_config() {  // :13-23
  ProblemConfig cfg;
  cfg.Nt = 4;
  cfg.Nd = 2;
  cfg.Nx = 3;
  cfg.Ny = 3;
  cfg.omega = 1e-2;
  cfg.precond = PrecondKind::two_level;
  cfg.coarse_variant = CoarseVariant::per_dof;
  return cfg;
}
}  // namespace

TEST_CASE("run_single solves the tiny benchmark reproducibly") {  // :73-81
  const auto rec1 = run_single(tiny_config(), nullptr, arith());
  CHECK(rec1.converged);
  CHECK(rec1.true_final_relres <= 1e-5);
  CHECK(rec1.objective > 0.0);
  const auto rec2 = run_single(tiny_config(), nullptr, arith());
  CHECK(rec1.iterations == rec2.iterations);
  CHECK(rec1.true_final_relres == rec2.true_final_relres);
}

TEST_CASE("unpreconditioned runs take more iterations than two-level") {  // :83-91
  ProblemConfig none = tiny_config();
  none.precond = PrecondKind::none;
  none.gmres.max_iters = 2000;
  const auto rec_none = run_single(none, nullptr, arith());
  const auto rec_two = run_single(tiny_config(), nullptr, arith());
  CHECK(rec_none.converged);
  CHECK(rec_none.iterations > rec_two.iterations);
}

TEST_CASE("non-convergence is recorded, not raised") {  // :185-192
  ProblemConfig cfg = tiny_config();
  cfg.precond = PrecondKind::none;
  cfg.gmres.max_iters = 2;
  cfg.gmres.tol = 1e-14;
  const auto rec = run_single(cfg, nullptr, arith());
  CHECK_FALSE(rec.converged);
  CHECK(rec.iterations == 2);
}
