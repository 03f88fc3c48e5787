// run_single_driver.cpp — run_single's wiring (reference src/experiments.cpp:33-69)
// through the reference-side binding: operators, partition, Schur solver, the model
// right-hand side, device GMRES, objective; prints the reference's JSON RunRecord
// keys (experiments.cpp:179-208).  Also runs the same solve through the one-call
// kkt_run_single entry point and checks the two agree.
//
//   run_single_driver [Nx Ny Nt Nd omega [scalar|per-dof] [strict]]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kktdd_gpu.hpp"

using namespace kktdd_gpu;

int main(int argc, char** argv) {
  ProblemConfig cfg;
  if (argc > 5) {
    cfg.Nx = std::atoi(argv[1]);
    cfg.Ny = std::atoi(argv[2]);
    cfg.Nt = std::atoi(argv[3]);
    cfg.Nd = std::atoi(argv[4]);
    cfg.omega = std::atof(argv[5]);
  }
  if (argc > 6 && std::strcmp(argv[6], "scalar") == 0) cfg.coarse_variant = CoarseVariant::scalar;
  const Arithmetic mode = (argc > 7 && std::strcmp(argv[7], "strict") == 0) ? Arithmetic::strict : Arithmetic::fast;
  try {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    HeatOperators ops(cfg, mode);                                   // experiments.cpp:39
    const TimePartition part = build_time_partition(cfg.Nt, cfg.Nd);  // :40
    const SchurSolver schur = make_schur_solver(ops, part, cfg);    // :41
    const RhsBundle rhs = assemble_rhs(ops, model_initial_condition, model_target);  // :42
    const KKTVector b = rhs.to_kkt();
    const double setup_s = std::chrono::duration<double>(clock::now() - t0).count();
    const auto t1 = clock::now();
    const GmresResult res = gmres_solve(ops, schur, b.data);        // :46-57
    const double solve_s = std::chrono::duration<double>(clock::now() - t1).count();
    const std::size_t nb = ops.layout.size();
    const std::span<const double> sol(res.solution);
    const double obj = evaluate_objective(ops, sol.subspan(0, nb), sol.subspan(nb, nb), model_target);  // :62-64
    const RunRecord one = run_single(cfg, nullptr, mode);
    const bool agree = one.iterations == res.iterations && one.true_final_relres == res.true_final_relres &&
                       one.objective == obj;
    std::printf("{\"nx\": %d, \"ny\": %d, \"nt\": %d, \"nd\": %d, \"omega\": %.17g, \"iterations\": %d, "
                "\"converged\": %s, \"true_final_relres\": %.17g, \"objective\": %.17g, \"setup_seconds\": %.6f, "
                "\"solve_seconds\": %.6f, \"kkt_run_single_agrees\": %s}\n",
                cfg.Nx, cfg.Ny, cfg.Nt, cfg.Nd, cfg.omega, res.iterations, res.converged ? "true" : "false",
                res.true_final_relres, obj, setup_s, solve_s, agree ? "true" : "false");
    return agree ? 0 : 3;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "configuration error: %s\n", e.what());
    return 1;  // the reference CLI's exit code for config errors (kktdd_cli.cpp:263-267)
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
