// sweep.cuh — step descriptors of the spatial-solve chains (strict + fast).
#pragma once

#include "ctx.cuh"

namespace kkt {

// One spatial solve of a chain (strict path).
//   out = Ahat^{-1} v   (transpose == 0, BandedLU::solve_in_place)
//   out = Ahat^{-T} v   (transpose == 1, BandedLU::solve_transpose_in_place)
//   v   = in * scale (if scale != 1) + add (if add != null)
// in == nullptr marks an idle step.  in == out is allowed (in place).
struct SolveStep {
  const double* in;
  const double* add;
  double* out;
  double scale;
  int transpose;
};

// One spatial solve of a fast chain.  v as above, optionally minus the
// analytic two-level residual term (Shat y_c)_node when node > 0; after the
// solve x goes to `out` and, if out2 != null, x + gamma[node2] to out2.
struct FastStep {
  const double* in;
  const double* add;
  double* out;
  double* out2;
  double scale;
  int node;    // 1-based node for the fused coarse residual, 0 = none
  int node2;   // 1-based node whose gamma is added into out2
};

void strict_chains(Ctx* c, const SolveStep* jobs_dev, int nchains, int nsteps);
void fast_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms);
bool tma_supported(const Ctx* c);
bool group_supported(const Ctx* c);
void build_group_operators(Ctx* c);
void group_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms);
void tma_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms);
bool v4_supported(const Ctx* c);
int v4_group_size(const Ctx* c);
void build_v4(Ctx* c, const double* G, const double* H, const double* Li, const double* dinv);
void v4_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms);
void v4_unregister(Ctx* c);
bool v5_supported(const Ctx* c);
void build_v5(Ctx* c);
void v5_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms);
bool v6_supported(const Ctx* c);
void build_v6(Ctx* c);
void v6_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms);

}  // namespace kkt
