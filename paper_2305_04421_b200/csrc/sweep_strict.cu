// sweep_strict.cu — STRICT (bitwise) spatial solves and the RASQ sweep.
//
// One warp per right-hand side reproduces BandedLU::solve_in_place
// (reference linalg.cpp:127-145) and solve_transpose_in_place (:147-162) in
// their exact floating-point order:
//  * L and U substitutions and the U^T substitution are column-oriented in
//    the reference (or equivalently ordered), so each step broadcasts one
//    final value and the warp applies <= kl independent updates to a
//    circular window of pending rows held in shared memory;
//  * the L^T substitution is a dot product whose order starts at the most
//    recently finalised entry, so it is a sequential chain per row (lane 0),
//    with the products formed in parallel.
// Factor columns are streamed through a cp.async ring.  The exactly-zero
// fill band of U (no row interchanges: SURVEY.md §8a-6) and b_j == 0 updates
// (linalg.cpp:133,141) are skipped, which is bitwise neutral.
// A fully general single-thread path (with the pivot swaps) covers factors
// that did interchange rows.
#include "ctx.cuh"

namespace kkt {
namespace {

constexpr int kRing = 8;

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Row-initialiser of a solve: value_i = (scale ? in_i*scale : in_i) [+ add_i]
// (window solves: x_k += x_{k-1} / x_{k+1}, heat_operators.cpp:146-150,162-166;
//  apply_rasq's win *= ms, schur.cpp:119).
struct RowInit {
  const double* in;
  const double* add;
  double scale;
  bool use_scale;
  __device__ __forceinline__ double operator()(int i) const {
    double v = in[i];
    if (use_scale) v = smul(v, scale);
    if (add) v = sadd(v, add[i]);
    return v;
  }
};

}  // namespace
}  // namespace kkt
#include "sweep.cuh"
namespace kkt {
namespace {

// ---------------------------------------------------------------------------
// Forward / back substitution with L then U (solve_in_place), no pivoting.
// ---------------------------------------------------------------------------
__device__ void warp_solve_LU(int n, int kl, int kuf, int ld, const double* __restrict__ ab,
                              RowInit init, double* out, double* win, int W,
                              double* ring, int KLP) {
  const int lane = threadIdx.x & 31;
  const int M = W - 1;
  // ---------------- L: for j ascending, b[i] -= L(i,j) b[j], i = j+1..j+kl
  for (int i = lane; i < W && i < n; i += 32) win[i] = init(i);
  auto issueL = [&](int col) {
    if (col < n) {
      const double* src = ab + int64_t(col) * ld + kuf + 1;
      double* dst = ring + (col % kRing) * KLP;
      for (int o = lane; o < kl; o += 32) cp_async8(dst + o, src + o);
    }
    cp_commit();
  };
  for (int c0 = 0; c0 < kRing - 1; ++c0) issueL(c0);
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    issueL(j + kRing - 1);
    cp_wait<kRing - 1>();
    const double bj = win[j & M];
    __syncwarp();
    if (lane == 0) {
      out[j] = bj;
      if (j + W < n) win[j & M] = init(j + W);
    }
    if (bj != 0.0) {
      const double* col = ring + (j % kRing) * KLP;
      const int lim = min(kl, n - 1 - j);
      for (int o = lane; o < lim; o += 32) {
        const int i = j + 1 + o;
        win[i & M] = ssub(win[i & M], smul(col[o], bj));
      }
    }
    __syncwarp();
  }
  cp_wait<0>();
  __syncwarp();
  // ---------------- U: for j descending, b[j] /= U(j,j); b[i] -= U(i,j) b[j], i = j-kl..j-1
  for (int t = lane; t < W && t < n; t += 32) {
    const int i = n - 1 - t;
    win[i & M] = out[i];
  }
  auto issueU = [&](int col) {  // col counts down
    if (col >= 0) {
      const double* src = ab + int64_t(col) * ld + kuf - kl;  // rows col-kl .. col-1
      double* dst = ring + (col % kRing) * KLP;
      for (int o = lane; o < kl; o += 32) cp_async8(dst + o, src + o);
    }
    cp_commit();
  };
  for (int c0 = 0; c0 < kRing - 1; ++c0) issueU(n - 1 - c0);
  __syncwarp();
  for (int j = n - 1; j >= 0; --j) {
    issueU(j - (kRing - 1));
    cp_wait<kRing - 1>();
    const double ujj = ab[int64_t(j) * ld + kuf];
    const double bj = sdiv(win[j & M], ujj);
    __syncwarp();
    if (lane == 0) {
      out[j] = bj;
      if (j - W >= 0) win[j & M] = out[j - W];
    }
    if (bj != 0.0) {
      const double* col = ring + (((j % kRing) + kRing) % kRing) * KLP;  // col[o] = U(j-kl+o, j)
      const int lo = max(0, j - kl);
      for (int i = lo + lane; i < j; i += 32) {
        win[i & M] = ssub(win[i & M], smul(col[i - (j - kl)], bj));
      }
    }
    __syncwarp();
  }
  cp_wait<0>();
}

// ---------------------------------------------------------------------------
// Transpose solve: U^T (forward, column-oriented via rows of U) then L^T
// (backward, sequential dot chains), no pivoting.
// ---------------------------------------------------------------------------
__device__ void warp_solve_T(int n, int kl, int kuf, int ld, const double* __restrict__ ab,
                             const double* __restrict__ ut, RowInit init, double* out,
                             double* win, int W, double* ring, int KLP, double* prod) {
  const int lane = threadIdx.x & 31;
  const int M = W - 1;
  // ---------------- U^T y = b: acc_j -= U(i,j) b[i] for i ascending; b[j] = acc_j / U(j,j)
  for (int i = lane; i < W && i < n; i += 32) win[i] = init(i);
  auto issue = [&](int row) {
    if (row < n) {
      const double* src = ut + int64_t(row) * kl;  // U(row, row+1 .. row+kl)
      double* dst = ring + (row % kRing) * KLP;
      for (int o = lane; o < kl; o += 32) cp_async8(dst + o, src + o);
    }
    cp_commit();
  };
  for (int c0 = 0; c0 < kRing - 1; ++c0) issue(c0);
  __syncwarp();
  for (int i = 0; i < n; ++i) {
    issue(i + kRing - 1);
    cp_wait<kRing - 1>();
    const double uii = ab[int64_t(i) * ld + kuf];
    const double bi = sdiv(win[i & M], uii);
    __syncwarp();
    if (lane == 0) {
      out[i] = bi;
      if (i + W < n) win[i & M] = init(i + W);
    }
    const double* row = ring + (i % kRing) * KLP;
    const int lim = min(kl, n - 1 - i);
    for (int o = lane; o < lim; o += 32) {
      const int j = i + 1 + o;
      win[j & M] = ssub(win[j & M], smul(row[o], bi));
    }
    __syncwarp();
  }
  cp_wait<0>();
  __syncwarp();
  // ---------------- L^T x = y, j descending: acc = y[j] - sum_{i=j+1..j+kl, ascending} L(i,j) x[i]
  // win holds the final x of rows j+1 .. j+kl (slots i & M).
  for (int j = n - 1; j >= 0; --j) {
    const int cnt = min(kl, n - 1 - j);
    const double* colL = ab + int64_t(j) * ld + kuf + 1;  // L(j+1+o, j)
    for (int o = lane; o < cnt; o += 32) prod[o] = smul(colL[o], win[(j + 1 + o) & M]);
    __syncwarp();
    if (lane == 0) {
      double acc = out[j];
      int o = 0;
      for (; o + 8 <= cnt; o += 8) {
        const double p0 = prod[o], p1 = prod[o + 1], p2 = prod[o + 2], p3 = prod[o + 3];
        const double p4 = prod[o + 4], p5 = prod[o + 5], p6 = prod[o + 6], p7 = prod[o + 7];
        acc = ssub(acc, p0); acc = ssub(acc, p1); acc = ssub(acc, p2); acc = ssub(acc, p3);
        acc = ssub(acc, p4); acc = ssub(acc, p5); acc = ssub(acc, p6); acc = ssub(acc, p7);
      }
      for (; o < cnt; ++o) acc = ssub(acc, prod[o]);
      win[j & M] = acc;
      out[j] = acc;
    }
    __syncwarp();
  }
}

// General path with row interchanges: the reference loops verbatim, one
// thread per right-hand side.
__device__ void thread_solve_general(int n, int kl, int kuf, int ld, const double* ab,
                                     const int* piv, RowInit init, double* b, bool transpose) {
  auto E = [&](int i, int j) { return ab[int64_t(j) * ld + (i - j + kuf)]; };
  for (int i = 0; i < n; ++i) b[i] = init(i);
  if (!transpose) {
    for (int j = 0; j < n; ++j) {
      if (piv[j] != j) { const double t = b[j]; b[j] = b[piv[j]]; b[piv[j]] = t; }
      const double bj = b[j];
      if (bj != 0.0)
        for (int i = j + 1; i <= min(n - 1, j + kl); ++i) b[i] = ssub(b[i], smul(E(i, j), bj));
    }
    for (int j = n - 1; j >= 0; --j) {
      b[j] = sdiv(b[j], E(j, j));
      const double bj = b[j];
      if (bj != 0.0)
        for (int i = max(0, j - kuf); i < j; ++i) b[i] = ssub(b[i], smul(E(i, j), bj));
    }
  } else {
    for (int j = 0; j < n; ++j) {
      double acc = b[j];
      for (int i = max(0, j - kuf); i < j; ++i) acc = ssub(acc, smul(E(i, j), b[i]));
      b[j] = sdiv(acc, E(j, j));
    }
    for (int j = n - 1; j >= 0; --j) {
      double acc = b[j];
      for (int i = j + 1; i <= min(n - 1, j + kl); ++i) acc = ssub(acc, smul(E(i, j), b[i]));
      b[j] = acc;
      if (piv[j] != j) { const double t = b[j]; b[j] = b[piv[j]]; b[piv[j]] = t; }
    }
  }
}

// Each CTA (one warp) runs its own chain of solves: jobs[blockIdx.x*nsteps + t].
__global__ void __launch_bounds__(32) strict_chain_kernel(
    int n, int kl, int kuf, int ld, const double* __restrict__ ab, const double* __restrict__ ut,
    const int* __restrict__ piv, bool pivoted, const SolveStep* __restrict__ jobs, int nsteps,
    int W, int KLP) {
  extern __shared__ double smem[];
  double* win = smem;
  double* ring = win + W;
  double* prod = ring + kRing * KLP;
  for (int t = 0; t < nsteps; ++t) {
    const SolveStep job = jobs[int64_t(blockIdx.x) * nsteps + t];
    if (!job.in) continue;
    RowInit init{job.in, job.add, job.scale, job.scale != 1.0};
    if (pivoted) {
      if (threadIdx.x == 0)
        thread_solve_general(n, kl, kuf, ld, ab, piv, init, job.out, job.transpose != 0);
    } else if (!job.transpose) {
      warp_solve_LU(n, kl, kuf, ld, ab, init, job.out, win, W, ring, KLP);
    } else {
      warp_solve_T(n, kl, kuf, ld, ab, ut, init, job.out, win, W, ring, KLP, prod);
    }
    __syncthreads();  // global writes of this step visible to the next (same CTA)
  }
}

int pow2_at_least(int v) {
  int w = 1;
  while (w < v) w <<= 1;
  return w;
}

}  // namespace

// Launch `nchains` independent chains of `nsteps` strict spatial solves
// (step: out = Ahat^{-1} init or Ahat^{-T} init, init = in*scale + add).
// `jobs_dev` is device memory, chain-major.
void strict_chains(Ctx* c, const SolveStep* jobs_dev, int nchains, int nsteps) {
  if (nchains <= 0 || nsteps <= 0) return;
  const int n = c->nsp;
  const int kl = c->kl;
  const int W = pow2_at_least(kl + 1);
  const int KLP = ((kl + 31) / 32) * 32 + 32;
  const size_t smem = sizeof(double) * (size_t(W) + size_t(kRing) * KLP + KLP);
  static bool attr_set = false;
  if (!attr_set) {
    KKT_CUDA(cudaFuncSetAttribute(strict_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr_set = true;
  }
  KKT_LAUNCH(c, strict_chain_kernel, nchains, 32, smem, n, kl, c->kuf, c->ld, c->ab.p, c->ut.p,
             c->piv.p, c->pivoted, jobs_dev, nsteps, W, KLP);
}

}  // namespace kkt
