// common.cuh — shared definitions of the B200 KKT hot path (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kktdd_b200.h"

namespace kkt {

// Error carrying a C-ABI status (mirrors the reference's exception taxonomy,
// see include/kktdd_b200.h).
struct Error : std::runtime_error {
  int status;
  int index;
  Error(int st, const std::string& what, int idx = -1)
      : std::runtime_error(what), status(st), index(idx) {}
};

#define KKT_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::kkt::Error(KKT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Launch bookkeeping: every kernel goes through KKT_LAUNCH so the context can
// report how many of its own kernels ran (bench.py's gpu_launches).
#define KKT_LAUNCH(ctx, kernel, grid, block, smem, ...)                     \
  do {                                                                     \
    kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);       \
    (ctx)->launches++;                                                     \
    cudaError_t e_ = cudaGetLastError();                                   \
    if (e_ != cudaSuccess)                                                 \
      throw ::kkt::Error(KKT_ECUDA, std::string(#kernel) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kSmCount = 148;  // B200

// Strict-mode arithmetic: no FMA contraction, IEEE round-to-nearest, the
// reference's operand order.  (nvcc would otherwise fuse a*b+c.)
__device__ __forceinline__ double smul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ssub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double sdiv(double a, double b) { return __ddiv_rn(a, b); }

// Stencil coefficients of A (or Ahat) = tridiag blocks: the reference's
// assemble_spatial_operator (heat_operators.cpp:24-44) + make_ahat (:16-20).
struct Stencil {
  int nx, ny;     // interior points per row / column
  double diag;    // 1 + 2cx + 2cy [- sigma*dt]
  double mcx;     // -cx
  double mcy;     // -cy
};

// Reference band_matvec row (linalg.cpp:45-54) for the 5-point band: terms
// in ascending column order p-nx, p-1, p, p+1, p+nx from acc = 0, each
// product separately rounded.  Zero band entries contribute (+-0), which is
// bitwise neutral for finite x, so they are skipped.
// A is symmetric, so band_matvec_transpose (:56-67) yields the same terms in
// the same order.
__device__ __forceinline__ double band_row_strict_ij(const Stencil& s, const double* __restrict__ x,
                                                     int p, int i, int j) {
  double acc = 0.0;
  if (j > 0) acc = sadd(acc, smul(s.mcy, x[p - s.nx]));
  if (i > 0) acc = sadd(acc, smul(s.mcx, x[p - 1]));
  acc = sadd(acc, smul(s.diag, x[p]));
  if (i < s.nx - 1) acc = sadd(acc, smul(s.mcx, x[p + 1]));
  if (j < s.ny - 1) acc = sadd(acc, smul(s.mcy, x[p + s.nx]));
  return acc;
}

__device__ __forceinline__ double band_row_strict(const Stencil& s, const double* __restrict__ x,
                                                  int p) {
  const int i = p % s.nx;
  const int j = p / s.nx;
  double acc = 0.0;
  if (j > 0) acc = sadd(acc, smul(s.mcy, x[p - s.nx]));
  if (i > 0) acc = sadd(acc, smul(s.mcx, x[p - 1]));
  acc = sadd(acc, smul(s.diag, x[p]));
  if (i < s.nx - 1) acc = sadd(acc, smul(s.mcx, x[p + 1]));
  if (j < s.ny - 1) acc = sadd(acc, smul(s.mcy, x[p + s.nx]));
  return acc;
}

}  // namespace kkt
