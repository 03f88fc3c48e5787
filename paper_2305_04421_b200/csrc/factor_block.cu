// factor_block.cu — K6 for large grids (FAST mode, nx > 128: configs 2-4).
//
// The reference's banded LU (linalg.cpp:69-125) of Ahat is pivot-free on these
// problems, and an unpivoted LU is unique, so its block form
// can be computed by the block recursion on the nx-by-nx diagonal blocks
//     D_0 = T,   D_J = T - cy^2 D_{J-1}^{-1},   D_J = L_JJ U_JJ,
// with T = tridiag(-cx, diag(Ahat), -cx) and D_{J-1}^{-1} = Ui_{J-1} Li_{J-1}.
// It produces the sweep operators Li_J = L_JJ^{-1}, Ui_J = U_JJ^{-1} directly
// (the same factors as the banded LU up to rounding) with dense, L2-resident
// work per block instead of ny*nx rank-1 updates over the whole band.
// A pivot below 1e-14 ||Ahat||_inf (linalg.cpp:10,98-103) raises
// SingularMatrixError with the global row index, as the banded LU would.
#include <cmath>

#include "ctx.cuh"

namespace kkt {
namespace {

constexpr int kLuThreads = 1024;

// D = T - cy^2 * S   (S == nullptr: D = T)
__global__ void form_d_kernel(int n, double diag, double mcx, double cy2, const double* __restrict__ S,
                              double* __restrict__ D) {
  const int64_t nn = int64_t(n) * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nn;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int a = int(e / n), b = int(e - int64_t(a) * n);
    double v = a == b ? diag : ((a - b == 1 || b - a == 1) ? mcx : 0.0);
    if (S) v -= cy2 * S[e];
    D[e] = v;
  }
}

// Unpivoted right-looking LU in place, one CTA (the matrix is L2-resident).
__global__ void __launch_bounds__(kLuThreads) dense_lu_nopiv_kernel(int n, double tol, double* A,
                                                                    int* status) {
  for (int j = 0; j < n; ++j) {
    const double d = A[int64_t(j) * n + j];
    if (!(fabs(d) > tol)) {
      if (threadIdx.x == 0) *status = j;
      return;
    }
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) A[int64_t(i) * n + j] /= d;
    __syncthreads();
    const int rows = n - j - 1;
    const int64_t pairs = int64_t(rows) * rows;
    for (int64_t t = threadIdx.x; t < pairs; t += blockDim.x) {
      const int i = j + 1 + int(t / rows);
      const int c = j + 1 + int(t % rows);
      A[int64_t(i) * n + c] = fma(-A[int64_t(i) * n + j], A[int64_t(j) * n + c], A[int64_t(i) * n + c]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = -1;
}

// Li = (unit lower of A)^{-1}, Ui = (upper of A)^{-1}; one thread per column,
// columns spread over CTAs.
// The same unpivoted LU, spread over a co-resident grid with a grid barrier
// after the multipliers and after the rank-1 update of every column: each
// element sees exactly the single-CTA kernel's operations in the same order
// (the division, then fma(-A[i][j], A[j][c], A[i][c]) for j ascending), so the
// factors are bitwise those of dense_lu_nopiv_kernel.  That kernel took
// ~148 ms per 1023 x 1023 block on one SM, 72% of the config-4 setup.
// All reads of A go through L2 (__ldcg): other CTAs wrote it since the last barrier.
constexpr int kLuCoopThreads = 512;

__global__ void __launch_bounds__(kLuCoopThreads) dense_lu_nopiv_coop_kernel(int n, double tol, double* A,
                                                                             int* status, unsigned* bar) {
  const int nt = gridDim.x * blockDim.x, gt = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned target = 0;
  auto gsync = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      target += gridDim.x;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
      } while (v < target);
    }
    __syncthreads();
  };
  for (int j = 0; j < n; ++j) {
    const double d = __ldcg(&A[int64_t(j) * n + j]);
    if (!(fabs(d) > tol)) {
      if (gt == 0) *status = j;
      return;  // every CTA reads the same pivot: a uniform exit
    }
    for (int i = j + 1 + gt; i < n; i += nt) A[int64_t(i) * n + j] = __ldcg(&A[int64_t(i) * n + j]) / d;
    gsync();
    const int rows = n - j - 1;
    const int64_t pairs = int64_t(rows) * rows;
    for (int64_t t = gt; t < pairs; t += nt) {
      const int i = j + 1 + int(t / rows);
      const int c = j + 1 + int(t % rows);
      A[int64_t(i) * n + c] =
          fma(-__ldcg(&A[int64_t(i) * n + j]), __ldcg(&A[int64_t(j) * n + c]), __ldcg(&A[int64_t(i) * n + c]));
    }
    gsync();
  }
  if (gt == 0) *status = -1;
}

// Threads 0..n-1 invert L (column b each), threads n..2n-1 invert U: the two
// sequential column solves run side by side (same operations per element).
__global__ void tri_inverse_kernel(int n, const double* __restrict__ A, double* __restrict__ Li,
                                   double* __restrict__ Ui) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * n) return;
  const bool upper = t >= n;
  const int b = upper ? t - n : t;
  if (!upper)
  for (int a = 0; a < n; ++a) {
    double acc = (a == b) ? 1.0 : 0.0;
    if (a > b)
      for (int k = b; k < a; ++k) acc = fma(-A[int64_t(a) * n + k], Li[int64_t(k) * n + b], acc);
    Li[int64_t(a) * n + b] = acc;
  }
  if (upper)
  for (int a = n - 1; a >= 0; --a) {
    double acc = 0.0;
    if (a <= b) {
      acc = (a == b) ? 1.0 : 0.0;
      for (int k = a + 1; k <= b; ++k) acc = fma(-A[int64_t(a) * n + k], Ui[int64_t(k) * n + b], acc);
      acc /= A[int64_t(a) * n + a];
    }
    Ui[int64_t(a) * n + b] = acc;
  }
}

// C = A * B (n x n, row-major), 32x32 tiles through shared memory.
__global__ void gemm_kernel(int n, const double* __restrict__ A, const double* __restrict__ B,
                            double* __restrict__ C) {
  __shared__ double As[32][33], Bs[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int row0 = blockIdx.y * 32, col = blockIdx.x * 32 + tx;
  double acc[4] = {0, 0, 0, 0};
  for (int k0 = 0; k0 < n; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const int ar = row0 + r, ac = k0 + tx;
      As[r][tx] = (ar < n && ac < n) ? A[int64_t(ar) * n + ac] : 0.0;
      const int br = k0 + r;
      Bs[r][tx] = (br < n && col < n) ? B[int64_t(br) * n + col] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double bv = Bs[k][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][k], bv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = row0 + ty + 8 * q;
    if (r < n && col < n) C[int64_t(r) * n + col] = acc[q];
  }
}

// B = f * A
__global__ void scale_copy_kernel(int64_t n, double f, const double* __restrict__ A, double* __restrict__ B) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    B[e] = f * A[e];
}

}  // namespace

// ||Ahat||_inf as in build_factor (linalg.cpp:35-43 order)
static double ahat_inf_norm(const Ctx* c) {
  const int nx = c->nx, ny = c->ny;
  double anorm = 0.0;
  for (int j = 1; j <= ny; ++j)
    for (int i = 1; i <= nx; ++i) {
      double row = 0.0;
      if (j > 1) row += std::abs(c->Ahat.mcy);
      if (i > 1) row += std::abs(c->Ahat.mcx);
      row += std::abs(c->Ahat.diag);
      if (i < nx) row += std::abs(c->Ahat.mcx);
      if (j < ny) row += std::abs(c->Ahat.mcy);
      anorm = std::max(anorm, row);
    }
  return anorm;
}

// D (nx x nx, overwritten by its unpivoted LU) -> Li = L^{-1}, Ui = U^{-1}; returns the failing
// pivot column or -1 (read back after the stream drains)
static int lu_and_inverses(Ctx* c, double tol, double* D, double* Li, double* Ui, DBuf<int>& st, DBuf<unsigned>& bar) {
  const int nx = c->nx;
  static const bool single = getenv("KKT_LU_SINGLE") != nullptr;  // testing: the one-CTA kernel
  if (single) {
    KKT_LAUNCH(c, dense_lu_nopiv_kernel, 1, kLuThreads, 0, nx, tol, D, st.p);
  } else {
    KKT_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(unsigned), c->stream));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kSmCount);
    cfg.blockDim = dim3(kLuCoopThreads);
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers: every CTA co-resident
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n_ = nx;
    double tol_ = tol;
    double* A_ = D;
    int* st_ = st.p;
    unsigned* bar_ = bar.p;
    void* args[] = {&n_, &tol_, &A_, &st_, &bar_};
    KKT_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(&dense_lu_nopiv_coop_kernel), args));
    c->launches++;
  }
  KKT_LAUNCH(c, tri_inverse_kernel, (2 * nx + 63) / 64, 64, 0, nx, D, Li, Ui);
  return 0;
}

void build_block_recursion(Ctx* c) {
  const int nx = c->nx, ny = c->ny;
  const int64_t nn = int64_t(nx) * nx;
  const double tol = 1e-14 * ahat_inf_norm(c);
  c->Li.alloc(size_t(ny) * nn);
  c->Ui.alloc(size_t(ny) * nn);
  DBuf<double> D(nn), S(nn);
  DBuf<int> st(1);
  DBuf<unsigned> bar(1);
  const double cy2 = c->cy * c->cy;
  const dim3 gg((nx + 31) / 32, (nx + 31) / 32), gb(32, 8);
  for (int J = 0; J < ny; ++J) {
    KKT_LAUNCH(c, form_d_kernel, kSmCount * 2, 256, 0, nx, c->Ahat.diag, c->Ahat.mcx, cy2,
               J > 0 ? S.p : nullptr, D.p);
    double* Li = c->Li.p + J * nn;
    double* Ui = c->Ui.p + J * nn;
    lu_and_inverses(c, tol, D.p, Li, Ui, st, bar);
    if (J + 1 < ny) KKT_LAUNCH(c, gemm_kernel, gg, gb, 0, nx, Ui, Li, S.p);
    int hs = -1;
    KKT_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    if (hs >= 0)
      throw Error(KKT_ESINGULAR,
                  "block LU: pivot below tolerance " + std::to_string(tol) + " at index " +
                      std::to_string(J * nx + hs),
                  J * nx + hs);
  }
  c->pivoted = false;
}

// Middle block of the two-sided (twisted) elimination, ny odd, M = (ny - 1) / 2 (sweep_v6.cu).
// Ahat's block rows are all (-cy I, T, -cy I), so eliminating upward from the last block row
// gives the mirror image of the downward recursion (D'_J = D_{ny-1-J}); the two eliminations
// meet in block row M, whose Schur complement is
//     Dm = T - cy^2 D_{M-1}^{-1} - cy^2 D'_{M+1}^{-1} = T - 2 cy^2 Ui_{M-1} Li_{M-1}.
// Outputs (nx x nx, row-major): Dinv = Dm^{-1}, E = cy Dm^{-1} Ui_{M-1}, so that
//     x_M = Dinv b_M + E (y_{M-1} + y'_{M+1}).
// E2 (optional) = cy Dm^{-1} H_{M-1} = cy^2 Dm^{-1} Ui_{M-1} Li_{M-1}: the same row in the inverse-block
// form of the elimination (sweep_v6.cu, "Thomas form"), where the chains carry y_J = b_J/cy + z_{J-1}
// and z_{M-1} = H_{M-1} y_{M-1}:  x_M = Dinv b_M + E2 (y_{M-1} + y'_{M+1}).
void build_twist_middle(Ctx* c, int M, double* Dinv, double* E, double* E2) {
  const int nx = c->nx;
  const int64_t nn = int64_t(nx) * nx;
  const double tol = 1e-14 * ahat_inf_norm(c);
  DBuf<double> D(nn), S(nn), Lm(nn), Um(nn);
  DBuf<int> st(1);
  DBuf<unsigned> bar(1);
  const dim3 gg((nx + 31) / 32, (nx + 31) / 32), gb(32, 8);
  const double* Lp = c->Li.p + int64_t(M - 1) * nn;
  const double* Up = c->Ui.p + int64_t(M - 1) * nn;
  KKT_LAUNCH(c, gemm_kernel, gg, gb, 0, nx, Up, Lp, S.p);
  DBuf<double> S2(E2 ? nn : 0);
  if (E2) KKT_CUDA(cudaMemcpyAsync(S2.p, S.p, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c->stream));
  KKT_LAUNCH(c, form_d_kernel, kSmCount * 2, 256, 0, nx, c->Ahat.diag, c->Ahat.mcx, 2.0 * c->cy * c->cy, S.p, D.p);
  lu_and_inverses(c, tol, D.p, Lm.p, Um.p, st, bar);
  KKT_LAUNCH(c, gemm_kernel, gg, gb, 0, nx, Um.p, Lm.p, Dinv);
  KKT_LAUNCH(c, gemm_kernel, gg, gb, 0, nx, Dinv, Up, S.p);
  KKT_LAUNCH(c, scale_copy_kernel, kSmCount * 2, 256, 0, nn, c->cy, S.p, E);
  if (E2) {
    KKT_LAUNCH(c, gemm_kernel, gg, gb, 0, nx, Dinv, S2.p, S.p);
    KKT_LAUNCH(c, scale_copy_kernel, kSmCount * 2, 256, 0, nn, c->cy * c->cy, S.p, E2);
  }
  int hs = -1;
  KKT_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  if (hs >= 0)
    throw Error(KKT_ESINGULAR,
                "block LU (middle block): pivot below tolerance " + std::to_string(tol) + " at index " +
                    std::to_string(M * nx + hs),
                M * nx + hs);
}

}  // namespace kkt
