// spectral.cu — SPECTRAL-mode RASQ (K5) in Ahat's eigenbasis (opt-in).
//
// Ahat = A - sigma*dt*I (heat_operators.cpp:16-20, :24-44) is the constant-
// coefficient 5-point operator on the nx-by-ny interior grid with homogeneous
// Dirichlet boundaries, so the 2-D sine transform diagonalises it:
//     Ahat = S Lambda S,   S = Sy (x) Sx,   S^2 = I,
//     Sx[k][i] = sqrt(2/(nx+1)) sin(pi (k+1)(i+1)/(nx+1)),
//     lambda_{l,k} = diag + 2 mcx cos(pi (k+1)/(nx+1)) + 2 mcy cos(pi (l+1)/(ny+1)).
// A plane X (ny x nx, row-major) maps to Sy X Sx.  Every window solve of the
// reference's RASQ (schur.cpp:103-130: forward_solve_window, * ms,
// adjoint_solve_window, heat_operators.cpp:139-169) then decouples into one
// scalar recurrence per eigenmode q:
//     forward  y_n = rho_q (r^_n + y_{n-1}),        n = first .. last
//     adjoint  x_n = rho_q (ms y_n + x_{n+1}),      n = last .. owned.first
// with rho_q = 1/lambda_q — the same operator as the reference's banded-LU
// solves, to rounding.  The multiplicative two-level residual r - Shat y_c and
// the + y_c of the scalar coarse space are per-mode too (T(1) = c^,
// T(Ahat v) = lambda T(v)), so one P^-1 Schur apply is
//     2 transform passes -> one recurrence pass -> 2 transform passes,
// the transforms as fp64 tensor-core GEMMs (mma.sync m8n8k4 f64) against the
// resident nx x nx / ny x ny sine matrices.  No sequential chain of spatial
// solves remains: the dependency depth per apply is 2m scalar steps.
//
// This is NOT the reference's spatial-solve method (banded LU, linalg.cpp:
// 127-162), so it runs only in the opt-in KKT_MODE_SPECTRAL; FAST keeps the
// LU block substitution (sweep_group.cu), STRICT the reference-order banded
// substitution (sweep_strict.cu).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "ctx.cuh"

namespace kkt {
namespace {

// ---------------------------------------------------------------------------
// C[b] = A[b] * B[b], row-major fp64, on the fp64 tensor cores.
// CTA tile 64 x 64, k-tile 16, 4 warps (2 x 2), warp tile 32 x 32 = 4 x 4
// m8n8k4 fragments.  Register-staged double buffering of the k-tiles.
// ---------------------------------------------------------------------------
constexpr int kBM = 64, kBN = 64, kBK = 16;
constexpr int kGemmThreads = 128;
constexpr int kApad = 4, kBpad = 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kGemmThreads) gemm_f64_kernel(GemmArgs g) {
  __shared__ __align__(16) double As[2][kBM][kBK + kApad];
  __shared__ __align__(16) double Bs[2][kBK][kBN + kBpad];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int gi = lane >> 2, ti = lane & 3;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  const int64_t b = blockIdx.z;
  const double* A = g.A + b * g.sA;
  const double* B = g.B + b * g.sB;
  double* C = g.C + b * g.sC;

  constexpr int kLoads = kBM * kBK / kGemmThreads;  // 8 (A) and 8 (B)
  double ra[kLoads], rb[kLoads];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
      const int e = tid + kGemmThreads * i;
      const int r = e / kBK, cc = e % kBK;
      const int gm = m0 + r, gk = k0 + cc;
      ra[i] = (gm < g.M && gk < g.K) ? __ldg(A + int64_t(gm) * g.lda + gk) : 0.0;
      const int rr = e / kBN, cn = e % kBN;
      const int gk2 = k0 + rr, gn = n0 + cn;
      rb[i] = (gk2 < g.K && gn < g.N) ? __ldg(B + int64_t(gk2) * g.ldb + gn) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
      const int e = tid + kGemmThreads * i;
      As[buf][e / kBK][e % kBK] = ra[i];
      Bs[buf][e / kBN][e % kBN] = rb[i];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.K + kBK - 1) / kBK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * kBK);
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        af[f] = As[buf][wm * 32 + f * 8 + gi][kk + ti];
        bf[f] = Bs[buf][kk + ti][wn * 32 + f * 8 + gi];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm * 32 + i * 8 + gi;
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cn = n0 + wn * 32 + j * 8 + 2 * ti;
      if (cn < g.N) C[int64_t(r) * g.ldc + cn] = acc[i][j][0];
      if (cn + 1 < g.N) C[int64_t(r) * g.ldc + cn + 1] = acc[i][j][1];
    }
  }
}

}  // namespace

void gemm_f64(Ctx* c, const GemmArgs& g, int batch) {
  const dim3 grid((g.N + kBN - 1) / kBN, (g.M + kBM - 1) / kBM, batch);
  KKT_LAUNCH(c, gemm_f64_kernel, grid, kGemmThreads, 0, g);
}

namespace {

void gemm(Ctx* c, const GemmArgs& g, int batch) { gemm_f64(c, g, batch); }

// planes (P of them, ny x nx each, contiguous) -> Sy X Sx, via `tmp`
void transform(Ctx* c, const double* in, double* tmp, double* out, int P) {
  const int nx = c->nx, ny = c->ny;
  GemmArgs g1{in, c->sp_x.p, tmp, nx, nx, nx, 0, 0, 0, P * ny, nx, nx};
  gemm(c, g1, 1);                                       // X Sx
  GemmArgs g2{c->sp_y.p, tmp, out, ny, nx, nx, 0, c->nsp, c->nsp, ny, nx, ny};
  gemm(c, g2, P);                                       // Sy (X Sx)
}

// inverse order (Sy first) so that the last pass writes `out` directly
void transform_sy_first(Ctx* c, const double* in, double* tmp, double* out, int P) {
  const int nx = c->nx, ny = c->ny;
  GemmArgs g1{c->sp_y.p, in, tmp, ny, nx, nx, 0, c->nsp, c->nsp, ny, nx, ny};
  gemm(c, g1, P);
  GemmArgs g2{tmp, c->sp_x.p, out, nx, nx, nx, 0, 0, 0, P * ny, nx, nx};
  gemm(c, g2, 1);
}

struct RecParams {
  const double* rh;     // transformed local planes (ntl x nsp)
  const double* hh;     // transformed halo plane of node n0-1 (nullable)
  double* o;            // transformed output (ntl x nsp)
  const double* lam;    // nsp
  const double* chat;   // T(1), nsp
  const double* gam;    // gamma_0 .. gamma_{Nt+1} (nullable: one-level)
  double ms, inv_ms;
  int nsp, m, n0, s0, ndl;
};

// one thread per (local subdomain, mode)
__global__ void rasq_modes_kernel(RecParams P) {
  const int64_t total = int64_t(P.ndl) * P.nsp;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int sl = int(t / P.nsp), q = int(t - int64_t(sl) * P.nsp);
    const int s = P.s0 + sl;
    const int first = s == 0 ? 1 : s * P.m;
    const int last = (s + 1) * P.m;
    const int ofirst = s == 0 ? 1 : s * P.m + 1;
    const double lam = P.lam[q];
    const double rho = 1.0 / lam;
    const double ch = P.gam ? P.chat[q] : 0.0;
    double y = 0.0;
    for (int n = first; n <= last; ++n) {
      double rv = n < P.n0 ? P.hh[q] : P.rh[int64_t(n - P.n0) * P.nsp + q];
      if (P.gam) {
        // T(Shat y_c)_n = c^ (g_n lam^2 - g_{n+1} lam + [n>1](g_n - g_{n-1} lam)) / ms
        const double gn = P.gam[n], gp = P.gam[n + 1], gm = P.gam[n - 1];
        double sh = gn * lam * lam - gp * lam;
        if (n != 1) sh += gn - gm * lam;
        rv -= ch * sh * P.inv_ms;
      }
      y = rho * (rv + y);
      if (n >= ofirst) P.o[int64_t(n - P.n0) * P.nsp + q] = P.ms * y;
    }
    double x = 0.0;
    for (int n = last; n >= ofirst; --n) {
      double* op = P.o + int64_t(n - P.n0) * P.nsp + q;
      x = rho * (*op + x);
      *op = P.gam ? x + P.gam[n] * ch : x;
    }
  }
}

}  // namespace

// only the opt-in mode: the sine matrices alone do not enable it (the per-dof coarse solve of
// coarse_kron.cu builds them too, and keeps the LU sweep)
bool spectral_enabled(const Ctx* c) { return c->spectral && c->sp_x.p != nullptr; }

void build_spectral(Ctx* c) {
  const int nx = c->nx, ny = c->ny, nsp = c->nsp;
  auto sine = [](int n) {
    std::vector<double> S(size_t(n) * n);
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double f = std::sqrt(2.0L / (n + 1));
    for (int k = 0; k < n; ++k)
      for (int i = 0; i < n; ++i)
        S[size_t(k) * n + i] = double(f * std::sin(pi * (long double)((k + 1) * (i + 1) % (2 * (n + 1))) / (n + 1)));
    return S;
  };
  const std::vector<double> Sx = sine(nx), Sy = sine(ny);
  std::vector<double> lam(nsp), chat(nsp);
  {
    const long double pi = 3.141592653589793238462643383279502884L;
    std::vector<long double> cxs(nx), cys(ny), sx(nx, 0.0L), sy(ny, 0.0L);
    for (int k = 0; k < nx; ++k) {
      cxs[k] = std::cos(pi * (k + 1) / (nx + 1));
      for (int i = 0; i < nx; ++i) sx[k] += (long double)Sx[size_t(k) * nx + i];
    }
    for (int l = 0; l < ny; ++l) {
      cys[l] = std::cos(pi * (l + 1) / (ny + 1));
      for (int j = 0; j < ny; ++j) sy[l] += (long double)Sy[size_t(l) * ny + j];
    }
    for (int l = 0; l < ny; ++l)
      for (int k = 0; k < nx; ++k) {
        const long double v = (long double)c->Ahat.diag + 2.0L * c->Ahat.mcx * cxs[k] +
                              (ny > 1 ? 2.0L * c->Ahat.mcy * cys[l] : 0.0L);
        lam[size_t(l) * nx + k] = double(v);
        chat[size_t(l) * nx + k] = double(sy[l] * sx[k]);
      }
  }
  auto up = [&](DBuf<double>& d, const std::vector<double>& h) {
    d.alloc(h.size());
    KKT_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream));
  };
  up(c->sp_x, Sx);
  up(c->sp_y, Sy);
  up(c->sp_lam, lam);
  up(c->sp_chat, chat);
  c->sp_halo.alloc(3 * size_t(nsp));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
}

// P planes (ny x nx each, contiguous): out = Sy X Sx per plane; S is its own inverse.
void spectral_transform(Ctx* c, const double* in, double* tmp, double* out, int P) { transform(c, in, tmp, out, P); }

// out = RASQ(r) or, fused, RASQ(r - Shat y_c) + y_c (see sweep.cu rasq_apply).
void spectral_rasq(Ctx* c, const double* r, const double* halo_prev, double* out, bool fused) {
  const size_t B = size_t(c->B);
  if (c->sp_w1.n < B) c->sp_w1.alloc(B);
  if (c->sp_w2.n < B) c->sp_w2.alloc(B);
  double* w1 = c->sp_w1.p;
  double* w2 = c->sp_w2.p;
  const double* hh = nullptr;
  if (halo_prev) {
    transform(c, halo_prev, c->sp_halo.p, c->sp_halo.p + c->nsp, 1);
    hh = c->sp_halo.p + c->nsp;
  }
  c->tbegin(3);
  transform(c, r, w1, w2, c->ntl);                  // r^ in w2
  RecParams P;
  P.rh = w2;
  P.hh = hh;
  P.o = w1;
  P.lam = c->sp_lam.p;
  P.chat = c->sp_chat.p;
  P.gam = fused ? c->gam.p : nullptr;
  P.ms = c->ms;
  P.inv_ms = 1.0 / c->ms;
  P.nsp = c->nsp;
  P.m = c->m;
  P.n0 = c->n0;
  P.s0 = c->s0;
  P.ndl = c->ndl;
  const int64_t total = int64_t(c->ndl) * c->nsp;
  const int grid = int(std::min<int64_t>((total + 255) / 256, int64_t(kSmCount) * 16));
  KKT_LAUNCH(c, rasq_modes_kernel, grid, 256, 0, P);
  transform_sy_first(c, w1, w2, out, c->ntl);       // S o^ -> out
  c->tend(3);
}

}  // namespace kkt
