// coarse_kron.cu — the per-dof Nicolaides coarse space beyond desk scale
// (the reference's default coarse_variant, config.hpp:47).
//
// The reference assembles S0 = Z^T Shat Z column by column (schur.cpp:266-398)
// and factors it with a banded LU of bandwidth ~3 n_sp (SparseLU -> BandedLU,
// linalg.cpp:312-331, schur.cpp:400-407): 63 s at config 0, ~600 GB at config 1.
// coarse_dof.cu reproduces that bitwise but stores S0 densely, which stops near
// dimension 1e4.  This file solves the SAME S0 from its structure.
//
// A per-dof column is (temporal profile of one subdomain) x (unit vector e_p):
// z_a,p = psi_a (x) e_p, psi_a = phi_{s,kind} on the owned nodes of s, zero
// elsewhere.  With (Jhat^T z)^n = Ahat z^n - z^{n+1} (heat_operators.cpp:125-137)
// and Shat = Jhat M^-1 Jhat^T, M = ms I (schur.cpp:71-78),
//   S0[(a,p),(b,p')] = <Jhat^T z_a,p , Jhat^T z_b,p'> / ms
//                    = ( T2[a,b] Ahat^2 + T1[a,b] Ahat + T0[a,b] I )[p,p'] / ms,
//   T2[a,b] =  sum_{n=1..Nt}   psi_a(n) psi_b(n)
//   T1[a,b] = -sum_{n=1..Nt-1} psi_a(n) psi_b(n+1) + psi_a(n+1) psi_b(n)
//   T0[a,b] =  sum_{n=2..Nt}   psi_a(n) psi_b(n)
// so S0 = (T2 (x) Ahat^2 + T1 (x) Ahat + T0 (x) I) / ms: every spatial factor is a
// polynomial in Ahat, and Ahat = S Lambda S with the 2-D sine transform S
// (spectral.cu: S symmetric, S^2 = I).  In that basis S0 is block diagonal: one
// D x D matrix M_q = (T2 lambda_q^2 + T1 lambda_q + T0) / ms per eigenmode q,
// D = dim / n_sp <= 2 Nd, symmetric positive definite and banded with
// half-bandwidth 3 (profiles of subdomains s, s' overlap after the one-node shift
// only for |s - s'| <= 1).  The solve is
//   c^ = (I (x) S) c;   M_q x_q = c^_q for every q;   c = (I (x) S) x,
// D plane transforms each way (fp64 tensor-core GEMMs against the resident sine
// matrices) and n_sp independent banded LDL^T solves, factored once at setup.
// It is a direct solve of the reference's S0, equal to its banded-LU solve to
// rounding (tests/test_gpu_perdof.py pins it against the compiled reference at
// config 0 and against the dense device path); it is used in FAST mode when the
// dense build does not fit, STRICT keeps the bitwise dense path.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>

#include "ctx.cuh"

namespace kkt {
void spectral_transform(Ctx* c, const double* in, double* tmp, double* out, int P);  // spectral.cu
void perdof_tables(Ctx* c, const std::vector<std::array<int, 2>>& col_start);        // coarse_dof.cu

namespace {

constexpr int kHB = 3;  // half-bandwidth of M_q

// LDL^T of M_q for every eigenmode q (one thread each).  W[(j*4 + t)*nsp + q]:
// t = 0 the pivot d_j, t = 1..3 the multipliers L[j+t][j].  Tb[(i*D + a)*4 + t] =
// T_i[a][a+t] (i = 0: T0, 1: T1, 2: T2).
__global__ void kron_factor_kernel(int D, int nsp, const double* __restrict__ lam, const double* __restrict__ Tb,
                                   double inv_ms, double tol, double* __restrict__ W, int* __restrict__ status) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsp) return;
  const double l = lam[q], l2 = l * l;
  auto Mq = [&](int a, int t) {  // M_q[a + t][a]
    const double* T0 = Tb + (size_t(0) * D + a) * 4 + t;
    const double* T1 = Tb + (size_t(1) * D + a) * 4 + t;
    const double* T2 = Tb + (size_t(2) * D + a) * 4 + t;
    return (T2[0] * l2 + T1[0] * l + T0[0]) * inv_ms;
  };
  auto Wd = [&](int j, int t) -> double& { return W[(size_t(j) * 4 + t) * nsp + q]; };
  for (int j = 0; j < D; ++j) {
    double dj = Mq(j, 0);
    for (int k = max(0, j - kHB); k < j; ++k) {
      const double ljk = Wd(k, j - k);
      dj -= ljk * ljk * Wd(k, 0);
    }
    if (!(dj > tol)) atomicMin(status, j);
    Wd(j, 0) = dj;
    for (int t = 1; t <= kHB; ++t) {
      const int i = j + t;
      double v = 0.0;
      if (i < D) {
        v = Mq(j, t);
        for (int k = max(0, i - kHB); k < j; ++k) v -= Wd(k, i - k) * Wd(k, j - k) * Wd(k, 0);
        v /= dj;
      }
      Wd(j, t) = v;
    }
  }
}

// x_q <- M_q^-1 x_q in place; x[(a*nsp) + q]
__global__ void kron_solve_kernel(int D, int nsp, const double* __restrict__ W, double* __restrict__ x) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsp) return;
  auto Wd = [&](int j, int t) { return W[(size_t(j) * 4 + t) * nsp + q]; };
  auto X = [&](int a) -> double& { return x[size_t(a) * nsp + q]; };
  for (int j = 0; j < D; ++j) {
    const double xj = X(j);
    for (int t = 1; t <= kHB && j + t < D; ++t) X(j + t) -= Wd(j, t) * xj;
  }
  for (int j = D - 1; j >= 0; --j) {
    double xj = X(j) / Wd(j, 0);
    for (int t = 1; t <= kHB && j + t < D; ++t) xj -= Wd(j, t) * X(j + t);
    X(j) = xj;
  }
}

}  // namespace

bool perdof_kron_wanted(const Ctx* c, double dense_bytes) {
  static const bool force = std::getenv("KKT_PERDOF_KRON") != nullptr;  // testing: also at desk scale
  return c->mode == KKT_MODE_FAST && (force || dense_bytes > 24e9);
}

// Called by build_coarse_perdof (coarse_dof.cu) with the profiles and columns in place.
void build_coarse_perdof_kron(Ctx* c, const std::vector<std::array<int, 2>>& col_start) {
  const int Nd = c->Nd, nsp = c->nsp, Nt = c->Nt;
  const int D = c->cdim / nsp;
  // planes a = 0..D-1 in column order; psi_a over global nodes
  std::vector<std::array<int, 2>> plane;  // (s, kind)
  for (int s = 0; s < Nd; ++s)
    for (int kind = 0; kind < 2; ++kind)
      if (col_start[s][kind] >= 0) plane.push_back({s, kind});
  if (int(plane.size()) != D) throw Error(KKT_EINVAL, "per-dof coarse planes do not match the column count");
  for (int a = 0; a < D; ++a)
    if (col_start[plane[a][0]][plane[a][1]] != a * nsp)
      throw Error(KKT_EINVAL, "per-dof coarse columns are not plane-contiguous");
  auto psi = [&](int a, int n) -> double {  // n: 1-based global node
    const int s = plane[a][0];
    const NodeRange ow = c->owned[s];
    if (n < ow.first || n > ow.last) return 0.0;
    const auto& phi = plane[a][1] == 0 ? c->phi_const[s] : c->phi_lin[s];
    return phi[n - ow.first];
  };
  std::vector<double> Tb(size_t(3) * D * 4, 0.0);
  for (int a = 0; a < D; ++a)
    for (int b = a; b < D; ++b) {
      const int sa = plane[a][0], sb = plane[b][0];
      if (std::abs(sa - sb) > 1) continue;
      const int lo = std::max(1, std::min(c->owned[sa].first, c->owned[sb].first) - 1);
      const int hi = std::min(Nt, std::max(c->owned[sa].last, c->owned[sb].last) + 1);
      double t2 = 0.0, t1 = 0.0, t0 = 0.0;
      for (int n = lo; n <= hi; ++n) {
        t2 += psi(a, n) * psi(b, n);
        if (n < Nt) t1 -= psi(a, n) * psi(b, n + 1) + psi(a, n + 1) * psi(b, n);
        if (n >= 2) t0 += psi(a, n) * psi(b, n);
      }
      if (t2 == 0.0 && t1 == 0.0 && t0 == 0.0) continue;
      if (b - a > kHB) throw Error(KKT_EINVAL, "per-dof coarse operator: temporal bandwidth above 3");
      Tb[(size_t(0) * D + a) * 4 + (b - a)] = t0;
      Tb[(size_t(1) * D + a) * 4 + (b - a)] = t1;
      Tb[(size_t(2) * D + a) * 4 + (b - a)] = t2;
    }
  if (!c->sp_x.p) build_spectral(c);  // sine matrices and Ahat's eigenvalues
  DBuf<double> dTb(Tb.size());
  KKT_CUDA(cudaMemcpyAsync(dTb.p, Tb.data(), sizeof(double) * Tb.size(), cudaMemcpyHostToDevice, c->stream));
  c->kron_w.alloc(size_t(D) * 4 * nsp);
  c->kron_tmp.alloc(size_t(2) * D * nsp);
  DBuf<int> status(1);
  const int big = 1 << 30;
  KKT_CUDA(cudaMemcpyAsync(status.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  // singularity threshold in the spirit of BandedLU's 1e-14 ||A||_inf: relative to the largest entry scale
  double tmax = 0.0;
  for (double v : Tb) tmax = std::max(tmax, std::abs(v));
  const double lmax = std::abs(c->Ahat.diag) + 2.0 * std::abs(c->Ahat.mcx) + 2.0 * std::abs(c->Ahat.mcy);
  const double tol = 1e-14 * tmax * std::max(1.0, lmax * lmax) / c->ms;
  KKT_LAUNCH(c, kron_factor_kernel, (nsp + 127) / 128, 128, 0, D, nsp, c->sp_lam.p, dTb.p, 1.0 / c->ms, tol,
             c->kron_w.p, status.p);
  int hst = big;
  KKT_CUDA(cudaMemcpyAsync(&hst, status.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  if (hst != big)
    throw Error(KKT_ECONFIG,
                "coarse operator (per-dof variant) is rank deficient: pivot below tolerance at coarse plane " +
                    std::to_string(hst), hst);
  c->kron = true;
  c->kron_D = D;
  c->h_S0.clear();
  perdof_tables(c, col_start);
}

void perdof_solve_kron(Ctx* c, double* cdev) {
  const int D = c->kron_D, nsp = c->nsp;
  double* hat = c->kron_tmp.p;
  double* tmp = hat + size_t(D) * nsp;
  spectral_transform(c, cdev, tmp, hat, D);
  KKT_LAUNCH(c, kron_solve_kernel, (nsp + 127) / 128, 128, 0, D, nsp, c->kron_w.p, hat);
  spectral_transform(c, hat, tmp, cdev, D);
}

}  // namespace kkt
