// stencil.cu — K1 (kkt_apply), the heat-operator blocks J/J^T/Jhat/Jhat^T,
// the diagonal blocks L/M_u/M_z, K8 (P^-1 u/z blocks) and Shat.
//
// The stencil kernels reproduce the reference's floating-point operation
// order in BOTH modes (band_row_strict, common.cuh): for a bandwidth-bound
// 5-point stencil the unfused mul/add costs nothing, and it makes K v bitwise
// equal to apply_K (kkt.cpp:50-65) — SURVEY.md §8a-5.
#include "ctx.cuh"

namespace kkt {
namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int threads = kThreads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = int64_t(kSmCount) * 16;
  return int(g < cap ? g : cap);
}

// out_n = S in_n - in_{n-1} (lower: apply_J / apply_Jhat, heat_operators.cpp:57-69,111-123)
// out_n = S in_n - in_{n+1} (upper: apply_JT / apply_JhatT, :71-83,125-137)
// post: optional division by `div` (apply_shat's t /= ms, schur.cpp:75).
template <bool kLower, bool kDiv>
__global__ void __launch_bounds__(kThreads) time_stencil_kernel(Stencil s, int nt, int nsp,
                                                                const double* __restrict__ in,
                                                                double* __restrict__ out,
                                                                double div) {
  const int64_t total = int64_t(nt) * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int n0 = int(idx / nsp);  // 0-based node
    const int p = int(idx - int64_t(n0) * nsp);
    const double* plane = in + int64_t(n0) * nsp;
    double acc = band_row_strict(s, plane, p);
    if (kLower) {
      if (n0 > 0) acc = ssub(acc, in[idx - nsp]);
    } else {
      if (n0 < nt - 1) acc = ssub(acc, in[idx + nsp]);
    }
    if (kDiv) acc = sdiv(acc, div);
    out[idx] = acc;
  }
}

template <bool kDivide>
__global__ void __launch_bounds__(kThreads) scale_kernel(int64_t n, const double* __restrict__ in,
                                                         double* __restrict__ out, double f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    out[i] = kDivide ? sdiv(in[i], f) : smul(f, in[i]);
  }
}

// K v for v = [u; z; w] (kkt.cpp:50-65), expression order kept:
//   ou = (A^T w_n - w_{n+1}) + ms*u      (:58-59)
//   oz = (omega*ms)*z - dt*w              (:61)
//   ow = (A u_n - u_{n-1}) - dt*z         (:63-64)
// With `bm` non-null the kernel writes bm - K v instead (the restart
// residual r = b - A x of gmres.cpp:50-51, same rounding as a separate pass).
__global__ void __launch_bounds__(kThreads) apply_K_kernel(Stencil s, int nt, int nsp, double ms,
                                                           double oms, double dt,
                                                           const double* __restrict__ v,
                                                           double* __restrict__ out,
                                                           const double* __restrict__ bm) {
  const int64_t B = int64_t(nt) * nsp;
  const double* u = v;
  const double* z = v + B;
  const double* w = v + 2 * B;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < B;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int n0 = int(idx / nsp);
    const int p = int(idx - int64_t(n0) * nsp);
    const int64_t off = int64_t(n0) * nsp;
    const double uu = u[idx], zz = z[idx], ww = w[idx];
    double ou = band_row_strict(s, w + off, p);
    if (n0 < nt - 1) ou = ssub(ou, w[idx + nsp]);
    ou = sadd(ou, smul(ms, uu));
    const double oz = ssub(smul(oms, zz), smul(dt, ww));
    double ow = band_row_strict(s, u + off, p);
    if (n0 > 0) ow = ssub(ow, u[idx - nsp]);
    ow = ssub(ow, smul(dt, zz));
    if (bm) {
      out[idx] = ssub(bm[idx], ou);
      out[idx + B] = ssub(bm[idx + B], oz);
      out[idx + 2 * B] = ssub(bm[idx + 2 * B], ow);
    } else {
      out[idx] = ou;
      out[idx + B] = oz;
      out[idx + 2 * B] = ow;
    }
  }
}

// apply_P_inv's diagonal blocks (kkt.cpp:76-79): divisions, as the reference.
__global__ void __launch_bounds__(kThreads) pinv_uz_kernel(int64_t B, double ms, double oms,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B;
       i += int64_t(gridDim.x) * blockDim.x) {
    out[i] = sdiv(r[i], ms);
    out[i + B] = sdiv(r[i + B], oms);
  }
}

}  // namespace

void op_time_stencil(Ctx* c, OpKind k, const double* in, double* out) {
  const int g = grid_for(c->B);
  switch (k) {
    case OpKind::J:
      KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->A, c->Nt, c->nsp, in, out, 1.0);
      break;
    case OpKind::JT:
      KKT_LAUNCH(c, (time_stencil_kernel<false, false>), g, kThreads, 0, c->A, c->Nt, c->nsp, in, out, 1.0);
      break;
    case OpKind::Jhat:
      KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->Ahat, c->Nt, c->nsp, in, out, 1.0);
      break;
    case OpKind::JhatT:
      KKT_LAUNCH(c, (time_stencil_kernel<false, false>), g, kThreads, 0, c->Ahat, c->Nt, c->nsp, in, out, 1.0);
      break;
  }
}

// Time-stencil over an arbitrary run of `nt` planes (the coarse build's
// windowed J^T / J passes, schur.cpp:333-357), optionally divided by `div`.
void op_time_stencil_n(Ctx* c, bool lower, const double* in, double* out, int nt, double div) {
  const int g = grid_for(int64_t(nt) * c->nsp);
  const bool d = div != 0.0;
  if (lower && d)
    KKT_LAUNCH(c, (time_stencil_kernel<true, true>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, div);
  else if (lower)
    KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, 1.0);
  else if (d)
    KKT_LAUNCH(c, (time_stencil_kernel<false, true>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, div);
  else
    KKT_LAUNCH(c, (time_stencil_kernel<false, false>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, 1.0);
}

void op_scale(Ctx* c, const double* in, double* out, double f, bool divide) {
  const int g = grid_for(c->B);
  if (divide)
    KKT_LAUNCH(c, scale_kernel<true>, g, kThreads, 0, c->B, in, out, f);
  else
    KKT_LAUNCH(c, scale_kernel<false>, g, kThreads, 0, c->B, in, out, f);
}

void op_apply_K(Ctx* c, const double* v, double* out, const double* b_minus) {
  KKT_LAUNCH(c, apply_K_kernel, grid_for(c->B), kThreads, 0, c->A, c->Nt, c->nsp, c->ms, c->oms,
             c->dt, v, out, b_minus);
}

void op_pinv_uz(Ctx* c, const double* r, double* out) {
  KKT_LAUNCH(c, pinv_uz_kernel, grid_for(c->B), kThreads, 0, c->B, c->ms, c->oms, r, out);
}

// apply_shat (schur.cpp:71-78): t = Jhat^T v; t /= ms; out = Jhat t.
void op_shat(Ctx* c, const double* v, double* out, double* tmp) {
  const int g = grid_for(c->B);
  KKT_LAUNCH(c, (time_stencil_kernel<false, true>), g, kThreads, 0, c->Ahat, c->Nt, c->nsp, v, tmp, c->ms);
  KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->Ahat, c->Nt, c->nsp, tmp, out, 1.0);
}

}  // namespace kkt
