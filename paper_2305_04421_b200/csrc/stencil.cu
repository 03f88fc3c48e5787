// stencil.cu — K1 (kkt_apply), the heat-operator blocks J/J^T/Jhat/Jhat^T,
// the diagonal blocks L/M_u/M_z, K8 (P^-1 u/z blocks) and Shat.
//
// The stencil kernels reproduce the reference's floating-point operation
// order in BOTH modes (band_row_strict, common.cuh): for a bandwidth-bound
// 5-point stencil the unfused mul/add costs nothing, and it makes K v bitwise
// equal to apply_K (kkt.cpp:50-65) — SURVEY.md §8a-5.
#include <algorithm>
#include <cstdlib>

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
// `prev` / `next`: the neighbouring rank's plane beyond the slab (null at the
// global first / last node, where the reference has no coupling term).
template <bool kLower, bool kDiv>
__global__ void __launch_bounds__(kThreads) time_stencil_kernel(Stencil s, int nt, int nsp,
                                                                const double* __restrict__ in,
                                                                double* __restrict__ out,
                                                                double div,
                                                                const double* __restrict__ prev,
                                                                const double* __restrict__ next) {
  const int64_t total = int64_t(nt) * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int n0 = int(idx / nsp);  // 0-based node
    const int p = int(idx - int64_t(n0) * nsp);
    const double* plane = in + int64_t(n0) * nsp;
    double acc = band_row_strict(s, plane, p);
    if (kLower) {
      if (n0 > 0) acc = ssub(acc, in[idx - nsp]);
      else if (prev) acc = ssub(acc, prev[p]);
    } else {
      if (n0 < nt - 1) acc = ssub(acc, in[idx + nsp]);
      else if (next) acc = ssub(acc, next[p]);
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
//
// Traffic: the algorithmic minimum is 3 reads + 3 writes per point.  A CTA owns
// a kTX x kTY spatial tile (so the j-1 / j+1 rows of u and w are fetched once
// per kTY rows, and merge in L1 with the neighbouring threads' own loads) and
// marches over kTP (16 or 8) consecutive time nodes: u_{n-1} stays in a register from the
// previous node, and w_{n+1}, loaded for node n, is node n+1's own w value, so
// the time neighbours cost no second pass over u and w.
constexpr int kTX = 64, kTY = 4;
template <int kTP>
__global__ void __launch_bounds__(kTX * kTY) apply_K_kernel(Stencil s, int nt, int nsp, double ms,
                                                            double oms, double dt,
                                                            const double* __restrict__ v,
                                                            double* __restrict__ out,
                                                            const double* __restrict__ bm,
                                                            const double* __restrict__ u_prev,
                                                            const double* __restrict__ w_next) {
  const int i = blockIdx.x * kTX + (threadIdx.x & (kTX - 1));
  const int j = blockIdx.y * kTY + (threadIdx.x / kTX);
  if (i >= s.nx || j >= s.ny) return;
  const int p = j * s.nx + i;
  const int64_t B = int64_t(nt) * nsp;
  const double* u = v;
  const double* z = v + B;
  const double* w = v + 2 * B;
  const int nA = blockIdx.z * kTP, nB = min(nt, nA + kTP);
  // time neighbours carried across the march
  double up = 0.0, ww = w[int64_t(nA) * nsp + p];
  bool has_up = false;
  if (nA > 0) {
    up = u[int64_t(nA - 1) * nsp + p];
    has_up = true;
  } else if (u_prev) {
    up = u_prev[p];
    has_up = true;
  }
  for (int n0 = nA; n0 < nB; ++n0) {
    const int64_t off = int64_t(n0) * nsp;
    const int64_t idx = off + p;
    double wn = 0.0;
    bool has_wn = false;
    if (n0 < nt - 1) {
      wn = w[idx + nsp];
      has_wn = true;
    } else if (w_next) {
      wn = w_next[p];
      has_wn = true;
    }
    const double uu = u[idx], zz = z[idx];
    double ou = band_row_strict_ij(s, w + off, p, i, j);
    if (has_wn) ou = ssub(ou, wn);
    ou = sadd(ou, smul(ms, uu));
    const double oz = ssub(smul(oms, zz), smul(dt, ww));
    double ow = band_row_strict_ij(s, u + off, p, i, j);
    if (has_up) ow = ssub(ow, up);
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
    up = uu;
    has_up = true;
    ww = wn;
  }
}

// apply_P_inv's diagonal blocks (kkt.cpp:76-79): divisions, as the reference.
__global__ void __launch_bounds__(kThreads) pinv_uz_kernel(int64_t B, int64_t i0, int64_t i1, double ms, double oms,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ out) {
  for (int64_t i = i0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < i1;
       i += int64_t(gridDim.x) * blockDim.x) {
    out[i] = sdiv(r[i], ms);
    out[i + B] = sdiv(r[i + B], oms);
  }
}

// memset as a kernel: a cudaMemsetAsync may be scheduled on a copy engine, where it queues behind
// whatever bulk host transfer another stream has in flight (kkt_apply_P_inv_host's uploads)
__global__ void __launch_bounds__(kThreads) fill_words_kernel(int64_t n, unsigned word, unsigned* __restrict__ p) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) p[i] = word;
}
__global__ void __launch_bounds__(kThreads) fill_quads_kernel(int64_t n, unsigned word, uint4* __restrict__ p) {
  const uint4 v = make_uint4(word, word, word, word);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) p[i] = v;
}

}  // namespace

Halo exchange_halo(Ctx* c, const double* v, int slot_prev, int slot_next, bool want_prev,
                   bool want_next) {
  Halo h{nullptr, nullptr};
  if (c->nranks == 1) return h;
  const size_t nsp = c->nsp;
  double* hp = c->halo.p + size_t(slot_prev) * nsp;
  double* hn = c->halo.p + size_t(slot_next) * nsp;
  // every rank that wants its `next` plane receives it from rank+1, which sends
  // its first plane backwards; `prev` planes travel forwards (last plane)
  c->comm->halo(want_next ? v : nullptr, want_next ? hn : nullptr,
                want_prev ? v + size_t(c->ntl - 1) * nsp : nullptr, want_prev ? hp : nullptr, nsp,
                c->stream);
  if (want_prev && c->rank > 0) h.prev = hp;
  if (want_next && c->rank + 1 < c->nranks) h.next = hn;
  return h;
}

void op_time_stencil(Ctx* c, OpKind k, const double* in, double* out) {
  const int g = grid_for(c->B);
  const bool lower = k == OpKind::J || k == OpKind::Jhat;
  const Halo h = exchange_halo(c, in, 0, 1, lower, !lower);
  switch (k) {
    case OpKind::J:
      KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->A, c->ntl, c->nsp, in, out, 1.0, h.prev, nullptr);
      break;
    case OpKind::JT:
      KKT_LAUNCH(c, (time_stencil_kernel<false, false>), g, kThreads, 0, c->A, c->ntl, c->nsp, in, out, 1.0, nullptr, h.next);
      break;
    case OpKind::Jhat:
      KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->Ahat, c->ntl, c->nsp, in, out, 1.0, h.prev, nullptr);
      break;
    case OpKind::JhatT:
      KKT_LAUNCH(c, (time_stencil_kernel<false, false>), g, kThreads, 0, c->Ahat, c->ntl, c->nsp, in, out, 1.0, nullptr, h.next);
      break;
  }
}

// Time-stencil over an arbitrary run of `nt` planes (the coarse build's
// windowed J^T / J passes, schur.cpp:333-357), optionally divided by `div`.
void op_time_stencil_n(Ctx* c, bool lower, const double* in, double* out, int nt, double div) {
  const int g = grid_for(int64_t(nt) * c->nsp);
  const bool d = div != 0.0;
  if (lower && d)
    KKT_LAUNCH(c, (time_stencil_kernel<true, true>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, div, nullptr, nullptr);
  else if (lower)
    KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, 1.0, nullptr, nullptr);
  else if (d)
    KKT_LAUNCH(c, (time_stencil_kernel<false, true>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, div, nullptr, nullptr);
  else
    KKT_LAUNCH(c, (time_stencil_kernel<false, false>), g, kThreads, 0, c->Ahat, nt, c->nsp, in, out, 1.0, nullptr, nullptr);
}

void op_scale(Ctx* c, const double* in, double* out, double f, bool divide) {
  const int g = grid_for(c->B);
  if (divide)
    KKT_LAUNCH(c, scale_kernel<true>, g, kThreads, 0, c->B, in, out, f);
  else
    KKT_LAUNCH(c, scale_kernel<false>, g, kThreads, 0, c->B, in, out, f);
}

// K v on the rank's slab: u needs the plane of node n0-1 (from rank-1), w the
// plane of node n0+ntl (from rank+1).
void op_apply_K(Ctx* c, const double* v, double* out, const double* b_minus) {
  const double* u = v;
  const double* w = v + 2 * c->B;
  Halo h{nullptr, nullptr};
  if (c->nranks > 1) {
    const size_t nsp = c->nsp;
    double* hp = c->halo.p;
    double* hn = c->halo.p + nsp;
    c->comm->halo(w, hn, u + size_t(c->ntl - 1) * nsp, hp, nsp, c->stream);
    if (c->rank > 0) h.prev = hp;
    if (c->rank + 1 < c->nranks) h.next = hn;
  }
  // nodes per march (compile-time so that the march unrolls): 16, or 8 when 16 would leave the grid
  // with too few CTAs to fill the device several times over (config 1)
  const int tiles = ((c->nx + kTX - 1) / kTX) * ((c->ny + kTY - 1) / kTY);
  static const int force_tp = std::getenv("KKT_K1_TP") ? std::atoi(std::getenv("KKT_K1_TP")) : 0;
  const bool small = force_tp ? force_tp < 16 : int64_t(tiles) * ((c->ntl + 15) / 16) < int64_t(kSmCount) * 32;
  const int tp = small ? 8 : 16;
  const dim3 gK((c->nx + kTX - 1) / kTX, (c->ny + kTY - 1) / kTY, (c->ntl + tp - 1) / tp);
  if (small)
    KKT_LAUNCH(c, apply_K_kernel<8>, gK, kTX * kTY, 0, c->A, c->ntl, c->nsp, c->ms, c->oms, c->dt, v, out,
               b_minus, h.prev, h.next);
  else
    KKT_LAUNCH(c, apply_K_kernel<16>, gK, kTX * kTY, 0, c->A, c->ntl, c->nsp, c->ms, c->oms, c->dt, v, out,
               b_minus, h.prev, h.next);
}

void op_pinv_uz(Ctx* c, const double* r, double* out) {
  KKT_LAUNCH(c, pinv_uz_kernel, grid_for(c->B), kThreads, 0, c->B, int64_t(0), c->B, c->ms, c->oms, r, out);
}

void op_pinv_uz_range(Ctx* c, const double* r, double* out, int64_t i0, int64_t i1) {
  if (i1 > i0) KKT_LAUNCH(c, pinv_uz_kernel, grid_for(i1 - i0), kThreads, 0, c->B, i0, i1, c->ms, c->oms, r, out);
}

void dev_fill(Ctx* c, void* p, int byte, size_t nbytes) {
  if (nbytes % 4 != 0 || reinterpret_cast<uintptr_t>(p) % 4 != 0) throw Error(KKT_EINVAL, "dev_fill: 4-byte granularity");
  const unsigned b = unsigned(byte) & 0xFFu, word = b | (b << 8) | (b << 16) | (b << 24);
  if (nbytes == 0) return;
  if (nbytes % 16 == 0 && reinterpret_cast<uintptr_t>(p) % 16 == 0)
    KKT_LAUNCH(c, fill_quads_kernel, grid_for(int64_t(nbytes / 16)), kThreads, 0, int64_t(nbytes / 16), word, static_cast<uint4*>(p));
  else
    KKT_LAUNCH(c, fill_words_kernel, grid_for(int64_t(nbytes / 4)), kThreads, 0, int64_t(nbytes / 4), word, static_cast<unsigned*>(p));
}

// apply_shat (schur.cpp:71-78): t = Jhat^T v; t /= ms; out = Jhat t.  On a
// slab, t at node n0-1 is recomputed from the received v plane so the lower
// pass has its coupling term.
void op_shat(Ctx* c, const double* v, double* out, double* tmp) {
  const int g = grid_for(c->B);
  const Halo hv = exchange_halo(c, v, 0, 1, true, true);
  KKT_LAUNCH(c, (time_stencil_kernel<false, true>), g, kThreads, 0, c->Ahat, c->ntl, c->nsp, v, tmp, c->ms, nullptr, hv.next);
  const double* tprev = nullptr;
  if (hv.prev) {
    double* tp = c->halo.p + 2 * size_t(c->nsp);
    KKT_LAUNCH(c, (time_stencil_kernel<false, true>), grid_for(c->nsp), kThreads, 0, c->Ahat, 1, c->nsp, hv.prev, tp, c->ms, nullptr, v);
    tprev = tp;
  }
  KKT_LAUNCH(c, (time_stencil_kernel<true, false>), g, kThreads, 0, c->Ahat, c->ntl, c->nsp, tmp, out, 1.0, tprev, nullptr);
}

}  // namespace kkt
