// coarse_dof.cu — the per-dof Nicolaides coarse space (the reference's
// default coarse_variant, config.hpp:47; schur.cpp:266-413) on the device.
//
// Columns are (subdomain, profile kind, spatial dof): dim = 2*Nd*n_sp.  S0 is
// assembled exactly as the reference does it — for every column the windowed
// Jhat^T -> /ms -> Jhat passes (all n_sp columns of a (subdomain, kind) batched
// as independent windows), then the sequential inner products with the
// neighbouring subdomains' columns (schur.cpp:368-395) — stored densely, and
// turned into the reference's banded matrix (SparseLU::to_banded,
// linalg.cpp:312-331: kl, ku from the non-zero pattern).  The banded LU with
// partial pivoting (BandedLU, linalg.cpp:69-125) runs as one pivot/scale CTA
// plus one grid-wide rank-1 update per column, preserving the reference's
// per-entry operation order, so the factor is bitwise identical; the solve is
// the reference's column-oriented substitution over a shared-memory copy of
// the right-hand side.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>

#include "ctx.cuh"

namespace kkt {
namespace {

constexpr int kT = 256;

int grid_for(int64_t n) {
  int64_t g = (n + kT - 1) / kT;
  const int64_t cap = int64_t(kSmCount) * 32;
  return int(g < cap ? g : cap);
}

// zwin for a batch of dof columns: window d (n_sp of them) has plane k equal
// to phi[k-off] at position d for off <= k < off+cnt, else 0.
__global__ void fill_dof_windows(int wlen, int nsp, int off, int cnt, const double* __restrict__ phi,
                                 double* __restrict__ z) {
  const int64_t total = int64_t(nsp) * wlen * nsp;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t wp = int64_t(wlen) * nsp;
    const int d = int(e / wp);
    const int64_t r = e - int64_t(d) * wp;
    const int k = int(r / nsp), p = int(r - int64_t(k) * nsp);
    z[e] = (p == d && k >= off && k < off + cnt) ? phi[k - off] : 0.0;
  }
}

// Batched windowed time stencil: `nwin` windows of `wlen` planes each; the
// time coupling never crosses a window boundary.  Reference order (common.cuh).
template <bool kLower, bool kDiv>
__global__ void window_stencil(Stencil s, int nwin, int wlen, int nsp, const double* __restrict__ in,
                               double* __restrict__ out, double div) {
  const int64_t total = int64_t(nwin) * wlen * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t plane = idx / nsp;
    const int p = int(idx - plane * nsp);
    const int k = int(plane % wlen);
    double acc = band_row_strict(s, in + plane * nsp, p);
    if (kLower) {
      if (k > 0) acc = ssub(acc, in[idx - nsp]);
    } else {
      if (k < wlen - 1) acc = ssub(acc, in[idx + nsp]);
    }
    if (kDiv) acc = sdiv(acc, div);
    out[idx] = acc;
  }
}

// S0[ri][ci] = sum_{k2 in owned(s2) and window} phi2[k2] * ywin_d[pos][d2]
// for the columns ci = cstart + d of one (s, kind) and the rows of one (s2, kind2).
__global__ void dof_entries(int nsp, int wlen, int e0, int e1, int of2, int oc2,
                            const double* __restrict__ phi2, const double* __restrict__ y,
                            int cstart, int rstart, int dim, double* __restrict__ S0) {
  const int64_t total = int64_t(nsp) * nsp;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int d = int(e / nsp), d2 = int(e - int64_t(d) * nsp);
    const double* yw = y + int64_t(d) * wlen * nsp;
    double acc = 0.0;
    for (int k2 = 0; k2 < oc2; ++k2) {
      const int n2 = of2 + k2;
      if (n2 < e0 || n2 > e1) continue;
      acc = sadd(acc, smul(phi2[k2], yw[int64_t(n2 - e0) * nsp + d2]));
    }
    S0[int64_t(rstart + d2) * dim + (cstart + d)] = acc;
  }
}

__global__ void band_extent(int dim, const double* __restrict__ S0, int* kl_ku) {
  const int64_t total = int64_t(dim) * dim;
  int kl = 0, ku = 0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    if (S0[e] != 0.0) {
      const int i = int(e / dim), j = int(e - int64_t(i) * dim);
      kl = max(kl, i - j);
      ku = max(ku, j - i);
    }
  }
  atomicMax(&kl_ku[0], kl);
  atomicMax(&kl_ku[1], ku);
}

// band storage of the fill-extended factor: entry(i,j) at ab[j*ld + i-j+kuf]
__global__ void to_band(int dim, int kl, int ku, int kuf, int ld, const double* __restrict__ S0,
                        double* __restrict__ ab) {
  const int64_t total = int64_t(dim) * ld;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(t / ld);
    const int i = int(t - int64_t(j) * ld) + j - kuf;
    double v = 0.0;
    if (i >= 0 && i < dim && i - j <= kl && j - i <= ku) v = S0[int64_t(i) * dim + j];
    ab[t] = v == 0.0 ? 0.0 : v;  // dropped zeros (schur.cpp:392) are +0
  }
}

// BandedLU step j, part 1 (one CTA): first-maximum pivot search, row swap over
// columns j..jmax, column scaling by division (linalg.cpp:89-110).
__global__ void __launch_bounds__(1024) lu_pivot_step(int j, int n, int kl, int kuf, int ld, double tol,
                                                      double* ab, int* piv, int* status) {
  __shared__ double s_best[32];
  __shared__ int s_idx[32];
  __shared__ int s_p;
  __shared__ double s_v;
  if (*status >= 0) return;  // an earlier column was singular: stop factoring
  auto E = [&](int i, int jj) -> double& { return ab[int64_t(jj) * ld + (i - jj + kuf)]; };
  const int imax = min(n - 1, j + kl), jmax = min(n - 1, j + kuf);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double best = -1.0;
  int bidx = 0x7fffffff;
  for (int i = j + tid; i <= imax; i += blockDim.x) {
    const double v = fabs(E(i, j));
    if (v > best || (v == best && i < bidx)) { best = v; bidx = i; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const int oi = __shfl_down_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  if (lane == 0) { s_best[wid] = best; s_idx[wid] = bidx; }
  __syncthreads();
  if (wid == 0) {
    best = lane < int(blockDim.x >> 5) ? s_best[lane] : -1.0;
    bidx = lane < int(blockDim.x >> 5) ? s_idx[lane] : 0x7fffffff;
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if (lane == 0) { s_p = bidx; s_v = best; }
  }
  __syncthreads();
  const int p = s_p;
  if (!(s_v > tol)) {
    if (tid == 0) *status = j;
    return;
  }
  if (tid == 0) piv[j] = p;
  if (p != j) {
    for (int c = j + tid; c <= jmax; c += blockDim.x) {
      const double a = E(j, c);
      E(j, c) = E(p, c);
      E(p, c) = a;
    }
    __syncthreads();
  }
  const double d = E(j, j);
  for (int i = j + 1 + tid; i <= imax; i += blockDim.x) E(i, j) = sdiv(E(i, j), d);
}

// part 2 (grid): rank-1 update of columns j+1..jmax, rows j+1..imax, skipping u_jc == 0
__global__ void lu_update_step(int j, int n, int kl, int kuf, int ld, double* ab, const int* status) {
  if (*status >= 0) return;
  const int imax = min(n - 1, j + kl), jmax = min(n - 1, j + kuf);
  const int rows = imax - j, cols = jmax - j;
  const int64_t pairs = int64_t(rows) * cols;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < pairs;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int cc = int(t / rows), r = int(t - int64_t(cc) * rows);
    const int c = j + 1 + cc, i = j + 1 + r;
    double* colc = ab + int64_t(c) * ld;
    const double ujc = colc[j - c + kuf];
    if (ujc != 0.0) {
      const double lij = ab[int64_t(j) * ld + (i - j + kuf)];
      colc[i - c + kuf] = ssub(colc[i - c + kuf], smul(lij, ujc));
    }
  }
}

// BandedLU::solve_in_place (linalg.cpp:127-145), b in shared memory, one CTA.
__global__ void __launch_bounds__(1024) band_solve_general(int n, int kl, int kuf, int ld,
                                                           const double* __restrict__ ab,
                                                           const int* __restrict__ piv, double* b) {
  extern __shared__ double sb[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sb[i] = b[i];
  __syncthreads();
  auto E = [&](int i, int jj) { return ab[int64_t(jj) * ld + (i - jj + kuf)]; };
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0 && piv[j] != j) {
      const double t = sb[j];
      sb[j] = sb[piv[j]];
      sb[piv[j]] = t;
    }
    __syncthreads();
    const double bj = sb[j];
    if (bj != 0.0) {
      const int hi = min(n - 1, j + kl);
      for (int i = j + 1 + threadIdx.x; i <= hi; i += blockDim.x) sb[i] = ssub(sb[i], smul(E(i, j), bj));
    }
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {
    if (threadIdx.x == 0) sb[j] = sdiv(sb[j], E(j, j));
    __syncthreads();
    const double bj = sb[j];
    if (bj != 0.0) {
      const int lo = max(0, j - kuf);
      for (int i = lo + threadIdx.x; i < j; i += blockDim.x) sb[i] = ssub(sb[i], smul(E(i, j), bj));
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = sb[i];
}

// c[ci] = sum_k phi[k] r[n_k, dof] for this rank's columns (schur.cpp:196-199)
__global__ void dof_restrict(int cdim, int nsp, int m_max, int n0, int cl0, int cl1,
                             const int* __restrict__ col_first, const int* __restrict__ col_count,
                             const double* __restrict__ col_phi, const double* __restrict__ r,
                             double* __restrict__ c) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= cdim) return;
  double acc = 0.0;
  if (ci >= cl0 && ci < cl1) {
    const int d = ci % nsp;  // columns of a (subdomain, kind) are dof-contiguous
    const int first = col_first[ci], cnt = col_count[ci];
    const double* phi = col_phi + int64_t(ci / nsp) * m_max;
    for (int k = 0; k < cnt; ++k)
      acc = sadd(acc, smul(phi[k], r[int64_t(first + k - n0) * nsp + d]));
  }
  c[ci] = acc;
}

// out[n,p] = (out + phi_0 c_(s,0,p)) + phi_1 c_(s,1,p)  (prolong_add column order)
__global__ void dof_prolong_add(int ntl, int nsp, int n0, const int* __restrict__ node_col,
                                const double* __restrict__ node_phi, const double* __restrict__ c,
                                double* __restrict__ out) {
  const int64_t total = int64_t(ntl) * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int nl = int(idx / nsp), p = int(idx - int64_t(nl) * nsp);
    const int n0g = nl + n0 - 1;  // 0-based global node
    double o = out[idx];
    for (int k = 0; k < 2; ++k) {
      const int cs = node_col[2 * n0g + k];  // first column of (owner, kind)
      if (cs >= 0) o = sadd(o, smul(node_phi[2 * n0g + k], c[cs + p]));
    }
    out[idx] = o;
  }
}

__global__ void sum_ranks(int cdim, int nranks, const double* __restrict__ call, double* __restrict__ c) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= cdim) return;
  double acc = 0.0;
  for (int r = 0; r < nranks; ++r) acc += call[int64_t(r) * cdim + ci];
  c[ci] = acc;
}

template <class T>
void h2d(Ctx* c, DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(h.size());
  if (!h.empty())
    KKT_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace

bool perdof_kron_wanted(const Ctx* c, double dense_bytes);                                    // coarse_kron.cu
void build_coarse_perdof_kron(Ctx* c, const std::vector<std::array<int, 2>>& col_start);      // coarse_kron.cu
void perdof_solve_kron(Ctx* c, double* cdev);                                                  // coarse_kron.cu

// per-column / per-node tables of restrict and prolong (column ids of a (subdomain, kind) are
// dof-contiguous), and the work vectors
void perdof_tables(Ctx* c, const std::vector<std::array<int, 2>>& col_start) {
  (void)col_start;
  const int Nd = c->Nd, nsp = c->nsp, Nt = c->Nt, dim = c->cdim;
  c->m_max = 0;
  for (int s = 0; s < Nd; ++s) c->m_max = std::max(c->m_max, c->owned[s].count());
  std::vector<int> cf(dim), cc(dim);
  std::vector<double> cphi(size_t(dim / nsp) * c->m_max, 0.0);
  std::vector<int> ncol(2 * size_t(Nt), -1);
  std::vector<double> nphi(2 * size_t(Nt), 0.0);
  for (int ci = 0; ci < dim; ++ci) {
    const CoarseColumn& col = c->cols[ci];
    const auto& phi = col.kind == 0 ? c->phi_const[col.s] : c->phi_lin[col.s];
    cf[ci] = c->owned[col.s].first;
    cc[ci] = c->owned[col.s].count();
    if (col.dof == 0) {
      for (int k = 0; k < cc[ci]; ++k) {
        cphi[size_t(ci / nsp) * c->m_max + k] = phi[k];
        const int n = cf[ci] + k;
        ncol[2 * (n - 1) + col.kind] = ci;
        nphi[2 * (n - 1) + col.kind] = phi[k];
      }
    }
  }
  c->col_lo = dim;
  c->col_hi = 0;
  for (int ci = 0; ci < dim; ++ci) {
    const int sd = c->cols[ci].s;
    if (sd >= c->s0 && sd < c->s0 + c->ndl) {
      c->col_lo = std::min(c->col_lo, ci);
      c->col_hi = std::max(c->col_hi, ci + 1);
    }
  }
  if (c->col_hi < c->col_lo) c->col_lo = c->col_hi = 0;
  h2d(c, c->col_first, cf);
  h2d(c, c->col_count, cc);
  h2d(c, c->col_phi, cphi);
  h2d(c, c->node_col, ncol);
  h2d(c, c->node_phi, nphi);
  c->cvec.alloc(dim);
  c->call.alloc(size_t(dim) * c->nranks);
  c->gam.alloc(Nt + 2);
  c->has_coarse = true;
  c->perdof = true;
}

void build_coarse_perdof(Ctx* c) {
  const int Nd = c->Nd, nsp = c->nsp, Nt = c->Nt;
  c->phi_const.clear();
  c->phi_lin.clear();
  for (int s = 0; s < Nd; ++s) {
    const int ns = c->nodes[s].count();
    const int skip = c->owned[s].first - c->nodes[s].first;
    std::vector<double> lin(ns, 0.0);
    if (ns > 1)
      for (int k = 0; k < ns; ++k) lin[k] = -1.0 + 2.0 * k / (ns - 1);
    c->phi_const.emplace_back(ns - skip, 1.0);
    c->phi_lin.emplace_back(lin.begin() + skip, lin.end());
  }
  c->cols.clear();
  std::vector<std::array<int, 2>> col_start(Nd, {-1, -1});
  for (int s = 0; s < Nd; ++s)
    for (int kind = 0; kind < 2; ++kind) {
      const auto& phi = kind == 0 ? c->phi_const[s] : c->phi_lin[s];
      if (std::all_of(phi.begin(), phi.end(), [](double x) { return x == 0.0; })) continue;
      if (kind == 1 && c->owned[s].count() < 2) continue;
      col_start[s][kind] = int(c->cols.size());
      for (int p = 0; p < nsp; ++p) c->cols.push_back({s, kind, p});
    }
  const int dim = int(c->cols.size());
  if (dim == 0) throw Error(KKT_ECONFIG, "coarse space is empty");
  c->cdim = dim;
  int wmax = 0;
  for (int s = 0; s < Nd; ++s) {
    const int e0 = std::max(1, c->owned[s].first - 1), e1 = std::min(Nt, c->owned[s].last + 1);
    wmax = std::max(wmax, e1 - e0 + 1);
  }
  const double win_bytes = 3.0 * 8.0 * double(nsp) * wmax * nsp;
  const double dense_bytes = 8.0 * double(dim) * dim;
  if (perdof_kron_wanted(c, win_bytes + dense_bytes)) {  // FAST beyond desk scale: S0 from its Kronecker structure
    build_coarse_perdof_kron(c, col_start);
    return;
  }
  if (win_bytes + dense_bytes > 24e9)
    throw Error(KKT_EUNSUPPORTED,
                "per-dof coarse space too large for the device build (dim " + std::to_string(dim) +
                    "); the reference's banded LU of it is infeasible as well (SURVEY.md §8a-21)");
  DBuf<double> S0((size_t)dim * dim);
  KKT_CUDA(cudaMemsetAsync(S0.p, 0, sizeof(double) * S0.n, c->stream));
  {
    const size_t wn = size_t(nsp) * wmax * nsp;
    DBuf<double> z{wn}, t{wn}, y{wn}, dphi{size_t(wmax)}, dphi2{size_t(wmax)};
    for (int s = 0; s < Nd; ++s) {
      const NodeRange ow = c->owned[s];
      const int e0 = std::max(1, ow.first - 1), e1 = std::min(Nt, ow.last + 1);
      const int wlen = e1 - e0 + 1, off = ow.first - e0;
      const int64_t total = int64_t(nsp) * wlen * nsp;
      for (int kind = 0; kind < 2; ++kind) {
        if (col_start[s][kind] < 0) continue;
        const auto& phi = kind == 0 ? c->phi_const[s] : c->phi_lin[s];
        KKT_CUDA(cudaMemcpyAsync(dphi.p, phi.data(), sizeof(double) * phi.size(), cudaMemcpyHostToDevice, c->stream));
        KKT_LAUNCH(c, fill_dof_windows, grid_for(total), kT, 0, wlen, nsp, off, ow.count(), dphi.p, z.p);
        KKT_LAUNCH(c, (window_stencil<false, true>), grid_for(total), kT, 0, c->Ahat, nsp, wlen, nsp, z.p, t.p, c->ms);
        KKT_LAUNCH(c, (window_stencil<true, false>), grid_for(total), kT, 0, c->Ahat, nsp, wlen, nsp, t.p, y.p, 1.0);
        for (int s2 = std::max(0, s - 1); s2 <= std::min(Nd - 1, s + 1); ++s2) {
          for (int kind2 = 0; kind2 < 2; ++kind2) {
            if (col_start[s2][kind2] < 0) continue;
            const auto& phi2 = kind2 == 0 ? c->phi_const[s2] : c->phi_lin[s2];
            KKT_CUDA(cudaMemcpyAsync(dphi2.p, phi2.data(), sizeof(double) * phi2.size(), cudaMemcpyHostToDevice, c->stream));
            KKT_LAUNCH(c, dof_entries, grid_for(int64_t(nsp) * nsp), kT, 0, nsp, wlen, e0, e1,
                       c->owned[s2].first, c->owned[s2].count(), dphi2.p, y.p, col_start[s][kind],
                       col_start[s2][kind2], dim, S0.p);
            KKT_CUDA(cudaStreamSynchronize(c->stream));  // dphi2 is reused
          }
        }
        KKT_CUDA(cudaStreamSynchronize(c->stream));
      }
    }
  }
  // ---- dense copy for kkt_coarse_matrix (the reference's dense limit: 4096)
  if (dim <= 4096 || std::getenv("KKT_KEEP_S0")) {  // KKT_KEEP_S0: diagnostics only
    c->h_S0.resize(size_t(dim) * dim);
    KKT_CUDA(cudaMemcpyAsync(c->h_S0.data(), S0.p, sizeof(double) * S0.n, cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
  } else {
    c->h_S0.clear();
  }
  // ---- band storage + banded LU with partial pivoting (SparseLU)
  DBuf<int> klku(2);
  KKT_CUDA(cudaMemsetAsync(klku.p, 0, sizeof(int) * 2, c->stream));
  KKT_LAUNCH(c, band_extent, grid_for(int64_t(dim) * dim), kT, 0, dim, S0.p, klku.p);
  int hk[2];
  KKT_CUDA(cudaMemcpyAsync(hk, klku.p, sizeof(hk), cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
  const int kl = hk[0], ku = hk[1];
  const int kuf = std::min(dim - 1, kl + ku);
  const int ld = kl + kuf + 1;
  c->cb_kl = kl;
  c->cb_kuf = kuf;
  c->cb_ld = ld;
  c->cb_ab.alloc(size_t(dim) * ld);
  c->cb_piv.alloc(dim);
  KKT_LAUNCH(c, to_band, grid_for(int64_t(dim) * ld), kT, 0, dim, kl, ku, kuf, ld, S0.p, c->cb_ab.p);
  // ||A||_inf of the banded matrix (linalg.cpp:35-43), host from the dense copy
  double anorm = 0.0;
  {
    std::vector<double> rowsum(dim, 0.0);
    std::vector<double> hs(size_t(dim) * dim);
    KKT_CUDA(cudaMemcpyAsync(hs.data(), S0.p, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < dim; ++i) {
      double row = 0.0;
      for (int j = std::max(0, i - kl); j <= std::min(dim - 1, i + ku); ++j) row += std::abs(hs[size_t(i) * dim + j]);
      anorm = std::max(anorm, row);
    }
  }
  S0.release();
  const double tol = 1e-14 * anorm;
  DBuf<int> status(1);
  KKT_CUDA(cudaMemsetAsync(status.p, 0xff, sizeof(int), c->stream));  // -1
  const int ugrid = kSmCount * 8;
  for (int j = 0; j < dim; ++j) {
    KKT_LAUNCH(c, lu_pivot_step, 1, 1024, 0, j, dim, kl, kuf, ld, tol, c->cb_ab.p, c->cb_piv.p, status.p);
    KKT_LAUNCH(c, lu_update_step, ugrid, kT, 0, j, dim, kl, kuf, ld, c->cb_ab.p, status.p);
  }
  int hst = -1;
  KKT_CUDA(cudaMemcpyAsync(&hst, status.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  if (hst >= 0)
    throw Error(KKT_ECONFIG,
                "coarse operator (per-dof variant) is rank deficient: banded LU: pivot below tolerance "
                "at index " + std::to_string(hst), hst);
  perdof_tables(c, col_start);
}

void perdof_restrict(Ctx* c, const double* r, double* cdev) {
  double* dst = c->nranks > 1 ? c->cvec.p : cdev;
  KKT_LAUNCH(c, dof_restrict, (c->cdim + 255) / 256, 256, 0, c->cdim, c->nsp, c->m_max, c->n0, c->col_lo,
             c->col_hi, c->col_first.p, c->col_count.p, c->col_phi.p, r, dst);
  if (c->nranks > 1) {
    c->comm->allgather(c->cvec.p, c->call.p, size_t(c->cdim), c->stream);
    KKT_LAUNCH(c, sum_ranks, (c->cdim + 255) / 256, 256, 0, c->cdim, c->nranks, c->call.p, cdev);
  }
}

void perdof_solve(Ctx* c, double* cdev) {
  if (c->kron) return perdof_solve_kron(c, cdev);
  const size_t smem = sizeof(double) * size_t(c->cdim);
  static bool attr = false;
  if (!attr) {
    KKT_CUDA(cudaFuncSetAttribute(band_solve_general, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  if (smem > 200 * 1024) throw Error(KKT_EUNSUPPORTED, "per-dof coarse solve: dimension too large");
  KKT_LAUNCH(c, band_solve_general, 1, 1024, smem, c->cdim, c->cb_kl, c->cb_kuf, c->cb_ld, c->cb_ab.p,
             c->cb_piv.p, cdev);
}

void perdof_prolong_add(Ctx* c, const double* cdev, double* out) {
  KKT_LAUNCH(c, dof_prolong_add, grid_for(c->B), kT, 0, c->ntl, c->nsp, c->n0, c->node_col.p,
             c->node_phi.p, cdev, out);
}

}  // namespace kkt
