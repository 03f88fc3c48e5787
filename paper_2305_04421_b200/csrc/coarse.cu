// coarse.cu — the two-level coarse-in-time correction (K2-K4) and the
// Schur / P^-1 dispatch.
//
// Scalar Nicolaides coarse space (reference schur.cpp:166-413): per time
// subdomain a constant and a linear-ramp temporal profile, masked to owned
// nodes and lifted constantly over space.  S0 = Z^T Shat Z is assembled
// column by column with the reference's windowed Jhat^T -> /ms -> Jhat passes
// and node sums (same operation order), then factored on the device with the
// reference's dense LU (linalg.cpp:199-234).
//
// Per application: node sums of r (K3), one single-CTA kernel for
// c = Z^T r, S0^{-1} c and the per-node prolongation values gamma_n (K4), and
// either the reference's explicit residual r - Shat y_c (strict) or the
// analytic residual fused into the sweep (fast, sweep_fast.cu).
#include <algorithm>
#include <array>
#include <cmath>

#include "ctx.cuh"

namespace kkt {
namespace {

constexpr int kCoarseThreads = 1024;

// Sequential node sums (schur.cpp:193-196, :358-364): one thread per node.
__global__ void nodesum_seq_kernel(int nplanes, int nsp, const double* __restrict__ x,
                                   double* __restrict__ out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nplanes) return;
  const double* p = x + int64_t(n) * nsp;
  double acc = 0.0;
  int i = 0;
  for (; i + 4 <= nsp; i += 4) {
    const double a = p[i], b = p[i + 1], c = p[i + 2], d = p[i + 3];
    acc = sadd(acc, a);
    acc = sadd(acc, b);
    acc = sadd(acc, c);
    acc = sadd(acc, d);
  }
  for (; i < nsp; ++i) acc = sadd(acc, p[i]);
  out[n] = acc;
}

// Fast node sums: one CTA per node, fixed-shape tree (deterministic).
__global__ void __launch_bounds__(256) nodesum_tree_kernel(int nsp, const double* __restrict__ x,
                                                           double* __restrict__ out) {
  __shared__ double part[8];
  const double* p = x + int64_t(blockIdx.x) * nsp;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nsp; i += blockDim.x) acc += p[i];
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    out[blockIdx.x] = s;
  }
}

struct CoarseTables {
  int cdim, Nt, m_max;
  int n0;                  // first local node (node sums are slab-local)
  int cl0, cl1;            // this rank's columns [cl0, cl1)
  int nranks;
  const int* col_first;
  const int* col_count;
  const double* col_phi;   // cdim * m_max
  const int* node_col;     // 2 per node (index n-1)
  const double* node_phi;  // 2 per node
  const double* lu;        // cdim * cdim row-major
  const int* piv;
};

// c = Z^T r from node sums (restrict_to_coarse, schur.cpp:181-204).  Only this
// rank's columns (its subdomains own their nodes); the others are zero and
// arrive through the all-gather.
__device__ void restrict_from_nodesums(const CoarseTables& T, const double* ns, double* c) {
  for (int ci = threadIdx.x; ci < T.cdim; ci += blockDim.x) {
    double acc = 0.0;
    if (ci >= T.cl0 && ci < T.cl1) {
      const int first = T.col_first[ci], cnt = T.col_count[ci];
      const double* phi = T.col_phi + int64_t(ci) * T.m_max;
      for (int k = 0; k < cnt; ++k) acc = sadd(acc, smul(phi[k], ns[first + k - T.n0]));
    }
    c[ci] = acc;
  }
}

// every position is non-zero on exactly one rank: the rank-ordered sum is exact
__device__ void gather_columns(const CoarseTables& T, const double* call, double* c) {
  for (int ci = threadIdx.x; ci < T.cdim; ci += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < T.nranks; ++r) acc += call[int64_t(r) * T.cdim + ci];
    c[ci] = acc;
  }
}

// DenseLU::solve_in_place (linalg.cpp:236-249), threads over rows.
__device__ void lu_solve_block(const CoarseTables& T, double* b) {
  const int n = T.cdim;
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    if (threadIdx.x == 0 && T.piv[j] != j) {
      const double t = b[j];
      b[j] = b[T.piv[j]];
      b[T.piv[j]] = t;
    }
    __syncthreads();
    const double bj = b[j];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
      b[i] = ssub(b[i], smul(T.lu[int64_t(i) * n + j], bj));
  }
  for (int j = n - 1; j >= 0; --j) {
    __syncthreads();
    if (threadIdx.x == 0) b[j] = sdiv(b[j], T.lu[int64_t(j) * n + j]);
    __syncthreads();
    const double bj = b[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x)
      b[i] = ssub(b[i], smul(T.lu[int64_t(i) * n + j], bj));
  }
  __syncthreads();
}

// gamma_n = (0 + phi_0 c_0) + phi_1 c_1: prolong_add into zeros (schur.cpp:206-226).
__device__ void gamma_from_c(const CoarseTables& T, const double* c, double* gam) {
  for (int n = 1 + threadIdx.x; n <= T.Nt; n += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < 2; ++k) {
      const int ci = T.node_col[2 * (n - 1) + k];
      if (ci >= 0) acc = sadd(acc, smul(T.node_phi[2 * (n - 1) + k], c[ci]));
    }
    gam[n] = acc;
  }
  if (threadIdx.x == 0) {
    gam[0] = 0.0;
    gam[T.Nt + 1] = 0.0;
  }
}

// restrict + solve + prolongation values in one single-CTA launch.  With
// several ranks, `call` holds every rank's restricted columns (all-gathered)
// and `ns` is unused.
__global__ void __launch_bounds__(kCoarseThreads) coarse_gamma_kernel(CoarseTables T,
                                                                      const double* __restrict__ ns,
                                                                      const double* __restrict__ call,
                                                                      double* c, double* gam) {
  extern __shared__ double sb[];
  if (call)
    gather_columns(T, call, sb);
  else
    restrict_from_nodesums(T, ns, sb);
  __syncthreads();
  lu_solve_block(T, sb);
  for (int i = threadIdx.x; i < T.cdim; i += blockDim.x) c[i] = sb[i];
  gamma_from_c(T, sb, gam);
}

__global__ void __launch_bounds__(kCoarseThreads) coarse_restrict_kernel(CoarseTables T,
                                                                         const double* __restrict__ ns,
                                                                         double* c) {
  restrict_from_nodesums(T, ns, c);
}

__global__ void __launch_bounds__(kCoarseThreads) coarse_gather_kernel(CoarseTables T,
                                                                       const double* __restrict__ call,
                                                                       double* c) {
  gather_columns(T, call, c);
}

__global__ void __launch_bounds__(kCoarseThreads) coarse_solve_kernel(CoarseTables T, double* c) {
  extern __shared__ double sb[];
  for (int i = threadIdx.x; i < T.cdim; i += blockDim.x) sb[i] = c[i];
  __syncthreads();
  lu_solve_block(T, sb);
  for (int i = threadIdx.x; i < T.cdim; i += blockDim.x) c[i] = sb[i];
}

// out[n,p] = (out[n,p] + phi_0 c_0) + phi_1 c_1 (prolong_add column order).
__global__ void prolong_add_kernel(CoarseTables T, int ntl, int nsp, const double* __restrict__ c,
                                   double* __restrict__ out) {
  const int64_t total = int64_t(ntl) * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int n0 = int(idx / nsp) + T.n0 - 1;  // 0-based global node
    double o = out[idx];
    for (int k = 0; k < 2; ++k) {
      const int ci = T.node_col[2 * n0 + k];
      if (ci >= 0) o = sadd(o, smul(T.node_phi[2 * n0 + k], c[ci]));
    }
    out[idx] = o;
  }
}

// y_c materialised from gamma: yc[n,p] = gamma_n.
__global__ void broadcast_gamma_kernel(int nt, int nsp, int n0, const double* __restrict__ gam,
                                       double* __restrict__ out) {
  const int64_t total = int64_t(nt) * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x)
    out[idx] = gam[n0 + idx / nsp];
}

// out = a - b / out = a + b elementwise (schur.cpp:437, :439).
template <bool kSub>
__global__ void axpb_kernel(int64_t n, const double* a, const double* b, double* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = kSub ? ssub(a[i], b[i]) : sadd(a[i], b[i]);
}

// Zone filled with a masked profile: plane k of the window gets value
// phi[k - off] for off <= k < off + cnt, else 0 (schur.cpp:320-331).
__global__ void fill_profile_kernel(int wlen, int nsp, int off, int cnt,
                                    const double* __restrict__ phi, double* __restrict__ z) {
  const int64_t total = int64_t(wlen) * nsp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int k = int(idx / nsp);
    z[idx] = (k >= off && k < off + cnt) ? phi[k - off] : 0.0;
  }
}

// DenseLU::DenseLU (linalg.cpp:199-234), single CTA, reference order.
__global__ void __launch_bounds__(kCoarseThreads) dense_lu_kernel(int n, double tol, double* A,
                                                                  int* piv, int* status) {
  __shared__ int s_p;
  __shared__ double s_best;
  auto at = [&](int i, int j) -> double& { return A[int64_t(i) * n + j]; };
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      int p = j;
      double best = fabs(at(j, j));
      for (int i = j + 1; i < n; ++i) {
        if (fabs(at(i, j)) > best) {
          best = fabs(at(i, j));
          p = i;
        }
      }
      s_p = p;
      s_best = best;
      piv[j] = p;
    }
    __syncthreads();
    if (!(s_best > tol)) {
      if (threadIdx.x == 0) *status = j;
      return;
    }
    const int p = s_p;
    if (p != j) {
      for (int cc = threadIdx.x; cc < n; cc += blockDim.x) {
        const double t = at(j, cc);
        at(j, cc) = at(p, cc);
        at(p, cc) = t;
      }
    }
    __syncthreads();
    const double d = at(j, j);
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) at(i, j) = sdiv(at(i, j), d);
    __syncthreads();
    const int rows = n - j - 1;
    const int64_t pairs = int64_t(rows) * rows;
    for (int64_t t = threadIdx.x; t < pairs; t += blockDim.x) {
      const int i = j + 1 + int(t / rows);
      const int cc = j + 1 + int(t % rows);
      at(i, cc) = ssub(at(i, cc), smul(at(i, j), at(j, cc)));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = -1;
}

CoarseTables tables(Ctx* c) {
  CoarseTables T;
  T.cdim = c->cdim;
  T.Nt = c->Nt;
  T.m_max = c->m_max;
  T.col_first = c->col_first.p;
  T.col_count = c->col_count.p;
  T.col_phi = c->col_phi.p;
  T.node_col = c->node_col.p;
  T.node_phi = c->node_phi.p;
  T.lu = c->S0lu.p;
  T.piv = c->S0piv.p;
  T.n0 = c->n0;
  T.cl0 = c->col_lo;
  T.cl1 = c->col_hi;
  T.nranks = c->nranks;
  return T;
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = int64_t(kSmCount) * 16;
  return int(g < cap ? g : cap);
}

template <class T>
void h2d(Ctx* c, DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(h.size());
  if (!h.empty())
    KKT_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace

// ---------------------------------------------------------------------------
// build_coarse_space, scalar variant (schur.cpp:266-413)
// ---------------------------------------------------------------------------
void build_coarse(Ctx* c) {
  const int Nd = c->Nd, nsp = c->nsp, Nt = c->Nt;
  if (c->desc.coarse_variant != KKT_COARSE_SCALAR) {
    build_coarse_perdof(c);
    return;
  }
  c->phi_const.clear();
  c->phi_lin.clear();
  for (int s = 0; s < Nd; ++s) {
    const int ns = c->nodes[s].count();
    const int skip = c->owned[s].first - c->nodes[s].first;
    std::vector<double> lin(ns, 0.0);  // linear_profile (schur.cpp:167-173)
    if (ns > 1)
      for (int k = 0; k < ns; ++k) lin[k] = -1.0 + 2.0 * k / (ns - 1);
    c->phi_const.emplace_back(ns - skip, 1.0);
    c->phi_lin.emplace_back(lin.begin() + skip, lin.end());
  }
  c->cols.clear();
  std::vector<std::array<int, 2>> col_start(Nd, {-1, -1});
  for (int s = 0; s < Nd; ++s) {
    for (int kind = 0; kind < 2; ++kind) {
      const auto& phi = kind == 0 ? c->phi_const[s] : c->phi_lin[s];
      if (std::all_of(phi.begin(), phi.end(), [](double x) { return x == 0.0; })) continue;
      if (kind == 1 && c->owned[s].count() < 2) continue;
      col_start[s][kind] = int(c->cols.size());
      c->cols.push_back({s, kind, -1});
    }
  }
  const int dim = int(c->cols.size());
  if (dim == 0) throw Error(KKT_ECONFIG, "coarse space is empty");
  c->cdim = dim;

  // ---- S0 columns: windowed Jhat^T -> /ms -> Jhat, node sums, neighbour products
  std::vector<double> S0(size_t(dim) * dim, 0.0);
  int wmax = 0;
  for (int s = 0; s < Nd; ++s) {
    const int e0 = std::max(1, c->owned[s].first - 1);
    const int e1 = std::min(Nt, c->owned[s].last + 1);
    wmax = std::max(wmax, e1 - e0 + 1);
  }
  const size_t wplanes = size_t(wmax) * nsp;
  DBuf<double> zwin{wplanes}, twin{wplanes}, ywin{wplanes};
  DBuf<double> dphi{size_t(wmax)}, dns{size_t(wmax)};
  std::vector<double> ns_host(wmax);
  for (int s = 0; s < Nd; ++s) {
    const NodeRange ow = c->owned[s];
    const int e0 = std::max(1, ow.first - 1);
    const int e1 = std::min(Nt, ow.last + 1);
    const int wlen = e1 - e0 + 1;
    const int off = ow.first - e0;
    for (int kind = 0; kind < 2; ++kind) {
      if (col_start[s][kind] < 0) continue;
      const auto& phi = kind == 0 ? c->phi_const[s] : c->phi_lin[s];
      const int ci = col_start[s][kind];
      KKT_CUDA(cudaMemcpyAsync(dphi.p, phi.data(), sizeof(double) * phi.size(),
                               cudaMemcpyHostToDevice, c->stream));
      KKT_LAUNCH(c, fill_profile_kernel, grid_for(int64_t(wlen) * nsp), 256, 0, wlen, nsp, off,
                 ow.count(), dphi.p, zwin.p);
      op_time_stencil_n(c, false, zwin.p, twin.p, wlen, c->ms);  // Jhat^T z, /ms
      op_time_stencil_n(c, true, twin.p, ywin.p, wlen, 0.0);     // Jhat t
      KKT_LAUNCH(c, nodesum_seq_kernel, (wlen + 127) / 128, 128, 0, wlen, nsp, ywin.p, dns.p);
      KKT_CUDA(cudaMemcpyAsync(ns_host.data(), dns.p, sizeof(double) * wlen, cudaMemcpyDeviceToHost,
                               c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
      for (int s2 = std::max(0, s - 1); s2 <= std::min(Nd - 1, s + 1); ++s2) {
        const NodeRange ow2 = c->owned[s2];
        for (int kind2 = 0; kind2 < 2; ++kind2) {
          if (col_start[s2][kind2] < 0) continue;
          const auto& phi2 = kind2 == 0 ? c->phi_const[s2] : c->phi_lin[s2];
          const int ri = col_start[s2][kind2];
          double acc = 0.0;
          for (int k2 = 0; k2 < ow2.count(); ++k2) {
            const int n2 = ow2.first + k2;
            if (n2 < e0 || n2 > e1) continue;
            acc += phi2[k2] * ns_host[n2 - e0];
          }
          S0[size_t(ri) * dim + ci] = acc;
        }
      }
    }
  }
  c->h_S0 = S0;

  // ---- factor S0 (DenseLU), singular -> ConfigError (schur.cpp:400-411)
  double anorm = 0.0;
  for (int i = 0; i < dim; ++i) {
    double row = 0.0;
    for (int j = 0; j < dim; ++j) row += std::abs(S0[size_t(i) * dim + j]);
    anorm = std::max(anorm, row);
  }
  h2d(c, c->S0lu, S0);
  c->S0piv.alloc(dim);
  DBuf<int> st(1);
  KKT_LAUNCH(c, dense_lu_kernel, 1, kCoarseThreads, 0, dim, 1e-14 * anorm, c->S0lu.p, c->S0piv.p,
             st.p);
  int hst = 0;
  KKT_CUDA(cudaMemcpyAsync(&hst, st.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  if (hst >= 0)
    throw Error(KKT_ECONFIG,
                "coarse operator (scalar variant) is rank deficient: dense LU: pivot below "
                "tolerance at index " + std::to_string(hst), hst);

  // ---- per-column and per-node tables
  c->m_max = 0;
  for (int s = 0; s < Nd; ++s) c->m_max = std::max(c->m_max, c->owned[s].count());
  std::vector<int> cf(dim), cc(dim);
  std::vector<double> cphi(size_t(dim) * c->m_max, 0.0);
  std::vector<int> ncol(2 * size_t(Nt), -1);
  std::vector<double> nphi(2 * size_t(Nt), 0.0);
  for (int ci = 0; ci < dim; ++ci) {
    const CoarseColumn& col = c->cols[ci];
    const auto& phi = col.kind == 0 ? c->phi_const[col.s] : c->phi_lin[col.s];
    cf[ci] = c->owned[col.s].first;
    cc[ci] = c->owned[col.s].count();
    for (int k = 0; k < cc[ci]; ++k) {
      cphi[size_t(ci) * c->m_max + k] = phi[k];
      const int n = cf[ci] + k;
      ncol[2 * (n - 1) + col.kind] = ci;
      nphi[2 * (n - 1) + col.kind] = phi[k];
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
  c->nodesum.alloc(c->ntl);
  c->cvec.alloc(dim);
  c->call.alloc(size_t(dim) * c->nranks);
  c->gam.alloc(Nt + 2);
  dev_fill(c, c->gam.p, 0, sizeof(double) * (Nt + 2));

  // ---- a1 = Ahat 1, a2 = Ahat a1 (fast analytic Shat y_c)
  c->a1.alloc(nsp);
  c->a2.alloc(nsp);
  {
    std::vector<double> ones(nsp, 1.0);
    DBuf<double> d1(nsp);
    KKT_CUDA(cudaMemcpyAsync(d1.p, ones.data(), sizeof(double) * nsp, cudaMemcpyHostToDevice, c->stream));
    // one plane, no time coupling: Ahat v
    op_time_stencil_n(c, true, d1.p, c->a1.p, 1, 0.0);
    op_time_stencil_n(c, true, c->a1.p, c->a2.p, 1, 0.0);
    KKT_CUDA(cudaStreamSynchronize(c->stream));
  }
  c->has_coarse = true;
}

// ---------------------------------------------------------------------------
// per-application pieces
// ---------------------------------------------------------------------------
static void node_sums(Ctx* c, const double* r) {
  if (c->mode == KKT_MODE_STRICT || (c->bisect & 2))
    KKT_LAUNCH(c, nodesum_seq_kernel, (c->ntl + 127) / 128, 128, 0, c->ntl, c->nsp, r, c->nodesum.p);
  else
    KKT_LAUNCH(c, nodesum_tree_kernel, c->ntl, 256, 0, c->nsp, r, c->nodesum.p);
}

// restricted columns of this rank -> every rank's columns (all-gather)
static const double* gather_all(Ctx* c, double* local) {
  c->comm->allgather(local, c->call.p, size_t(c->cdim), c->stream);
  return c->call.p;
}

void coarse_restrict(Ctx* c, const double* r, double* cdev) {
  if (c->perdof) return perdof_restrict(c, r, cdev);
  node_sums(c, r);
  KKT_LAUNCH(c, coarse_restrict_kernel, 1, kCoarseThreads, 0, tables(c), c->nodesum.p,
             c->nranks > 1 ? c->cvec.p : cdev);
  if (c->nranks > 1)
    KKT_LAUNCH(c, coarse_gather_kernel, 1, kCoarseThreads, 0, tables(c), gather_all(c, c->cvec.p), cdev);
}

void coarse_solve(Ctx* c, double* cdev) {
  if (c->perdof) return perdof_solve(c, cdev);
  KKT_LAUNCH(c, coarse_solve_kernel, 1, kCoarseThreads, sizeof(double) * c->cdim, tables(c), cdev);
}

void coarse_prolong_add(Ctx* c, const double* cdev, double* out) {
  if (c->perdof) return perdof_prolong_add(c, cdev, out);
  KKT_LAUNCH(c, prolong_add_kernel, grid_for(c->B), 256, 0, tables(c), c->ntl, c->nsp, cdev, out);
}

void coarse_gamma(Ctx* c, const double* r) {
  node_sums(c, r);
  const double* call = nullptr;
  if (c->nranks > 1) {
    KKT_LAUNCH(c, coarse_restrict_kernel, 1, kCoarseThreads, 0, tables(c), c->nodesum.p, c->cvec.p);
    call = gather_all(c, c->cvec.p);
  }
  KKT_LAUNCH(c, coarse_gamma_kernel, 1, kCoarseThreads, sizeof(double) * c->cdim, tables(c),
             c->nodesum.p, call, c->cvec.p, c->gam.p);
}

static void ensure_tmp(Ctx* c) {
  if (c->tmpB1.n < size_t(c->B)) c->tmpB1.alloc(c->B);
  if (c->tmpB2.n < size_t(c->B)) c->tmpB2.alloc(c->B);
}

// apply_two_level (schur.cpp:415-444).
void two_level_apply(Ctx* c, const double* r, double* out, int form) {
  if (!c->has_coarse) throw Error(KKT_ECONFIG, "two-level apply: no coarse space");
  ensure_tmp(c);
  double* yc = c->tmpB1.p;
  const int g = grid_for(c->B);
  if (c->perdof) {
    // y_c = prolong_add(S0^{-1} restrict(r)) into zeros (schur.cpp:421-424)
    coarse_restrict(c, r, c->cvec.p);
    perdof_solve(c, c->cvec.p);
    dev_fill(c, yc, 0, sizeof(double) * c->B);
    perdof_prolong_add(c, c->cvec.p, yc);
  } else {
    coarse_gamma(c, r);
    const bool fast = c->mode == KKT_MODE_FAST && c->has_fast() && !(c->bisect & 5);
    if (form == KKT_FORM_MULTIPLICATIVE && fast) {
      rasq_apply(c, r, out, true);
      return;
    }
    KKT_LAUNCH(c, broadcast_gamma_kernel, g, 256, 0, c->ntl, c->nsp, c->n0, c->gam.p, yc);
  }
  switch (form) {
    case KKT_FORM_LITERAL:
      rasq_apply(c, yc, out, false);
      return;
    case KKT_FORM_ADDITIVE:
      rasq_apply(c, r, out, false);
      KKT_LAUNCH(c, axpb_kernel<false>, g, 256, 0, c->B, out, yc, out);
      return;
    case KKT_FORM_MULTIPLICATIVE: {
      double* res = c->tmpB2.p;
      // Shat y_c needs a B-sized temporary: reuse `out` (overwritten by the sweep).
      op_shat(c, yc, res, out);
      KKT_LAUNCH(c, axpb_kernel<true>, g, 256, 0, c->B, r, res, res);
      rasq_apply(c, res, out, false);
      KKT_LAUNCH(c, axpb_kernel<false>, g, 256, 0, c->B, out, yc, out);
      return;
    }
  }
  throw Error(KKT_EINVAL, "unknown two-level form");
}

// SchurSolver::apply (schur.cpp:494-533) for the device-supported kinds.
void schur_apply(Ctx* c, const double* r, double* out) {
  switch (c->desc.precond) {
    case KKT_PRECOND_NONE:
      KKT_CUDA(cudaMemcpyAsync(out, r, sizeof(double) * c->B, cudaMemcpyDeviceToDevice, c->stream));
      return;
    case KKT_PRECOND_ONE_LEVEL:
      rasq_apply(c, r, out, false);
      return;
    case KKT_PRECOND_TWO_LEVEL:
      two_level_apply(c, r, out, c->desc.two_level_form);
      return;
    default:
      throw Error(KKT_EUNSUPPORTED, "dense Schur preconditioners are desk-scale oracles, not on the device path");
  }
}

// apply_P_inv (kkt.cpp:71-81).
void pinv_apply(Ctx* c, const double* r, double* out) {
  op_pinv_uz(c, r, out);
  schur_apply(c, r + 2 * c->B, out + 2 * c->B);
}

}  // namespace kkt
