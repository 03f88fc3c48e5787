// sweep.cu — host orchestration of the spatial-solve chains: band solves,
// window solves (heat_operators.cpp:139-169) and the one-level RASQ sweep
// (apply_rasq, schur.cpp:103-130), in both arithmetic modes.
//
// RASQ without dead work: for subdomain s with node set
// [first, last] (first = s*m, or 1 for s = 0) the reference solves a window
// [W-node, first..last] forward, scales by ms, solves it adjoint, drops the
// W-node and keeps only owned nodes.  The W-node's forward value is
// Ahat^{-1} 0 = 0 and the adjoint values at the W-node and at `first` (owned
// by s-1) are discarded, so the chain here is
//   forward  x_n  = Ahat^{-1} (r_n + x_{n-1}),   n = first .. last
//   adjoint  x'_n = Ahat^{-T} (ms*x_n + x'_{n+1}), n = last .. owned.first
// and out[n] = x'_n (+ y_c[n] for the two-level forms).  All subdomains run
// as independent chains of one kernel launch.
#include <cstring>
#include <type_traits>
#include <vector>

#include "sweep.cuh"

namespace kkt {

namespace {

// Job descriptors go to a per-context device arena.  The H2D copy from
// pageable memory returns only after the data is staged, and the stream
// orders it after every kernel still reading the previous descriptors.
// The fast chains fold the previous step's inflow correction into the next
// step (sweep_v4.cu), which needs every step's `add` to be the same chain's
// previous `out` (or null).  All job builders below satisfy this; check it.
void check_fast_jobs(const std::vector<FastStep>& jobs, int nchains, int nsteps) {
  for (int s = 0; s < nchains; ++s)
    for (int t = 0; t < nsteps; ++t) {
      const FastStep& j = jobs[size_t(s) * nsteps + t];
      if (!j.in || !j.add) continue;
      const FastStep* pv = t > 0 ? &jobs[size_t(s) * nsteps + t - 1] : nullptr;
      if (!pv || !pv->in || pv->out != j.add)
        throw Error(KKT_EINVAL, "fast chain step: add is not the previous step's out");
    }
}

template <class T>
const T* upload(Ctx* c, DBuf<char>& buf, const std::vector<T>& v) {
  static_assert(std::is_trivially_copyable<T>::value, "chain descriptors are plain data");
  const size_t bytes = v.size() * sizeof(T);
  std::vector<char>& held = &buf == &c->jobs_fast ? c->jobs_fast_held : c->jobs_strict_held;
  if (buf.n >= bytes && held.size() == bytes && std::memcmp(held.data(), v.data(), bytes) == 0)
    return reinterpret_cast<const T*>(buf.p);  // the device copy is this table already (see Ctx)
  if (buf.n < bytes) {
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    buf.alloc(bytes);
  }
  // the copy below is from pageable memory: the driver has taken the bytes when the call returns,
  // but the table it overwrites may still be read by kernels queued earlier on the stream (stream
  // order covers that)
  KKT_CUDA(cudaMemcpyAsync(buf.p, v.data(), bytes, cudaMemcpyHostToDevice, c->stream));
  held.assign(reinterpret_cast<const char*>(v.data()), reinterpret_cast<const char*>(v.data()) + bytes);
  return reinterpret_cast<const T*>(buf.p);
}

}  // namespace

void band_solve(Ctx* c, double* b, int nrhs, bool transpose) {
  const size_t nsp = c->nsp;
  if (c->mode == KKT_MODE_STRICT || !c->has_fast() || (c->bisect & 4)) {
    std::vector<SolveStep> jobs(nrhs);
    for (int k = 0; k < nrhs; ++k) jobs[k] = {b + k * nsp, nullptr, b + k * nsp, 1.0, transpose ? 1 : 0};
    strict_chains(c, upload(c, c->jobs_strict, jobs), nrhs, 1);
  } else {
    std::vector<FastStep> jobs(nrhs);
    for (int k = 0; k < nrhs; ++k) jobs[k] = {b + k * nsp, nullptr, b + k * nsp, nullptr, 1.0, 0, 0};
    check_fast_jobs(jobs, nrhs, 1);
    fast_chains(c, upload(c, c->jobs_fast, jobs), nrhs, 1, false);
  }
}

void window_solve(Ctx* c, double* b, int len, bool adjoint) {
  const size_t nsp = c->nsp;
  if (len <= 0) return;
  if (c->mode == KKT_MODE_STRICT || !c->has_fast() || (c->bisect & 4)) {
    std::vector<SolveStep> jobs;
    for (int t = 0; t < len; ++t) {
      const int k = adjoint ? len - 1 - t : t;
      const double* add = nullptr;
      if (!adjoint && k > 0) add = b + (k - 1) * nsp;
      if (adjoint && k < len - 1) add = b + (k + 1) * nsp;
      jobs.push_back({b + k * nsp, add, b + k * nsp, 1.0, adjoint ? 1 : 0});
    }
    strict_chains(c, upload(c, c->jobs_strict, jobs), 1, len);
  } else {
    std::vector<FastStep> jobs;
    for (int t = 0; t < len; ++t) {
      const int k = adjoint ? len - 1 - t : t;
      const double* add = nullptr;
      if (!adjoint && k > 0) add = b + (k - 1) * nsp;
      if (adjoint && k < len - 1) add = b + (k + 1) * nsp;
      jobs.push_back({b + k * nsp, add, b + k * nsp, nullptr, 1.0, 0, 0});
    }
    check_fast_jobs(jobs, 1, len);
    fast_chains(c, upload(c, c->jobs_fast, jobs), 1, len, false);
  }
}

// out = RASQ(r) (one-level), or in fast mode with `fused_coarse`:
// out = RASQ(r - Shat y_c) + y_c with y_c = gamma (c->gam) per node.
// On a time slab the chains are this rank's subdomains s0 .. s0+ndl-1 and
// plane(n) addresses global node n in the local slab; the first local
// subdomain's shared node (n0-1, owned by the previous rank) arrives as a halo.
void rasq_apply(Ctx* c, const double* r, double* out, bool fused_coarse) {
  const int64_t nsp = c->nsp;
  const int Nd = c->ndl, m = c->m;
  const int nsteps = 2 * m + 1;
  const Halo hr = exchange_halo(c, r, 3, 3, true, false);
  auto plane = [&](const double* base, int n) {
    if (n == c->n0 - 1 && base == r) return hr.prev;  // shared node of the first local subdomain
    return base + (n - c->n0) * nsp;
  };
  auto wplane = [&](double* base, int n) { return base + (n - c->n0) * nsp; };
  if (c->mode == KKT_MODE_FAST && spectral_enabled(c)) {
    spectral_rasq(c, r, c->s0 > 0 ? hr.prev : nullptr, out, fused_coarse);
    return;
  }
  if (c->mode == KKT_MODE_STRICT || !c->has_fast() || (c->bisect & 4)) {
    // scratch: one plane per subdomain for the shared node's forward value
    const size_t need = size_t(Nd) * nsp;
    if (c->tmpB3.n < need) c->tmpB3.alloc(need);
    // out starts at zero (the reference accumulates into layout.zeros())
    dev_fill(c, out, 0, sizeof(double) * c->B);
    std::vector<SolveStep> jobs(size_t(Nd) * nsteps, SolveStep{nullptr, nullptr, nullptr, 1.0, 0});
    for (int sl = 0; sl < Nd; ++sl) {
      const int s = c->s0 + sl;
      double* shared = c->tmpB3.p + sl * nsp;
      SolveStep* J = jobs.data() + size_t(sl) * nsteps;
      const int first = s == 0 ? 1 : s * m;
      // forward over first..last
      for (int t = 0; t <= m; ++t) {
        const int n = s * m + t;
        if (n < first) continue;
        const double* add = nullptr;
        if (n > first) add = (n - 1 == first && s > 0) ? shared : plane(out, n - 1);
        double* dst = (s > 0 && n == first) ? shared : wplane(out, n);
        J[t] = {plane(r, n), add, dst, 1.0, 0};
      }
      // adjoint over last..owned.first
      for (int t = 0; t < m; ++t) {
        const int n = (s + 1) * m - t;
        const double* add = t == 0 ? nullptr : plane(out, n + 1);
        J[m + 1 + t] = {plane(out, n), add, wplane(out, n), c->ms, 1};
      }
    }
    strict_chains(c, upload(c, c->jobs_strict, jobs), Nd, nsteps);
    return;
  }
  // ---- fast
  const size_t need = size_t(Nd) * 3 * nsp;
  if (c->tmpB3.n < need) c->tmpB3.alloc(need);
  std::vector<FastStep> jobs(size_t(Nd) * nsteps, FastStep{nullptr, nullptr, nullptr, nullptr, 1.0, 0, 0});
  for (int sl = 0; sl < Nd; ++sl) {
    const int s = c->s0 + sl;
    double* shared = c->tmpB3.p + (3 * sl) * nsp;
    double* adj[2] = {c->tmpB3.p + (3 * sl + 1) * nsp, c->tmpB3.p + (3 * sl + 2) * nsp};
    FastStep* J = jobs.data() + size_t(sl) * nsteps;
    const int first = s == 0 ? 1 : s * m;
    for (int t = 0; t <= m; ++t) {
      const int n = s * m + t;
      if (n < first) continue;
      const double* add = nullptr;
      if (n > first) add = (n - 1 == first && s > 0) ? shared : plane(out, n - 1);
      double* dst = (s > 0 && n == first) ? shared : wplane(out, n);
      J[t] = {plane(r, n), add, dst, nullptr, 1.0, fused_coarse ? n : 0, 0};
    }
    for (int t = 0; t < m; ++t) {
      const int n = (s + 1) * m - t;
      const double* add = t == 0 ? nullptr : adj[(t - 1) & 1];
      J[m + 1 + t] = {plane(out, n), add, adj[t & 1], wplane(out, n), c->ms, 0,
                      fused_coarse ? n : 0};
    }
  }
  check_fast_jobs(jobs, Nd, nsteps);
  // kkt_apply_P_inv_host with this RASQ output as the final w block: adjoint step t writes the
  // final planes of nodes (s+1) m - t, one per local subdomain and m planes apart, which no later
  // step touches; a step-by-step sweep (v6) sends them to the host behind each step.
  if (c->e2e_w_host && c->v6_ops.p && !c->v4_ops.p) {
    double* host = c->e2e_w_host;
    c->e2e_trailed = true;
    c->step_hook = [c, host, out, Nd, m, nsp](int t) {
      if (t <= m) return;
      const int tp = t - (m + 1);
      const size_t off = size_t(m - 1 - tp) * nsp;  // node (s0 + 1) m - tp of the local slab
      KKT_CUDA(cudaEventRecord(c->e2e_step_ev, c->stream));
      KKT_CUDA(cudaStreamWaitEvent(c->e2e_trail, c->e2e_step_ev, 0));
      KKT_CUDA(cudaMemcpy2DAsync(host + off, sizeof(double) * size_t(m) * nsp, out + off, sizeof(double) * size_t(m) * nsp,
                                 sizeof(double) * nsp, size_t(Nd), cudaMemcpyDeviceToHost, c->e2e_trail));
    };
  }
  try {
    fast_chains(c, upload(c, c->jobs_fast, jobs), Nd, nsteps, fused_coarse);
  } catch (...) {
    c->step_hook = nullptr;
    throw;
  }
  c->step_hook = nullptr;
}

}  // namespace kkt
