// factor.cu — K6: LU factorisation of Ahat on the device.
//
// band_lu_kernel restates BandedLU::BandedLU (reference linalg.cpp:69-125) on
// the reference's own band storage (linalg.hpp:65-74): partial pivoting with
// the first-maximum rule, column scaling by division, rank-1 update column by
// column with the zero-u skip.  Every entry sees the same sequence of
// separately rounded operations as in the reference, so the factor is
// bitwise identical (tests/test_gpu_parity.py::test_factor_bitwise).
//
// build_block_inverses then views the (pivot-free) factor in
// nx-by-nx blocks and inverts the diagonal blocks: Li_J = L_JJ^{-1} (unit
// lower) and Ui_J = U_JJ^{-1} (upper), the operators of the fast blocked
// substitution (sweep.cu).
#include <cmath>
#include <cstdlib>

#include "sweep.cuh"

namespace kkt {
namespace {

constexpr int kLuThreads = 1024;

__global__ void fill_band_kernel(int n, int nx, int bw, int kuf, int ld, Stencil s, double* ab) {
  const int64_t total = int64_t(n) * ld;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(t / ld);
    const int o = int(t - int64_t(j) * ld);
    const int i = o + j - kuf;  // row
    double v = 0.0;
    if (i >= 0 && i < n && i - j <= bw && j - i <= bw) {
      const int d = i - j;
      if (d == 0) {
        v = s.diag;
      } else if ((d == 1 || d == -1) && (i / nx == j / nx) && nx > 1) {
        v = s.mcx;
      } else if (d == nx || d == -nx) {
        v = s.mcy;
      }
    }
    ab[t] = v;
  }
}

struct LuStatus {
  int singular_at;  // -1 = ok
  int pivoted;
  double best;
};

// Single-CTA right-looking banded LU, the reference's loop nest verbatim.
__global__ void __launch_bounds__(kLuThreads) band_lu_kernel(int n, int kl, int kuf, int ld,
                                                             double tol, double* ab, int* piv,
                                                             LuStatus* st) {
  __shared__ int s_p;
  __shared__ double s_best;
  __shared__ double s_rbest[32];
  __shared__ int s_ridx[32];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  int pivoted = 0;
  auto E = [&](int i, int j) -> double& { return ab[int64_t(j) * ld + (i - j + kuf)]; };

  for (int j = 0; j < n; ++j) {
    const int imax = min(n - 1, j + kl);
    const int jmax = min(n - 1, j + kuf);
    // ---- pivot search: first maximum of |entry(i, j)|, i = j..imax (linalg.cpp:89-97)
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int i = j + tid; i <= imax; i += blockDim.x) {
      const double v = fabs(E(i, j));
      if (v > best || (v == best && i < bidx)) { best = v; bidx = i; }
    }
    for (int off = 16; off; off >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, off);
      const int oi = __shfl_down_sync(0xffffffffu, bidx, off);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if (lane == 0) { s_rbest[wid] = best; s_ridx[wid] = bidx; }
    __syncthreads();
    if (wid == 0) {
      best = lane < nwarps ? s_rbest[lane] : -1.0;
      bidx = lane < nwarps ? s_ridx[lane] : 0x7fffffff;
      for (int off = 16; off; off >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, off);
        const int oi = __shfl_down_sync(0xffffffffu, bidx, off);
        if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
      }
      if (lane == 0) {
        // The reference starts from best = |entry(j,j)| and replaces only on a
        // strictly larger value: ties keep the smallest row index, as here.
        s_p = bidx;
        s_best = best;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (!(s_best > tol)) {
      if (tid == 0) { st->singular_at = j; st->best = s_best; st->pivoted = pivoted; }
      return;
    }
    if (tid == 0) piv[j] = p;
    if (p != j) {
      pivoted = 1;
      for (int c = j + tid; c <= jmax; c += blockDim.x) {
        const double a = E(j, c);
        E(j, c) = E(p, c);
        E(p, c) = a;
      }
      __syncthreads();
    }
    const double d = E(j, j);
    for (int i = j + 1 + tid; i <= imax; i += blockDim.x) E(i, j) = sdiv(E(i, j), d);
    __syncthreads();
    // ---- rank-1 update, column by column (linalg.cpp:112-121)
    const int rows = imax - j;
    const int cols = jmax - j;
    if (rows > 0 && cols > 0) {
      const int64_t pairs = int64_t(rows) * cols;
      for (int64_t t = tid; t < pairs; t += blockDim.x) {
        const int cc = int(t / rows);
        const int r = int(t - int64_t(cc) * rows);
        const int c = j + 1 + cc;
        const int i = j + 1 + r;
        const double ujc = E(j, c);
        if (ujc != 0.0) E(i, c) = ssub(E(i, c), smul(E(i, j), ujc));
      }
    }
    __syncthreads();
  }
  if (tid == 0) { st->singular_at = -1; st->pivoted = pivoted; st->best = 0.0; }
}

// Row-major copy of U's strict upper band: ut[i*kl + k-1] = U(i, i+k), k=1..kl,
// for the strict transpose solve (linalg.cpp:150-154 reads U column-wise).
__global__ void ut_kernel(int n, int kl, int kuf, int ld, const double* __restrict__ ab,
                          double* __restrict__ ut) {
  const int64_t total = int64_t(n) * kl;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / kl);
    const int k = int(t - int64_t(i) * kl) + 1;
    const int c = i + k;
    ut[t] = c < n ? ab[int64_t(c) * ld + (kuf - k)] : 0.0;
  }
}

// One CTA per block row J, one thread per column b: Li_J e_b and Ui_J e_b by
// substitution on the diagonal blocks of the band factor.
__global__ void block_inverse_kernel(int nx, int kl, int kuf, int ld, const double* __restrict__ ab,
                                     double* __restrict__ Li, double* __restrict__ Ui) {
  const int J = blockIdx.x;
  const int b = threadIdx.x;
  if (b >= nx) return;
  const int base = J * nx;
  const int64_t off = int64_t(J) * nx * nx;
  // entries outside the stored band are zero (ny == 1 gives a band narrower than nx)
  auto E = [&](int a, int k) {
    const int d = a - k;
    return (d > kl || -d > kuf) ? 0.0 : ab[int64_t(base + k) * ld + (d + kuf)];
  };
  double* X = Li + off;
  // L_JJ X = I, L unit lower: X(a,b) = [a==b] - sum_{k<a} L(a,k) X(k,b)
  for (int a = 0; a < nx; ++a) {
    double acc = (a == b) ? 1.0 : 0.0;
    if (a > b) {
      for (int k = b; k < a; ++k) acc = fma(-E(a, k), X[int64_t(k) * nx + b], acc);
    }
    X[int64_t(a) * nx + b] = acc;
  }
  double* Y = Ui + off;
  // U_JJ Y = I, U upper: Y(a,b) = ([a==b] - sum_{k>a} U(a,k) Y(k,b)) / U(a,a)
  for (int a = nx - 1; a >= 0; --a) {
    double acc = 0.0;
    if (a <= b) {
      acc = (a == b) ? 1.0 : 0.0;
      for (int k = a + 1; k <= b; ++k) acc = fma(-E(a, k), Y[int64_t(k) * nx + b], acc);
      acc = acc / E(a, a);
    }
    Y[int64_t(a) * nx + b] = acc;
  }
}

// Packed Li_J (row a: entries 0..a at a(a+1)/2) followed by D_J^{-1}
// (1 / U(Jnx+a, Jnx+a)), one `stride`-double block per block row.
__global__ void pack_lower_kernel(int nx, int ny, int kuf, int ld, int stride,
                                  const double* __restrict__ ab, const double* __restrict__ Li,
                                  double* __restrict__ Lpk) {
  const int J = blockIdx.x;
  const int T = nx * (nx + 1) / 2;
  const double* X = Li + int64_t(J) * nx * nx;
  double* dst = Lpk + int64_t(J) * stride;
  for (int e = threadIdx.x; e < stride; e += blockDim.x) {
    double v = 0.0;
    if (e < T) {
      // row a: e in [a(a+1)/2, a(a+1)/2 + a]
      int a = int((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      while (a * (a + 1) / 2 > e) --a;
      const int b = e - a * (a + 1) / 2;
      v = X[int64_t(a) * nx + b];
    } else if (e < T + nx) {
      const int a = e - T;
      v = 1.0 / ab[int64_t(J * nx + a) * ld + kuf];
    }
    dst[e] = v;
  }
}

}  // namespace

void build_factor(Ctx* c) {
  const int n = c->nsp;
  const int nx = c->nx, ny = c->ny;
  // assemble_spatial_operator's band (heat_operators.cpp:31-32)
  const int bw = ny > 1 ? nx : (nx > 1 ? 1 : 0);
  c->kl = bw;
  c->kuf = std::min(n > 0 ? n - 1 : 0, bw + bw);
  c->ld = c->kl + c->kuf + 1;
  c->ab.alloc(size_t(n) * c->ld);
  c->piv.alloc(n);

  // ||Ahat||_inf with the reference's summation order (linalg.cpp:35-43);
  // zero band entries add nothing.
  double anorm = 0.0;
  for (int j = 1; j <= ny; ++j) {
    for (int i = 1; i <= nx; ++i) {
      double row = 0.0;
      if (j > 1) row += std::abs(c->Ahat.mcy);
      if (i > 1) row += std::abs(c->Ahat.mcx);
      row += std::abs(c->Ahat.diag);
      if (i < nx) row += std::abs(c->Ahat.mcx);
      if (j < ny) row += std::abs(c->Ahat.mcy);
      anorm = std::max(anorm, row);
    }
  }
  const double tol = 1e-14 * anorm;  // kSingularTol (linalg.cpp:10)

  KKT_LAUNCH(c, fill_band_kernel, kSmCount * 4, 256, 0, n, nx, bw, c->kuf, c->ld, c->Ahat, c->ab.p);
  DBuf<LuStatus> st(1);
  KKT_LAUNCH(c, band_lu_kernel, 1, kLuThreads, 0, n, c->kl, c->kuf, c->ld, tol, c->ab.p, c->piv.p,
             st.p);
  LuStatus hs{};
  KKT_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(hs), cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  if (hs.singular_at >= 0) {
    throw Error(KKT_ESINGULAR,
                "banded LU: pivot " + std::to_string(hs.best) + " at index " +
                    std::to_string(hs.singular_at) + " below tolerance " + std::to_string(tol),
                hs.singular_at);
  }
  c->pivoted = hs.pivoted != 0;

  if (c->kl > 0) {
    c->ut.alloc(size_t(n) * c->kl);
    KKT_LAUNCH(c, ut_kernel, kSmCount * 4, 256, 0, n, c->kl, c->kuf, c->ld, c->ab.p, c->ut.p);
  }
}

void build_block_inverses(Ctx* c) {
  if (c->pivoted) return;  // blocked path needs the pivot-free block structure
  const int nx = c->nx, ny = c->ny;
  c->Li.alloc(size_t(ny) * nx * nx);
  c->Ui.alloc(size_t(ny) * nx * nx);
  const int threads = ((nx + 31) / 32) * 32;
  KKT_LAUNCH(c, block_inverse_kernel, ny, threads, 0, nx, c->kl, c->kuf, c->ld, c->ab.p, c->Li.p, c->Ui.p);
  if (tma_supported(c)) {
    // v2 sweep: packed Li + D^{-1} only (U_JJ = D_J L_JJ^T for the symmetric Ahat)
    const int T = nx * (nx + 1) / 2;
    c->Lpk_stride = (T + nx + 1) & ~1;
    c->Lpk.alloc(size_t(ny) * c->Lpk_stride);
    KKT_LAUNCH(c, pack_lower_kernel, ny, 256, 0, nx, ny, c->kuf, c->ld, c->Lpk_stride, c->ab.p,
               c->Li.p, c->Lpk.p);
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    if (group_supported(c) && getenv("KKT_SWEEP_V2") == nullptr) build_group_operators(c);
    c->Li.release();
    c->Ui.release();
  }
}

}  // namespace kkt
