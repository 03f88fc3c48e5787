// sweep_fast.cu — FAST blocked spatial solves (K5 inner kernel).
//
// Ahat = L U with the reference's (pivot-free) banded factor viewed in
// nx-by-nx blocks: L = blockbidiag(L_{J,J-1}, L_JJ),
// U = blockbidiag(U_JJ, U_{J,J+1}).  Because Ahat's off-diagonal blocks are
// -cy*I, the block LU gives L_{J,J-1} = -cy * U_{J-1,J-1}^{-1} and
// U_{J,J+1} = -cy * L_JJ^{-1}, so the two substitutions become
//     y_J = Li_J ( b_J + cy * Ui_{J-1} y_{J-1} )          J = 0 .. ny-1
//     x_J = Ui_J ( y_J + cy * Li_J x_{J+1} )              J = ny-1 .. 0
// with Li_J = L_JJ^{-1}, Ui_J = U_JJ^{-1} precomputed (factor.cu).  This is
// the same LU solve as BandedLU::solve_in_place (linalg.cpp:127-145), with
// explicit inverses of the diagonal blocks: every block step is two
// triangular mat-vecs instead of a dependent row-by-row chain.  Ahat is
// symmetric (and centro-symmetric), so the transpose solve of the adjoint
// sweep uses the same operators.
//
// v1 layout: one CTA per chain (a time subdomain's window of solves),
// factor blocks streamed from L2/HBM, the L-solve intermediate in a
// per-chain global plane.  The two-level residual r - Shat y_c of the
// multiplicative form (schur.cpp:435-437) is generated on the fly from the
// per-node coarse values gamma and the precomputed a1 = Ahat 1, a2 = Ahat a1.
#include "sweep.cuh"

namespace kkt {
namespace {

constexpr int kFastThreads = 256;

struct FastParams {
  const double* Li;
  const double* Ui;
  int nx, ny, nsp;
  double cy;
  const double* a1;
  const double* a2;
  const double* gam;  // gamma_0 .. gamma_{Nt+1}
  double inv_ms;
  double* ws;         // per chain: kWsPlanes planes; plane 0 = L-solve intermediate
  int ws_stride;      // doubles per chain
};

// out[a] = sum_b M[a, b] v[b] over the stored triangle (zeros elsewhere).
template <bool kLower>
__device__ __forceinline__ void tri_mv(const double* __restrict__ M, const double* v, double* out,
                                       int nx) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int a0 = warp * 4; a0 < nx; a0 += nw * 4) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    const int lo = kLower ? 0 : a0;
    const int hi = kLower ? min(a0 + 3, nx - 1) : nx - 1;
    const double* r0 = M + int64_t(a0) * nx;
    const bool v1 = a0 + 1 < nx, v2 = a0 + 2 < nx, v3 = a0 + 3 < nx;
    for (int b = lo + lane; b <= hi; b += 32) {
      const double vb = v[b];
      acc0 = fma(r0[b], vb, acc0);
      if (v1) acc1 = fma(r0[nx + b], vb, acc1);
      if (v2) acc2 = fma(r0[2 * nx + b], vb, acc2);
      if (v3) acc3 = fma(r0[3 * nx + b], vb, acc3);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      acc0 += __shfl_xor_sync(0xffffffffu, acc0, off);
      acc1 += __shfl_xor_sync(0xffffffffu, acc1, off);
      acc2 += __shfl_xor_sync(0xffffffffu, acc2, off);
      acc3 += __shfl_xor_sync(0xffffffffu, acc3, off);
    }
    if (lane == 0) {
      out[a0] = acc0;
      if (v1) out[a0 + 1] = acc1;
      if (v2) out[a0 + 2] = acc2;
      if (v3) out[a0 + 3] = acc3;
    }
  }
}

__global__ void __launch_bounds__(kFastThreads) fast_chain_kernel(FastParams P,
                                                                  const FastStep* __restrict__ steps,
                                                                  int nsteps, bool coarse) {
  extern __shared__ double sm[];
  const int nx = P.nx, ny = P.ny;
  double* vA = sm;
  double* vB = sm + nx;
  double* vT = sm + 2 * nx;
  double* y = P.ws + int64_t(blockIdx.x) * P.ws_stride;
  const int64_t nn = int64_t(nx) * nx;
  for (int t = 0; t < nsteps; ++t) {
    const FastStep st = steps[int64_t(blockIdx.x) * nsteps + t];
    if (!st.in) continue;
    double gn = 0.0, gm = 0.0, gp = 0.0;
    const bool cres = coarse && st.node > 0;
    if (cres) {
      gn = P.gam[st.node];
      gm = P.gam[st.node - 1];
      gp = P.gam[st.node + 1];
    }
    const bool first_node = st.node == 1;
    // ---------------- L sweep
    double* yprev = vA;
    double* ycur = vB;
    for (int J = 0; J < ny; ++J) {
      const int base = J * nx;
      if (J > 0) {
        tri_mv<false>(P.Ui + int64_t(J - 1) * nn, yprev, vT, nx);
        __syncthreads();
      }
      for (int a = threadIdx.x; a < nx; a += blockDim.x) {
        const int p = base + a;
        double v = st.in[p] * st.scale;
        if (st.add) v += st.add[p];
        if (cres) {
          // (Shat y_c)_n with y_c = gamma_n * 1 per node (schur.cpp:71-78 analytically)
          double sh = gn * P.a2[p] - gp * P.a1[p];
          if (!first_node) sh += gn - gm * P.a1[p];
          v -= sh * P.inv_ms;
        }
        if (J > 0) v = fma(P.cy, vT[a], v);
        vT[a] = v;
      }
      __syncthreads();
      tri_mv<true>(P.Li + int64_t(J) * nn, vT, ycur, nx);
      __syncthreads();
      for (int a = threadIdx.x; a < nx; a += blockDim.x) y[base + a] = ycur[a];
      double* tmp = yprev;
      yprev = ycur;
      ycur = tmp;
    }
    // ---------------- U sweep
    double* xprev = vA;
    double* xcur = vB;
    const double g2 = (st.out2 && st.node2 > 0 && P.gam) ? P.gam[st.node2] : 0.0;
    for (int J = ny - 1; J >= 0; --J) {
      const int base = J * nx;
      __syncthreads();
      if (J < ny - 1) {
        tri_mv<true>(P.Li + int64_t(J) * nn, xprev, vT, nx);
        __syncthreads();
      }
      for (int a = threadIdx.x; a < nx; a += blockDim.x) {
        double v = y[base + a];
        if (J < ny - 1) v = fma(P.cy, vT[a], v);
        vT[a] = v;
      }
      __syncthreads();
      tri_mv<false>(P.Ui + int64_t(J) * nn, vT, xcur, nx);
      __syncthreads();
      for (int a = threadIdx.x; a < nx; a += blockDim.x) {
        const double x = xcur[a];
        if (st.out) st.out[base + a] = x;
        if (st.out2) st.out2[base + a] = x + g2;
      }
      double* tmp = xprev;
      xprev = xcur;
      xcur = tmp;
    }
    __syncthreads();  // this step's global writes before the next step's reads
  }
}

}  // namespace

void fast_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms) {
  if (nchains <= 0 || nsteps <= 0) return;
  if (c->v4_ops.p) {
    v4_chains(c, jobs_dev, nchains, nsteps, coarse_terms);
    return;
  }
  if (c->v6_ops.p) {
    v6_chains(c, jobs_dev, nchains, nsteps, coarse_terms);
    return;
  }
  if (c->v5_ops.p) {
    v5_chains(c, jobs_dev, nchains, nsteps, coarse_terms);
    return;
  }
  if (c->Phi.p) {
    group_chains(c, jobs_dev, nchains, nsteps, coarse_terms);
    return;
  }
  if (c->Lpk.p) {
    tma_chains(c, jobs_dev, nchains, nsteps, coarse_terms);
    return;
  }
  const size_t need = size_t(nchains) * c->nsp;
  if (c->sweep_ws.n < need) c->sweep_ws.alloc(need);
  FastParams P;
  P.Li = c->Li.p;
  P.Ui = c->Ui.p;
  P.nx = c->nx;
  P.ny = c->ny;
  P.nsp = c->nsp;
  P.cy = c->cy;
  P.a1 = c->a1.p;
  P.a2 = c->a2.p;
  P.gam = c->gam.p;
  P.inv_ms = 1.0 / c->ms;
  P.ws = c->sweep_ws.p;
  P.ws_stride = c->nsp;
  const size_t smem = sizeof(double) * 3 * size_t(c->nx);
  c->tbegin(3);
  KKT_LAUNCH(c, fast_chain_kernel, nchains, kFastThreads, smem, P, jobs_dev, nsteps, coarse_terms);
  c->tend(3);
}

}  // namespace kkt
