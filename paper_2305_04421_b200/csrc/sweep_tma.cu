// sweep_tma.cu — FAST blocked spatial solves, v2 (nx <= 128: configs 0 and 1).
//
// Same block substitution as sweep_fast.cu, with two changes that cut the
// factor traffic of every block step by 2x and take its latency off the
// critical path:
//
//  1. Only Li_J = L_JJ^{-1} is stored.  Ahat is symmetric and the reference's
//     factor is pivot-free, so Ahat = L U = L D L^T with D = diag(U); hence
//     U_JJ = D_J L_JJ^T and Ui_J = Li_J^T D_J^{-1}.  The substitutions become
//        y_J = Li_J ( b_J + cy * Li_{J-1}^T (D_{J-1}^{-1} y_{J-1}) )
//        x_J = Li_J^T D_J^{-1} ( y_J + cy * Li_J x_{J+1} )
//     Li_J is packed (lower triangle row by row, then D_J^{-1}): one
//     nx(nx+1)/2 + nx double block per block row.
//  2. The block rows are visited in a zig-zag (0..ny-1, ny-2..0, 1..) over
//     the L and U sweeps of consecutive solves, so each visit needs exactly
//     ONE new packed block.  It is brought into shared memory by a TMA bulk
//     copy (cp.async.bulk + mbarrier) one step ahead, into a 3-slot ring, and
//     the triangle resident from the previous step is reused.
//
// One CTA (16 warps) per chain; lanes own the columns b = lane + 32k, so the
// lower mat-vec reduces across the warp and the transposed one accumulates
// per lane and reduces across warps through shared memory.
#include "sweep_tma.cuh"

namespace kkt {
namespace {
using namespace tma;

struct TmaParams {
  const double* Lpk;   // ny packed blocks of TP doubles
  int TP;              // doubles per packed block (even)
  int T;               // nx(nx+1)/2: offset of D^{-1} inside a block
  int nx, ny, nsp;
  double cy;
  const double* a1;
  const double* a2;
  const double* gam;
  double inv_ms;
  double* ws;          // per chain: one plane (L-solve intermediate)
  int ws_stride;
};

__global__ void __launch_bounds__(kThreads, 1) tma_chain_kernel(TmaParams P,
                                                              const FastStep* __restrict__ steps,
                                                              int nsteps, bool coarse) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[kSlots];
  const int nx = P.nx, ny = P.ny;
  auto slot = [&](long q) { return sm + int(q % kSlots) * P.TP; };
  double* V = sm + kSlots * P.TP;         // vectors
  double* Y0 = V;                         // y ping-pong
  double* Y1 = V + kMaxNx;
  double* TV = V + 2 * kMaxNx;            // t / s
  double* WV = V + 3 * kMaxNx;            // D^{-1}-scaled input of the transposed mat-vec
  double* UV = V + 4 * kMaxNx;            // mat-vec outputs
  double* PART = V + 5 * kMaxNx;          // kWarps x kMaxNx
  double* y = P.ws + int64_t(blockIdx.x) * P.ws_stride;
  const int tid = threadIdx.x;
  const uint32_t bytes = uint32_t(P.TP) * 8u;
  int roff[kR];
  row_offsets(roff);

  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // issue / wait on zig-zag positions
  auto issue = [&](long q) {
    if (tid == 0) {
      const int J = zig(q, ny);
      tma_load(slot(q), P.Lpk + int64_t(J) * P.TP, bytes, &bars[q % kSlots]);
    }
  };
  auto wait = [&](long q) { mbar_wait(&bars[q % kSlots], uint32_t((q / kSlots) & 1)); };
  const long Pz = ny > 1 ? 2L * (ny - 1) : 0;
  long hi_issued = -1, hi_waited = -1;
  auto issue_t = [&](long q) {
    issue(q);
    hi_issued = q > hi_issued ? q : hi_issued;
  };
  auto wait_t = [&](long q) {
    wait(q);
    hi_waited = q > hi_waited ? q : hi_waited;
  };
  issue_t(0);
  if (ny > 1) issue_t(1);
  long base = 0;  // zig-zag position of this solve's J = 0 in the L sweep

  for (int t = 0; t < nsteps; ++t) {
    const FastStep st = steps[int64_t(blockIdx.x) * nsteps + t];
    if (!st.in) continue;
    const bool cres = coarse && st.node > 0;
    double gn = 0.0, gm = 0.0, gp = 0.0;
    if (cres) {
      gn = P.gam[st.node];
      gm = P.gam[st.node - 1];
      gp = P.gam[st.node + 1];
    }
    const bool first_node = st.node == 1;
    auto rhs = [&](int p) {
      double v = st.in[p] * st.scale;
      if (st.add) v += st.add[p];
      if (cres) {
        double sh = gn * P.a2[p] - gp * P.a1[p];
        if (!first_node) sh += gn - gm * P.a1[p];
        v -= sh * P.inv_ms;
      }
      return v;
    };
    // ---------------- L sweep: y_J = Li_J (b_J + cy Li_{J-1}^T D_{J-1}^{-1} y_{J-1})
    double* yprev = Y0;
    double* ycur = Y1;
    double bnext = (tid < nx) ? rhs(tid) : 0.0;
    for (int J = 0; J < ny; ++J) {
      const long q = base + J;
      if (tid < nx) TV[tid] = bnext;
      if (tid < nx && J + 1 < ny) bnext = rhs((J + 1) * nx + tid);  // prefetch next block's rhs
      wait_t(q);
      double vr[kK];
      if (J > 0) {
        const double* Lp = slot(q - 1);
        lowerT_mv(Lp, roff, Lp + P.T, yprev, nullptr, 0.0, PART, UV, nx);
        __syncthreads();
        load_vr(TV, UV, P.cy, vr, nx);
      } else {
        __syncthreads();
        load_vr(TV, nullptr, 0.0, vr, nx);
      }
      lower_mv(slot(q), roff, vr, ycur, nx);
      __syncthreads();
      if (tid < nx) y[J * nx + tid] = ycur[tid];
      if (J >= 1 && ny > 1) issue_t(q + 1);  // position q-1 is dead
      double* tmp = yprev;
      yprev = ycur;
      ycur = tmp;
    }
    // ---------------- U sweep: x_J = Li_J^T D_J^{-1} (y_J + cy Li_J x_{J+1})
    double* xprev = Y0;
    double* xcur = Y1;
    const double g2 = (st.out2 && st.node2 > 0 && P.gam) ? P.gam[st.node2] : 0.0;
    double ynext = (tid < nx) ? y[(ny - 1) * nx + tid] : 0.0;
    for (int J = ny - 1; J >= 0; --J) {
      const long q = (J == ny - 1) ? base + ny - 1 : base + Pz - J;
      if (tid < nx) TV[tid] = ynext;
      if (tid < nx && J > 0) ynext = y[(J - 1) * nx + tid];
      wait_t(q);
      const double* Lp = slot(q);
      if (J < ny - 1) {
        double vr[kK];
        load_vr(xprev, nullptr, 0.0, vr, nx);
        lower_mv(Lp, roff, vr, UV, nx);
        __syncthreads();
        lowerT_mv(Lp, roff, Lp + P.T, TV, UV, P.cy, PART, xcur, nx);
      } else {
        __syncthreads();
        lowerT_mv(Lp, roff, Lp + P.T, TV, nullptr, 0.0, PART, xcur, nx);
      }
      __syncthreads();
      if (tid < nx) {
        const double x = xcur[tid];
        if (st.out) st.out[J * nx + tid] = x;
        if (st.out2) st.out2[J * nx + tid] = x + g2;
      }
      if (ny > 1 && J >= 1) issue_t(q + 2);  // position q is dead after this step
      double* tmp = xprev;
      xprev = xcur;
      xcur = tmp;
    }
    base += Pz;
    __syncthreads();
  }
  // drain: every issued copy must land before the CTA exits
  for (long q = hi_waited + 1; q <= hi_issued; ++q) wait(q);
}

}  // namespace

bool tma_supported(const Ctx* c) { return c->nx <= kMaxNx && c->nx >= 1; }

size_t tma_smem_bytes(int TP) {
  return sizeof(double) * (size_t(kSlots) * TP + size_t(5 + kWarps) * kMaxNx);
}

void tma_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms) {
  const size_t need = size_t(nchains) * c->nsp;
  if (c->sweep_ws.n < need) c->sweep_ws.alloc(need);
  TmaParams P;
  P.Lpk = c->Lpk.p;
  P.TP = c->Lpk_stride;
  P.T = c->nx * (c->nx + 1) / 2;
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
  const size_t smem = tma_smem_bytes(P.TP);
  static bool attr = false;
  if (!attr) {
    KKT_CUDA(cudaFuncSetAttribute(tma_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(tma_smem_bytes(((kMaxNx * (kMaxNx + 1)) / 2 + kMaxNx + 1) & ~1))));
    attr = true;
  }
  c->tbegin(3);
  KKT_LAUNCH(c, tma_chain_kernel, nchains, kThreads, smem, P, jobs_dev, nsteps, coarse_terms);
  c->tend(3);
}

}  // namespace kkt
