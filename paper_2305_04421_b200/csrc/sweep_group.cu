// sweep_group.cu — FAST spatial solves, v3: group-parallel block substitution
// (nx <= 128: configs 0 and 1).
//
// Each spatial solve is the reference's LU solve (linalg.cpp:127-145) in the
// block form of sweep_tma.cu:
//     L sweep  y_J = c_J + G_J y_{J-1},   c_J = Li_J b_J,
//              G_J = cy Li_J Li_{J-1}^T D_{J-1}^{-1}
//     U sweep  x_J = d_J + H_J x_{J+1},   d_J = Li_J^T D_J^{-1} y_J,
//              H_J = cy Li_J^T D_J^{-1} Li_J
// Both are affine block recurrences.  The ny block rows are cut into groups of
// g rows; the dependent chain of 2*ny block steps per solve becomes
//   A  every (chain, group) runs its g steps with zero inflow       (parallel)
//   B  every (chain, group) forms its boundary value
//        e_g = ytilde_end(g) + Phi_end(g) e_{g-1}  (unrolled, see phase B)
//   C  every block row adds its inflow term  y_J += Phi_J e_{g-1}   (parallel,
//      one CTA per J, all chains at once with fp64 DMMA)
// with Phi_J = G_J ... G_{first(g)} (and Psi_J = H_J ... H_{last(g)} for the
// U sweep) precomputed at setup — the superposition of the zero-inflow
// solution and the propagated inflow is exact in exact arithmetic, so this is
// the same substitution with a re-associated recurrence (rounding-level
// differences, gated like the rest of the fast mode).
//
// Phase B is unrolled into independent sums with precomputed products of the
// group-boundary propagators, so per spatial solve there are 6 launches
// (A/B/C for L and U) and the dependent depth per sweep drops from ny block
// steps to g steps + 2 parallel GEMM-like phases, with ~NG*Nd SMs at work.
#include <cstdlib>
#include <vector>

#include "sweep_tma.cuh"

namespace kkt {
namespace {
using namespace tma;

constexpr int kLd = kMaxNx;            // dense matrices: kMaxNx x kMaxNx, zero padded
constexpr int kDense = kLd * kLd;      // doubles per dense matrix
constexpr int kCBatch = 16;            // chains per DMMA pass in phase C

struct GrpParams {
  const double* Lpk;
  int TP, T;
  int nx, ny, nsp;
  double cy;
  const double* a1;
  const double* a2;
  const double* gam;
  double inv_ms;
  const double* Phi;   // ny dense matrices (L sweep inflow propagators)
  const double* Psi;   // ny dense matrices (U sweep)
  const double* Tl;    // NG(NG-1)/2 dense: products of group-end Phi's (L boundary pass)
  const double* Tu;    // NG(NG-1)/2 dense: products of group-start Psi's (U boundary pass)
  int g, NG, Nd;
  double* Ytil;        // per chain nsp
  double* Xtil;        // per chain nsp
  double* E;           // per chain NG x kMaxNx (L group-boundary values)
  double* F;           // per chain NG x kMaxNx (U)
};

__device__ __forceinline__ double rhs_value(const GrpParams& P, const FastStep& st, bool cres,
                                            double gn, double gm, double gp, int p) {
  double v = st.in[p] * st.scale;
  if (st.add) v += st.add[p];
  if (cres) {
    double sh = gn * P.a2[p] - gp * P.a1[p];
    if (st.node != 1) sh += gn - gm * P.a1[p];
    v -= sh * P.inv_ms;
  }
  return v;
}

// ---------------------------------------------------------------------------
// phase A, L sweep: ytilde_J = Li_J (b_J + cy Li_{J-1}^T D^{-1} ytilde_{J-1}),
// zero inflow at the group's first row
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) grpA_L_kernel(GrpParams P, const FastStep* steps,
                                                            int nsteps, int t, bool coarse) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[kSlots];
  const int grp = blockIdx.x, s = blockIdx.y;
  const FastStep st = steps[int64_t(s) * nsteps + t];
  if (!st.in) return;
  const int nx = P.nx;
  const int J0 = grp * P.g, J1 = min(P.ny, J0 + P.g) - 1;
  const int len = J1 - J0 + 1;
  auto slot = [&](int q) { return sm + (q % kSlots) * P.TP; };
  double* V = sm + kSlots * P.TP;
  double* Y0 = V;
  double* Y1 = V + kMaxNx;
  double* TV = V + 2 * kMaxNx;
  double* UV = V + 4 * kMaxNx;
  double* PART = V + 5 * kMaxNx;
  double* yt = P.Ytil + int64_t(s) * P.nsp;
  const int tid = threadIdx.x;
  const uint32_t bytes = uint32_t(P.TP) * 8u;
  int roff[kR];
  row_offsets(roff);
  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {
    if (tid == 0 && q < len) tma_load(slot(q), P.Lpk + int64_t(J0 + q) * P.TP, bytes, &bars[q % kSlots]);
  };
  auto wait = [&](int q) { mbar_wait(&bars[q % kSlots], uint32_t((q / kSlots) & 1)); };
  issue(0);
  issue(1);
  issue(2);
  const bool cres = coarse && st.node > 0;
  double gn = 0.0, gm = 0.0, gp = 0.0;
  if (cres) {
    gn = P.gam[st.node];
    gm = P.gam[st.node - 1];
    gp = P.gam[st.node + 1];
  }
  double* yprev = Y0;
  double* ycur = Y1;
  double bnext = (tid < nx) ? rhs_value(P, st, cres, gn, gm, gp, J0 * nx + tid) : 0.0;
  for (int k = 0; k < len; ++k) {
    const int J = J0 + k;
    if (tid < nx) TV[tid] = bnext;
    if (tid < nx && k + 1 < len) bnext = rhs_value(P, st, cres, gn, gm, gp, (J + 1) * nx + tid);
    wait(k);
    double vr[kK];
    if (k > 0) {
      const double* Lp = slot(k - 1);
      lowerT_mv(Lp, roff, Lp + P.T, yprev, nullptr, 0.0, PART, UV, nx);
      __syncthreads();
      load_vr(TV, UV, P.cy, vr, nx);
    } else {
      __syncthreads();
      load_vr(TV, nullptr, 0.0, vr, nx);
    }
    lower_mv(slot(k), roff, vr, ycur, nx);
    __syncthreads();
    if (tid < nx) yt[J * nx + tid] = ycur[tid];
    if (k >= 1) issue(k + 2);  // slot of position k-1 is free
    double* tmp = yprev;
    yprev = ycur;
    ycur = tmp;
  }
}

// ---------------------------------------------------------------------------
// phase A, U sweep: xtilde_J = Li_J^T D_J^{-1} (y_J + cy Li_J xtilde_{J+1}),
// zero inflow at the group's last row; one factor block per step
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) grpA_U_kernel(GrpParams P, const FastStep* steps,
                                                            int nsteps, int t) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[kSlots];
  const int grp = blockIdx.x, s = blockIdx.y;
  const FastStep st = steps[int64_t(s) * nsteps + t];
  if (!st.in) return;
  const int nx = P.nx;
  const int J0 = grp * P.g, J1 = min(P.ny, J0 + P.g) - 1;
  const int len = J1 - J0 + 1;
  auto slot = [&](int q) { return sm + (q % kSlots) * P.TP; };
  double* V = sm + kSlots * P.TP;
  double* X0 = V;
  double* X1 = V + kMaxNx;
  double* TV = V + 2 * kMaxNx;
  double* UV = V + 4 * kMaxNx;
  double* PART = V + 5 * kMaxNx;
  const double* y = P.Ytil + int64_t(s) * P.nsp;
  double* xt = P.Xtil + int64_t(s) * P.nsp;
  const int tid = threadIdx.x;
  const uint32_t bytes = uint32_t(P.TP) * 8u;
  int roff[kR];
  row_offsets(roff);
  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {
    if (tid == 0 && q < len) tma_load(slot(q), P.Lpk + int64_t(J1 - q) * P.TP, bytes, &bars[q % kSlots]);
  };
  auto wait = [&](int q) { mbar_wait(&bars[q % kSlots], uint32_t((q / kSlots) & 1)); };
  issue(0);
  issue(1);
  issue(2);
  double* xprev = X0;
  double* xcur = X1;
  double ynext = (tid < nx) ? y[J1 * nx + tid] : 0.0;
  for (int k = 0; k < len; ++k) {
    const int J = J1 - k;
    if (tid < nx) TV[tid] = ynext;
    if (tid < nx && k + 1 < len) ynext = y[(J - 1) * nx + tid];
    wait(k);
    const double* Lp = slot(k);
    if (k > 0) {
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
    if (tid < nx) xt[J * nx + tid] = xcur[tid];
    issue(k + 3);  // slot of position k is free
    double* tmp = xprev;
    xprev = xcur;
    xcur = tmp;
  }
}

// ---------------------------------------------------------------------------
// phase B: group-boundary values, all groups in parallel.  The boundary
// recurrence  e_g = yt_end(g) + Phi_end(g) e_{g-1}  (e_0 = yt_end(0)) is
// unrolled with the precomputed products T_{g,i} = Phi_end(g)...Phi_end(i+1):
//     e_g = yt_end(g) + sum_{i<g} T_{g,i} yt_end(i)
// and likewise f_g = xt_first(g) + sum_{i>g} S_{g,i} xt_first(i) for the U
// sweep (S on mirrored group indices).  One CTA per (group, chain).
// ---------------------------------------------------------------------------
__host__ __device__ inline int tri_index(int g, int i) { return g * (g - 1) / 2 + i; }  // i < g

template <bool kUpper>
__global__ void __launch_bounds__(kThreads, 1) grpB_kernel(GrpParams P, const FastStep* steps,
                                                          int nsteps, int t) {
  // let phase C launch now: its prologue (TMA of Phi_J / Psi_J) does not
  // depend on this kernel and overlaps it (programmatic dependent launch)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ double ov[kMaxNx];
  const int grp = blockIdx.x, s = blockIdx.y;
  const FastStep st = steps[int64_t(s) * nsteps + t];
  if (!st.in) return;
  const int nx = P.nx, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* til = (kUpper ? P.Xtil : P.Ytil) + int64_t(s) * P.nsp;
  double* outv = (kUpper ? P.F : P.E) + int64_t(s) * P.NG * kMaxNx;
  auto row_of = [&](int gg) { return kUpper ? gg * P.g : min(P.ny, (gg + 1) * P.g) - 1; };
  // mirrored index for the U sweep: group gg -> NG-1-gg
  const int gm = kUpper ? P.NG - 1 - grp : grp;
  double acc[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) acc[r] = 0.0;
  for (int im = 0; im < gm; ++im) {
    const int i = kUpper ? P.NG - 1 - im : im;  // source group
    const double* src = til + row_of(i) * nx;
    double vr[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      const int b = lane + 32 * k;
      vr[k] = b < nx ? src[b] : 0.0;
    }
    const double* M = (kUpper ? P.Tu : P.Tl) + int64_t(tri_index(gm, im)) * kDense;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int a = warp + kWarps * r;
      if (a < nx) {
        const double* row = M + a * kLd;
#pragma unroll
        for (int k = 0; k < kK; ++k) acc[r] = fma(row[lane + 32 * k], vr[k], acc[r]);
      }
    }
  }
  rows_reduce_store(acc, ov, nx);
  __syncthreads();
  if (tid < kMaxNx) {
    const double v = tid < nx ? til[row_of(grp) * nx + tid] + (gm > 0 ? ov[tid] : 0.0) : 0.0;
    outv[grp * kMaxNx + tid] = v;
  }
}

// ---------------------------------------------------------------------------
// phase C: one CTA per block row J; all chains at once as a small GEMM on the
// fp64 tensor cores (mma.sync m8n8k4 f64):  Out[a][s] = sum_b M_J[a][b] In[s][b]
//   L: Ytil[s][J] += Phi_J E[s][g-1]                     (g > 0)
//   U: out[s][J] = Xtil[s][J] + Psi_J F[s][g+1] (g < NG-1), out2 = out + gamma
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool kUpper>
__global__ void __launch_bounds__(kThreads, 1) grpC_kernel(GrpParams P, const FastStep* steps,
                                                          int nsteps, int t) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double* s_out[kCBatch];
  __shared__ double* s_out2[kCBatch];
  __shared__ double s_g2[kCBatch];
  __shared__ int s_act[kCBatch];
  const int J = blockIdx.x;
  const int grp = J / P.g;
  const bool has_inflow = kUpper ? (grp < P.NG - 1) : (grp > 0);
  if (!kUpper && !has_inflow) return;  // ytilde is already y in the first group
  const int nx = P.nx, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Mj = sm;                       // kDense
  double* In = sm + kDense;              // kCBatch x kLd   (operand, then the product)
  if (has_inflow && tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_load(Mj, (kUpper ? P.Psi : P.Phi) + int64_t(J) * kDense, uint32_t(kDense) * 8u, &bar);
  }
  // everything below reads phase B's outputs
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int src_grp = kUpper ? grp + 1 : grp - 1;
  const double* til = kUpper ? P.Xtil : P.Ytil;
  const double* bv = kUpper ? P.F : P.E;
  bool waited = false;
  for (int s0 = 0; s0 < P.Nd; s0 += kCBatch) {
    const int nb = min(kCBatch, P.Nd - s0);
    if (tid < kCBatch) {
      const int s = s0 + tid;
      int act = 0;
      double* o = nullptr;
      double* o2 = nullptr;
      double g2 = 0.0;
      if (tid < nb) {
        const FastStep st = steps[int64_t(s) * nsteps + t];
        act = st.in != nullptr;
        o = st.out;
        o2 = st.out2;
        g2 = (st.out2 && st.node2 > 0 && P.gam) ? P.gam[st.node2] : 0.0;
      }
      s_act[tid] = act;
      s_out[tid] = o;
      s_out2[tid] = o2;
      s_g2[tid] = g2;
    }
    __syncthreads();
    if (has_inflow) {
      for (int i = tid; i < kCBatch * kLd; i += blockDim.x) {
        const int c = i / kLd, b = i - c * kLd;
        In[i] = (c < nb && b < nx && s_act[c]) ? bv[(int64_t(s0 + c) * P.NG + src_grp) * kMaxNx + b] : 0.0;
      }
      if (!waited) {
        mbar_wait(&bar, 0);
        waited = true;
      }
      __syncthreads();
      // 16 row tiles x 2 chain tiles: warp w -> row tile w; K = 128 in 32 steps of 4
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
      const int ar = warp * 8 + (lane >> 2);
      const int kc = lane & 3;
#pragma unroll 8
      for (int ks = 0; ks < kLd / 4; ++ks) {
        const double a = Mj[ar * kLd + ks * 4 + kc];
        const double b0 = In[(lane >> 2) * kLd + ks * 4 + kc];
        const double b1 = In[(8 + (lane >> 2)) * kLd + ks * 4 + kc];
        dmma(d00, d01, a, b0);
        dmma(d10, d11, a, b1);
      }
      __syncthreads();  // In is overwritten with the product below
      // D fragment: row = 8w + lane/4, chain = 2*(lane%4) + {0,1} (+8 for tile 1)
      const int c0 = 2 * (lane & 3);
      In[c0 * kLd + ar] = d00;
      In[(c0 + 1) * kLd + ar] = d01;
      In[(8 + c0) * kLd + ar] = d10;
      In[(9 + c0) * kLd + ar] = d11;
      __syncthreads();
    }
    // coalesced row updates: chain c, rows a
    for (int i = tid; i < nb * nx; i += blockDim.x) {
      const int c = i / nx, a = i - c * nx;
      if (!s_act[c]) continue;
      const int s = s0 + c;
      const int64_t p = int64_t(J) * nx + a;
      const double d = has_inflow ? In[c * kLd + a] : 0.0;
      if (!kUpper) {
        P.Ytil[int64_t(s) * P.nsp + p] += d;
      } else {
        const double x = til[int64_t(s) * P.nsp + p] + d;
        if (s_out[c]) s_out[c][p] = x;
        if (s_out2[c]) s_out2[c][p] = x + s_g2[c];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// setup: dense G_J, H_J and the in-group products Phi_J, Psi_J (kLd x kLd,
// zero padded), from the square inverse blocks Li (nx x nx) and D^{-1}.
// ---------------------------------------------------------------------------
// G_J(a,b) = cy Dinv_{J-1}(b) sum_{k<=min(a,b)} Li_J(a,k) Li_{J-1}(b,k)   (J >= 1)
// H_J(a,b) = cy sum_{k>=max(a,b)} Li_J(k,a) Dinv_J(k) Li_J(k,b)
__global__ void gh_kernel(int nx, int ny, double cy, const double* __restrict__ Li,
                          const double* __restrict__ dinv, double* __restrict__ G,
                          double* __restrict__ H) {
  const int J = blockIdx.x;
  const int64_t nn = int64_t(nx) * nx;
  const double* LJ = Li + J * nn;
  const double* LP = J > 0 ? Li + (J - 1) * nn : nullptr;
  for (int e = threadIdx.x; e < kDense; e += blockDim.x) {
    const int a = e / kLd, b = e - a * kLd;
    double g = 0.0, h = 0.0;
    if (a < nx && b < nx) {
      if (LP) {
        const int kmax = min(a, b);
        for (int k = 0; k <= kmax; ++k) g = fma(LJ[a * nx + k], LP[b * nx + k], g);
        g *= cy * dinv[(J - 1) * nx + b];
      }
      const int kmin = max(a, b);
      for (int k = kmin; k < nx; ++k) h = fma(LJ[k * nx + a] * dinv[J * nx + k], LJ[k * nx + b], h);
      h *= cy;
    }
    G[int64_t(J) * kDense + e] = g;
    H[int64_t(J) * kDense + e] = h;
  }
}

// C_i = A_i B_i for a batch of (dst, a, b) matrix index triples (kLd x kLd)
__global__ void mm_batch_kernel(const int* __restrict__ trip, const double* __restrict__ Abase,
                                const double* __restrict__ Bbase, double* __restrict__ Cbase) {
  const int* tr = trip + 3 * blockIdx.x;
  const double* A = Abase + int64_t(tr[1]) * kDense;
  const double* B = Bbase + int64_t(tr[2]) * kDense;
  double* C = Cbase + int64_t(tr[0]) * kDense;
  for (int e = threadIdx.x; e < kDense; e += blockDim.x) {
    const int a = e / kLd, b = e - a * kLd;
    double acc = 0.0;
    for (int k = 0; k < kLd; ++k) acc = fma(A[a * kLd + k], B[k * kLd + b], acc);
    C[e] = acc;
  }
}

__global__ void copy_mat_kernel(const int* __restrict__ pairs, const double* __restrict__ src,
                                double* __restrict__ dst) {
  const int* pr = pairs + 2 * blockIdx.x;
  for (int e = threadIdx.x; e < kDense; e += blockDim.x)
    dst[int64_t(pr[0]) * kDense + e] = src[int64_t(pr[1]) * kDense + e];
}

__global__ void dinv_kernel(int nx, int ny, int kuf, int ld, const double* __restrict__ ab,
                            double* __restrict__ dinv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nx * ny) dinv[i] = 1.0 / ab[int64_t(i) * ld + kuf];
}

GrpParams params(Ctx* c) {
  GrpParams P;
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
  P.Phi = c->Phi.p;
  P.Psi = c->Psi.p;
  P.Tl = c->grp_tl.p;
  P.Tu = c->grp_tu.p;
  P.g = c->grp_g;
  P.NG = c->grp_n;
  P.Nd = c->Nd;
  P.Ytil = c->grp_y.p;
  P.Xtil = c->grp_x.p;
  P.E = c->grp_e.p;
  P.F = c->grp_f.p;
  return P;
}

size_t smemA(const Ctx* c) {
  return sizeof(double) * (size_t(kSlots) * c->Lpk_stride + size_t(5 + kWarps) * kMaxNx);
}
size_t smemC() { return sizeof(double) * (size_t(kDense) + size_t(kCBatch) * kLd); }

// Launch with programmatic stream serialization: the kernel may start while
// its predecessor runs and must call griddepcontrol.wait before reading it.
template <class K>
void launch_pdl(Ctx* c, K kernel, int grid, size_t smem, const GrpParams& P, const FastStep* jobs,
                int nsteps, int t) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KKT_CUDA(cudaLaunchKernelEx(&cfg, kernel, P, jobs, nsteps, t));
  c->launches++;
}

}  // namespace

bool group_supported(const Ctx* c) { return c->nx <= kMaxNx && c->ny >= 2; }

// Move Lpk, Phi, Psi, Tl, Tu into one allocation; with KKT_L2PIN=1 it is also
// marked L2-persisting on the context stream (the sweep re-reads these 50 MB
// every time step while the 198 MB Krylov vectors stream through L2).
void pin_operators_in_l2(Ctx* c) {
  DBuf<double>* parts[] = {&c->Lpk, &c->Phi, &c->Psi, &c->grp_tl, &c->grp_tu};
  size_t total = 0;
  for (auto* b : parts) total += (b->n + 31) & ~size_t(31);  // 256-byte aligned pieces
  c->arena.alloc(total);
  size_t off = 0;
  for (auto* b : parts) {
    const size_t n = b->n;
    KKT_CUDA(cudaMemcpyAsync(c->arena.p + off, b->p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    b->view(c->arena.p + off, n);
    off += (n + 31) & ~size_t(31);
  }
  int max_persist = 0, max_window = 0;
  KKT_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device));
  KKT_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device));
  // opt-in: measured neutral at config 1 (409.8 vs 411.6 ms per solve), and the
  // persisting carve-out is a device-wide setting
  if (max_persist <= 0 || max_window <= 0 || !getenv("KKT_L2PIN")) return;
  const size_t bytes = std::min(sizeof(double) * total, size_t(max_window));
  const size_t carve = std::min(bytes, size_t(max_persist));
  KKT_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
  cudaStreamAttrValue attr{};
  attr.accessPolicyWindow.base_ptr = c->arena.p;
  attr.accessPolicyWindow.num_bytes = bytes;
  attr.accessPolicyWindow.hitRatio = float(std::min(1.0, double(carve) / double(bytes)));
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  KKT_CUDA(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr));
}

// Build Phi/Psi from the square inverse blocks (called while Li is alive).
void build_group_operators(Ctx* c) {
  const int nx = c->nx, ny = c->ny;
  // group size: balance phase A (g steps) against phase B (NG-1 steps), keeping
  // NG * Nd phase-A CTAs within one wave of the 148 SMs
  const bool v4 = v4_supported(c);
  int g = 16;
  while (g > 4 && (ny + g - 1) / g * c->Nd <= kSmCount / 2) g /= 2;
  while ((ny + g - 1) / g * c->Nd > kSmCount && g < ny) g *= 2;
  if (v4) g = v4_group_size(c);  // v4: one wave of 8-CTA clusters per chain set
  if (g > ny) g = ny;
  c->grp_g = g;
  c->grp_n = (ny + g - 1) / g;
  DBuf<double> dinv(size_t(nx) * ny);
  KKT_LAUNCH(c, dinv_kernel, (nx * ny + 255) / 256, 256, 0, nx, ny, c->kuf, c->ld, c->ab.p, dinv.p);
  DBuf<double> G(size_t(ny) * kDense), H(size_t(ny) * kDense);
  KKT_LAUNCH(c, gh_kernel, ny, 256, 0, nx, ny, c->cy, c->Li.p, dinv.p, G.p, H.p);
  c->Phi.alloc(size_t(ny) * kDense);
  c->Psi.alloc(size_t(ny) * kDense);
  KKT_CUDA(cudaMemsetAsync(c->Phi.p, 0, sizeof(double) * c->Phi.n, c->stream));
  KKT_CUDA(cudaMemsetAsync(c->Psi.p, 0, sizeof(double) * c->Psi.n, c->stream));
  DBuf<int> idx(size_t(3) * c->grp_n);
  // Phi: first row of each group (J0 >= 1): Phi = G; then Phi_J = G_J Phi_{J-1}
  // Psi: last row of each group (J1 <= ny-2): Psi = H; then Psi_J = H_J Psi_{J+1}
  std::vector<int> pairs, trips;
  for (int grp = 0; grp < c->grp_n; ++grp) {
    const int J0 = grp * g, J1 = std::min(ny, J0 + g) - 1;
    if (J0 >= 1) { pairs.push_back(J0); pairs.push_back(J0); }
  }
  auto run_copy = [&](const double* src, double* dst) {
    if (pairs.empty()) return;
    DBuf<int> d(pairs.size());
    KKT_CUDA(cudaMemcpyAsync(d.p, pairs.data(), sizeof(int) * pairs.size(), cudaMemcpyHostToDevice, c->stream));
    KKT_LAUNCH(c, copy_mat_kernel, int(pairs.size() / 2), 256, 0, d.p, src, dst);
    KKT_CUDA(cudaStreamSynchronize(c->stream));
  };
  run_copy(G.p, c->Phi.p);
  pairs.clear();
  for (int grp = 0; grp < c->grp_n; ++grp) {
    const int J0 = grp * g, J1 = std::min(ny, J0 + g) - 1;
    if (J1 <= ny - 2) { pairs.push_back(J1); pairs.push_back(J1); }
  }
  run_copy(H.p, c->Psi.p);
  for (int k = 1; k < g; ++k) {
    // Phi chains
    trips.clear();
    for (int grp = 0; grp < c->grp_n; ++grp) {
      const int J0 = grp * g, J1 = std::min(ny, J0 + g) - 1;
      const int J = J0 + k;
      if (J0 >= 1 && J <= J1) { trips.push_back(J); trips.push_back(J); trips.push_back(J - 1); }
    }
    if (!trips.empty()) {
      DBuf<int> d(trips.size());
      KKT_CUDA(cudaMemcpyAsync(d.p, trips.data(), sizeof(int) * trips.size(), cudaMemcpyHostToDevice, c->stream));
      KKT_LAUNCH(c, mm_batch_kernel, int(trips.size() / 3), 256, 0, d.p, G.p, c->Phi.p, c->Phi.p);
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
    // Psi chains
    trips.clear();
    for (int grp = 0; grp < c->grp_n; ++grp) {
      const int J0 = grp * g, J1 = std::min(ny, J0 + g) - 1;
      const int J = J1 - k;
      if (J1 <= ny - 2 && J >= J0) { trips.push_back(J); trips.push_back(J); trips.push_back(J + 1); }
    }
    if (!trips.empty()) {
      DBuf<int> d(trips.size());
      KKT_CUDA(cudaMemcpyAsync(d.p, trips.data(), sizeof(int) * trips.size(), cudaMemcpyHostToDevice, c->stream));
      KKT_LAUNCH(c, mm_batch_kernel, int(trips.size() / 3), 256, 0, d.p, H.p, c->Psi.p, c->Psi.p);
      KKT_CUDA(cudaStreamSynchronize(c->stream));
    }
  }
  (void)idx;
  // boundary-pass products: Tl_{g,i} = Phi_end(g) Tl_{g-1,i}, Tl_{g,g-1} = Phi_end(g);
  // Tu on mirrored indices with Psi_first
  const int NG = c->grp_n;
  const int ntri = std::max(1, NG * (NG - 1) / 2);
  c->grp_tl.alloc(size_t(ntri) * kDense);
  c->grp_tu.alloc(size_t(ntri) * kDense);
  auto end_row = [&](int gg) { return std::min(ny, (gg + 1) * g) - 1; };
  auto first_row = [&](int gg) { return gg * g; };
  for (int side = 0; side < 2; ++side) {
    const double* src = side == 0 ? c->Phi.p : c->Psi.p;
    double* T = side == 0 ? c->grp_tl.p : c->grp_tu.p;
    for (int gm = 1; gm < NG; ++gm) {
      const int gg = side == 0 ? gm : NG - 1 - gm;
      const int J = side == 0 ? end_row(gg) : first_row(gg);
      // T_{gm, gm-1} = M_J
      KKT_CUDA(cudaMemcpyAsync(T + size_t(tri_index(gm, gm - 1)) * kDense, src + size_t(J) * kDense,
                               sizeof(double) * kDense, cudaMemcpyDeviceToDevice, c->stream));
      if (gm >= 2) {
        // T_{gm, i} = M_J T_{gm-1, i}, i < gm-1: dst/A/B index triples relative to
        // separate bases -> stage M_J as matrix 0 of a scratch base
        trips.clear();
        for (int i = 0; i < gm - 1; ++i) {
          trips.push_back(tri_index(gm, i));
          trips.push_back(J);
          trips.push_back(tri_index(gm - 1, i));
        }
        DBuf<int> d(trips.size());
        KKT_CUDA(cudaMemcpyAsync(d.p, trips.data(), sizeof(int) * trips.size(), cudaMemcpyHostToDevice, c->stream));
        KKT_LAUNCH(c, mm_batch_kernel, int(trips.size() / 3), 256, 0, d.p, src, T, T);
        KKT_CUDA(cudaStreamSynchronize(c->stream));
      }
    }
  }
  if (v4) {
    build_v4(c, G.p, H.p, c->Li.p, dinv.p);
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    c->Phi.release();
    c->Psi.release();
    c->grp_tl.release();
    c->grp_tu.release();
    return;
  }
  pin_operators_in_l2(c);
  c->grp_y.alloc(size_t(c->Nd) * c->nsp);
  c->grp_x.alloc(size_t(c->Nd) * c->nsp);
  c->grp_e.alloc(size_t(c->Nd) * c->grp_n * kMaxNx);
  c->grp_f.alloc(size_t(c->Nd) * c->grp_n * kMaxNx);
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  static bool attr = false;
  if (!attr) {
    const int big = int(sizeof(double) * (size_t(kSlots) * (((kMaxNx * (kMaxNx + 1)) / 2 + kMaxNx + 1) & ~1) +
                                          size_t(5 + kWarps) * kMaxNx));
    KKT_CUDA(cudaFuncSetAttribute(grpA_L_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    KKT_CUDA(cudaFuncSetAttribute(grpA_U_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    KKT_CUDA(cudaFuncSetAttribute(grpC_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemC())));
    KKT_CUDA(cudaFuncSetAttribute(grpC_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemC())));
    attr = true;
  }
}

// Run `nsteps` lock-step spatial solves of `nchains` chains (chain-major job
// table on the device), phases A/B/C for the L then the U sweep per step.
void group_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms) {
  GrpParams P = params(c);
  P.Nd = nchains;
  if (size_t(nchains) * c->nsp > c->grp_y.n) {
    c->grp_y.alloc(size_t(nchains) * c->nsp);
    c->grp_x.alloc(size_t(nchains) * c->nsp);
    c->grp_e.alloc(size_t(nchains) * c->grp_n * kMaxNx);
    c->grp_f.alloc(size_t(nchains) * c->grp_n * kMaxNx);
    P = params(c);
    P.Nd = nchains;
  }
  const dim3 gA(c->grp_n, nchains);
  const size_t sA = smemA(c), sC = smemC();
  auto sequence = [&]() {
    for (int t = 0; t < nsteps; ++t) {
      KKT_LAUNCH(c, grpA_L_kernel, gA, kThreads, sA, P, jobs_dev, nsteps, t, coarse_terms);
      KKT_LAUNCH(c, grpB_kernel<false>, gA, kThreads, 0, P, jobs_dev, nsteps, t);
      launch_pdl(c, grpC_kernel<false>, c->ny, sC, P, jobs_dev, nsteps, t);
      KKT_LAUNCH(c, grpA_U_kernel, gA, kThreads, sA, P, jobs_dev, nsteps, t);
      KKT_LAUNCH(c, grpB_kernel<true>, gA, kThreads, 0, P, jobs_dev, nsteps, t);
      launch_pdl(c, grpC_kernel<true>, c->ny, sC, P, jobs_dev, nsteps, t);
    }
  };
  // The 6*nsteps launches of one application are replayed from a CUDA graph:
  // the job table is a fixed device buffer refreshed before each replay, so
  // the captured kernel arguments stay valid.
  static const bool no_graph = getenv("KKT_NO_GRAPH") != nullptr;
  if (no_graph) {
    c->tbegin(3);
    sequence();
    c->tend(3);
    return;
  }
  Ctx::Graph* gr = nullptr;
  for (auto& e : c->graphs)
    if (e.jobs == jobs_dev && e.nchains == nchains && e.nsteps == nsteps && e.coarse == coarse_terms &&
        e.y == c->grp_y.p)
      gr = &e;
  if (!gr) {
    Ctx::Graph e;
    e.jobs = jobs_dev;
    e.nchains = nchains;
    e.nsteps = nsteps;
    e.coarse = coarse_terms;
    e.y = c->grp_y.p;
    const int64_t l0 = c->launches;
    cudaGraph_t graph;
    KKT_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    sequence();
    KKT_CUDA(cudaStreamEndCapture(c->stream, &graph));
    KKT_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
    KKT_CUDA(cudaGraphDestroy(graph));
    e.nlaunch = c->launches - l0;
    c->launches = l0;
    c->graphs.push_back(e);
    gr = &c->graphs.back();
  }
  c->tbegin(3);
  KKT_CUDA(cudaGraphLaunch(gr->exec, c->stream));
  c->launches += gr->nlaunch;
  c->tend(3);
}

}  // namespace kkt
