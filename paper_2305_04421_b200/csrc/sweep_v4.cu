// sweep_v4.cu — FAST spatial-solve chains, v4: cluster-cooperative block
// substitution with every local subdomain batched into fp64 tensor-core tiles
// (nx <= 128: configs 0 and 1).
//
// The method is the reference's LU solve (BandedLU::solve_in_place /
// solve_transpose_in_place, linalg.cpp:127-162) in the block form of
// sweep_group.cu, for the pivot-free factor of the symmetric Ahat:
//     L sweep  y_J = c_J + G_J y_{J-1},  c_J = Li_J b_J,
//              G_J = cy Li_J Li_{J-1}^T D_{J-1}^{-1}
//     U sweep  x_J = d_J + H_J x_{J+1},  d_J = Ut_J y_J,  Ut_J = Li_J^T D_J^{-1},
//              H_J = cy Ut_J Li_J
// with the ny block rows cut into NG groups of g rows (zero-inflow chains per
// group, group-boundary values from precomputed propagator products, inflow
// corrections y_J += Phi_J e_{G-1} / x_J += Psi_J f_{G+1}) exactly as in v3.
// What changes is the mapping onto the machine:
//
//  * A time step is two kernels, one per sweep direction (A_L, A_U); one
//    RASQ application is 2(2m+1)+1 launches, chained with programmatic
//    dependent launch and replayed from a CUDA graph.
//  * Each group's chain of g block steps runs on a cluster of 8 CTAs.  CTA r
//    owns block rows 16r..16r+15 of every step and computes them for ALL 16
//    chains of a chain set at once as 2x2 m8n8k4 fp64 DMMA tiles, so each
//    operator element read from shared memory serves 16 right-hand sides.
//    The 16-row result slice of a step goes to the 7 peer CTAs with st.async
//    (DSMEM, mbarrier transaction counts), double-buffered.
//  * Warp specialisation: warps 0-3 run the dependent chain (one tile each);
//    warps 4-7 compute the off-chain term of the rows ahead (c_J / d_J),
//    handed over through shared memory (mbarriers cready/cfree), write the
//    previous step's outputs and keep two TMA rings of operator slices full.
//  * The inflow correction of the previous direction is folded into the
//    off-chain term through precomputed products: the L sweep's right-hand
//    side x_{t-1} = x~_{t-1} + Psi f enters as Li x~ + (Li Psi) f, the U
//    sweep's y = y~ + Phi e as Ut y~ + (Ut Phi) e, so no correction pass
//    sits between the chains.
//  * B (group-boundary values from precomputed propagator products) runs at
//    the tail of each A kernel: each cluster multiplies its own group-end
//    vector (exchanged to all its CTAs) into its targets' partials, pairs of
//    clusters i <-> NG-1-i balance the work, and a release/acquire flag
//    publishes the vector a partner borrows.  The consumer sums the partials
//    in a fixed order: deterministic.  All clusters of the grid are
//    co-resident (v4_group_size), so the cross-cluster waits cannot deadlock.
//
// Layouts.  Matrices (128x128, zero padded) are stored "fragment ordered":
// slice r (rows 16r..16r+15) = [ks 32][rt 2][lane 32] with element
// M[16r+8rt+lane/4][4ks+lane%4], the A operand of m8n8k4 read as 32
// consecutive doubles per warp.  A block vector of 128 rows x 16 chains is
// [ks 32][ct 2][kl 4][nl 8] (row 4ks+kl, chain 8ct+nl): the B operand reads
// 32 consecutive doubles, the D fragment writes chain pairs as double2, and
// the rows of CTA r are the contiguous doubles [256r, 256r+256).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sweep_tma.cuh"

namespace kkt {
namespace {
using namespace tma;

constexpr int kN = 128;              // padded block size (== kMaxNx)
constexpr int kCs = 16;              // chains per chain set
constexpr int kCl = 8;               // CTAs per cluster
constexpr int kRows = kN / kCl;      // 16 block rows per CTA
constexpr int kSlice = kRows * kN;   // doubles per matrix slice (16 KB)
constexpr int kMat = kN * kN;        // doubles per matrix
constexpr int kVec = kN * kCs;       // doubles per block vector of a chain set
constexpr int kThr4 = 256;
constexpr int kCMax = 9;
constexpr int kMaxSrc = 18;          // group-boundary sources per inflow vector (NG - 1 <= 148 / kCl)             // C-part operator slices in flight (the slab aliases ring + X + V)

__host__ __device__ inline int tri_idx(int g, int i) { return g * (g - 1) / 2 + i; }  // i < g

__device__ __forceinline__ int vidx(int k, int n) {
  return (k >> 2) * 64 + (n >> 3) * 32 + (k & 3) * 8 + (n & 7);
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(par)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void dmma4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// All 8 warps: D[16 rows x 16 chains] (+)= A_slice[16 x 128] x B[128 x 16]
// over k-steps [kb, ke).  Warp w owns tile (rt, ct) = ((w&3)>>1, w&1) and half
// of the k range; the halves are summed through `part`, leaving the result in
// the kh == 0 warps (w < 4), in D-fragment layout.  Contains __syncthreads.
__device__ __forceinline__ void cta_mma(const double* A, const double* B, int kb, int ke, double* part,
                                        double& d0, double& d1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = warp & 3, rt = t >> 1, ct = t & 1, kh = warp >> 2;
  const int mid = kb + (((ke - kb) >> 1) & ~3);
  const int lo = kh ? mid : kb, hi = kh ? ke : mid;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
  const int boff = ct * 32 + (lane & 3) * 8 + (lane >> 2);
  int ks = lo;
  for (; ks + 4 <= hi; ks += 4) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      av[u] = A[((ks + u) * 2 + rt) * 32 + lane];
      bv[u] = B[(ks + u) * 64 + boff];
    }
    dmma4(a0, a1, av[0], bv[0]);
    dmma4(b0, b1, av[1], bv[1]);
    dmma4(c0, c1, av[2], bv[2]);
    dmma4(e0, e1, av[3], bv[3]);
  }
  for (; ks < hi; ++ks) dmma4(a0, a1, A[(ks * 2 + rt) * 32 + lane], B[ks * 64 + boff]);
  double p0 = (a0 + b0) + (c0 + e0), p1 = (a1 + b1) + (c1 + e1);
  if (kh) {
    part[(t * 32 + lane) * 2] = p0;
    part[(t * 32 + lane) * 2 + 1] = p1;
  }
  __syncthreads();
  if (!kh) {
    d0 += p0 + part[(t * 32 + lane) * 2];
    d1 += p1 + part[(t * 32 + lane) * 2 + 1];
  }
  __syncthreads();  // part reusable, all operand reads done
}

// One warp: tile (rt, ct) of D[16 rows x 16 chains] (+)= A_slice x B over
// k-steps [kb, ke): 4 independent accumulators, operands of the next 4
// k-steps loaded while the current ones are in the tensor pipe.
__device__ __forceinline__ void warp_mma(const double* A, const double* B, int kb, int ke, int rt, int ct,
                                         double& d0, double& d1) {
  const int lane = threadIdx.x & 31;
  double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  const double* Ap = A + rt * 32 + lane;                               // + ks * 64
  const double* Bp = B + ct * 32 + (lane & 3) * 8 + (lane >> 2);      // + ks * 64
  int ks = kb;
  const int n4 = (ke - kb) >> 2;
  if (n4 > 0) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      av[u] = Ap[(ks + u) * 64];
      bv[u] = Bp[(ks + u) * 64];
    }
    for (int it = 1; it < n4; ++it) {
      double an[4], bn[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        an[u] = Ap[(ks + 4 + u) * 64];
        bn[u] = Bp[(ks + 4 + u) * 64];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma4(acc[u][0], acc[u][1], av[u], bv[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = an[u];
        bv[u] = bn[u];
      }
      ks += 4;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma4(acc[u][0], acc[u][1], av[u], bv[u]);
    ks += 4;
  }
  for (; ks < ke; ++ks) dmma4(acc[0][0], acc[0][1], Ap[ks * 64], Bp[ks * 64]);
  d0 += (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
  d1 += (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

struct V4Params {
  // fragment-ordered operators, ny matrices each (T: NG(NG-1)/2)
  const double* OnL;   // G_J
  const double* OffL;  // Li_J
  const double* OnU;   // H_J
  const double* OffU;  // Ut_J
  const double* UPhi;  // Ut_J Phi_J: L inflow propagators seen by the U sweep's d_J
  const double* Psi;   // U inflow propagators (outputs of the L kernel)
  const double* LPsi;  // Li_J Psi_J: U inflow propagators seen by the L sweep's c_J
  const double* TL;    // L boundary products
  const double* TU;    // U boundary products (mirrored indices)
  // state
  double* Yt;          // [set][ny][kVec]: y~ per block row, block-vector fragment layout
  double* Xh;          // [step][set][ny][kVec]: x~ of every step (fragment layout)
  double* Fh;          // [step][set][NG][kVec]: the U boundary values f_G of every step
  double* Rin;         // [step][set][ny][kVec]: the external `in` operands, gathered
  const int* insrc;    // [chain][step]: t' when in(t) == out(t') (t' < t), else -1
  const int* live;     // [chain][step]: bit 0 out, bit 1 out2 is the plane's final write
  double* Yend;        // [set][NG][kVec]: ytilde at each group's last row
  double* Xend;        // [set][NG][kVec]: xtilde at each group's first row
  double* EP;          // [set][NG target][NG source][kVec]: TL products (L)
  double* FP;          // [set][NG target][NG source][kVec]: TU products (U)
  unsigned* flagL;     // [set][NG]: group-end vector published (L kernel)
  unsigned* flagU;     // [set][NG] (U kernel)
  // problem
  const double* a1;
  const double* a2;
  const double* gam;
  double inv_ms;
  int nx, ny, nsp, g, NG, nchains, nsets;
  const FastStep* jobs;
  int nsteps;
  int coarse;
  long long* tim;      // debug (KKT_V4_TIM): per-CTA clock64 marks, null in production
  unsigned long long* tl;  // debug (KKT_V4_TL): [2*step + kU][CTA][4] globaltimer marks
  const double* zeros; // kN zeros: load target of masked-out lanes (branch-free loads)
  const double* LA;    // [J][3][kN]: Li_J a2, Li_J a1, Li_J 1 (two-level residual term)
  int empty;           // debug: KKT_V4_EMPTY=1 kernels return at once (launch floor)
};


// ---------------------------------------------------------------------------
// A kernel: the zero-inflow chain of one group for one chain set on one 8-CTA
// cluster (CTA r: block rows 16r..16r+15).  Time step t:
//   L (kU = false):  y~_J = c_J + G_J y~_{J-1},
//        c_J = Li_J b~_J + (Li Psi)_J f~ - coarse_J
//     Every step output is x_t = x~_t + Psi f(t) (the inflow correction of the
//     U sweep); x~_t and f(t) are kept per step (Xh, Fh), so an operand that is
//     an earlier output — add = x_{t-1} (FastStep.add is the previous step's
//     out, sweep.cu), or in = x_{t'} at the adjoint steps — enters as
//     b~ = in*scale + x~_{t-1} (x~_{t'} for in) and f~ = f(t-1) (+ scale
//     f(t')) per chain, through the precomputed Li_J Psi_J.  External `in`
//     planes are gathered into fragment layout once per application (Rin);
//     the outputs are written once at the end (v4_out_kernel).
//   U (kU = true):   x~_J = d_J + H_J x~_{J+1},
//        d_J = Ut_J y~_J + (Ut Phi)_J e_{G-1}      (y_J = y~_J + Phi_J e_{G-1})
// Warps 0-3 run the dependent chain (one output tile each): wait for the
// peers' slices of the previous row, + G_J y~_{J-1} (H_J x~_{J+1}), + the
// off-chain tile, send the slice to the peers.  Warps 4-7 compute the
// off-chain tiles of the rows ahead, load the operands and refill the
// operator rings.
// ---------------------------------------------------------------------------
template <bool kU>
__global__ void __launch_bounds__(kThr4, 1) v4A_kernel(V4Params P, int t, int final_only) {
  extern __shared__ __align__(128) double sm[];
  double* ringC = sm;                    // 3 on-chain slices
  double* ringO = ringC + 3 * kSlice;    // 2 x (triangle, M1, M2) off-chain slices
  double* X = ringO + 6 * kSlice;        // 2 exchange buffers
  double* V = X + 2 * kVec;              // off-chain operand
  double* EV = V + kVec;                 // inflow vector f_{G+1} (L) / e_{G-1} (U)
  double* Cb = EV + kVec;                // 2 x 256: off-chain tiles
  double* part = Cb + 2 * 256;           // k-half partials (B tail)
  __shared__ __align__(8) uint64_t tbarC[3], tbarO[2], sfreeC[3], sfreeO[2], xbar[2], cready[2], cfree[2];
  __shared__ __align__(8) uint64_t cbar[kCMax];
  __shared__ FastStep sj[kCs];   // jobs of step t
  __shared__ int sinp[kCs];      // per chain: t' when in(t) == out(t'), else -1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = int(cta_rank());
  const int cid = blockIdx.x / kCl;
  const int G = cid % P.NG, set = cid / P.NG;
  const int J0 = G * P.g, J1 = min(P.ny, J0 + P.g) - 1, len = J1 - J0 + 1;
  const int NG = P.NG;
  const bool inflow = kU ? (G > 0) : (G < NG - 1);
  // chain state of block row J (this chain set), block-vector fragment layout
  auto frow = [&](double* base, int J) { return base + (size_t(set) * P.ny + J) * kVec; };
  const size_t hstep = size_t(P.nsets) * P.ny * kVec;  // one step of Xh / Rin
  const bool chain = !final_only;
  const double* On = kU ? P.OnU : P.OnL;
  const double* Off = kU ? P.OffU : P.OffL;
  const double* M1 = kU ? P.UPhi : P.LPsi;
  // off-chain triangle: Li lower (ks < 4r+4), Ut upper (ks >= 4r)
  const int okb = kU ? 4 * r : 0, oke = kU ? 32 : 4 * r + 4;
  auto rowQ = [&](int q) { return kU ? J1 - q : J0 + q; };
  const uint32_t tri_bytes = uint32_t(oke - okb) * 64 * 8;
  // on-chain stage u = row u+1 (row 0 has no inflow), slot u % 3
  auto issue_on = [&](int u) {
    if (u + 1 >= len) return;
    const int J = rowQ(u + 1);
    mbar_expect_tx(&tbarC[u % 3], kSlice * 8);
    bulk_g2s(ringC + (u % 3) * kSlice, On + (size_t(J) * kCl + r) * kSlice, kSlice * 8, &tbarC[u % 3]);
  };
  // off-chain stage q = row q, slot q % 2: triangle (+ M1)
  const bool use_m1 = inflow && (kU || t > 0);
  // (U: the third slot takes the operand y~_J itself, 16 KB from the previous
  // kernel, so it is copied only after griddepcontrol.wait: issue_off_v)
  auto issue_off = [&](int q) {
    if (q >= len) return;
    const int J = rowQ(q);
    double* dst = ringO + (q & 1) * 3 * kSlice;
    const size_t sl = (size_t(J) * kCl + r) * kSlice;
    mbar_expect_tx(&tbarO[q & 1], tri_bytes + (use_m1 ? kSlice * 8 : 0) + (kU ? kSlice * 8 : 0));
    bulk_g2s(dst + okb * 64, Off + sl + okb * 64, tri_bytes, &tbarO[q & 1]);
    if (use_m1) bulk_g2s(dst + kSlice, M1 + sl, kSlice * 8, &tbarO[q & 1]);
  };
  auto issue_off_v = [&](int q) {
    if (!kU || q >= len) return;
    bulk_g2s(ringO + (q & 1) * 3 * kSlice + 2 * kSlice, frow(P.Yt, rowQ(q)), kVec * 8, &tbarO[q & 1]);
  };
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(&tbarC[i], 1);
      mbar_init(&sfreeC[i], 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tbarO[i], 1);
      mbar_init(&sfreeO[i], 128);
      mbar_init(&xbar[i], 1);
      mbar_init(&cready[i], 128);
      mbar_init(&cfree[i], 128);
    }
    for (int i = 0; i < kCMax; ++i) mbar_init(&cbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // the job table and the operators are constant during the graph: load them
  // before waiting for the predecessor kernel
  if (tid < kCs) {
    const int c = set * kCs + tid;
    FastStep z{nullptr, nullptr, nullptr, nullptr, 1.0, 0, 0};
    sj[tid] = (chain && c < P.nchains) ? P.jobs[int64_t(c) * P.nsteps + t] : z;
    sinp[tid] = (!kU && c < P.nchains) ? P.insrc[int64_t(c) * P.nsteps + t] : -1;
  }
  if (P.empty == 1) {  // debug: launch-overhead floor
    pdl_wait();
    pdl_launch();
    cluster_sync_all();
    return;
  }
  if (tid == 0 && chain) {
    issue_on(0);
    issue_on(1);
    issue_on(2);
    issue_off(0);
    issue_off(1);
  }
  __syncthreads();

  // L: f(t') of the steps whose output is this step's `in` (t' < t-1) was
  // recorded by kernels that completed before the predecessor started, so it
  // can be fetched before griddepcontrol.wait
  // this CTA sums rows 16r..16r+15 of the inflow vector (its contiguous 256
  // elements of the block-vector layout, one per thread) and broadcasts them
  const int ev_e = kRows * kCs * r + tid;
  double fpre = 0.0;
  if (!kU && inflow && t > 0) {
    const int n = 8 * ((ev_e >> 5) & 1) + (ev_e & 7);
    const int ts = sinp[n];
    if (sj[n].in && ts >= 0 && ts != t - 1)
      fpre = P.Fh[((size_t(ts) * P.nsets + set) * NG + G + 1) * kVec + ev_e];
  }
  long long* tim = (P.tim && tid == 0) ? P.tim + (size_t(kU) * gridDim.x + blockIdx.x) * 32 : nullptr;
  unsigned long long* tlm = (P.tl && tid == 0) ? P.tl + ((size_t(2 * t + kU)) * gridDim.x + blockIdx.x) * 4 : nullptr;
  auto gtime = []() {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    return g;
  };
  if (tlm) tlm[0] = gtime();
  if (tim) tim[0] = clock64();
  pdl_wait();  // everything below reads the predecessors' outputs
  // (dependents launch only after every CTA of this grid has started and
  // triggered, so the cross-cluster waits below cannot be starved by them)
  pdl_launch();
  if (tid == 0 && chain) {
    issue_off_v(0);
    issue_off_v(1);
  }
  if (tim) tim[1] = clock64();
  if (tlm) tlm[1] = gtime();

  const int t4 = warp & 3, rt = t4 >> 1, ct = t4 & 1;
  const int krow = r * kRows + rt * 8 + (lane >> 2);  // this lane's block row
  const int nch = ct * 8 + 2 * (lane & 3);            // this lane's chain pair
  const int cpair = set * kCs + nch;                  // global chain of the pair's first

  // inflow vector e_{G-1} (U) / f_{G+1} (L): the group-end value plus the
  // products T y~_end(src) written by the previous kernel of the other
  // direction, one partial per source group, summed in a fixed order
  if (inflow && (kU || t > 0)) {
    const int Gs = kU ? G - 1 : G + 1;
    const double* endv = (kU ? P.Yend : P.Xend) + (size_t(set) * NG + Gs) * kVec;
    const double* pp = (kU ? P.EP : P.FP) + (size_t(set) * NG + Gs) * NG * kVec;
    // sources: L (e_Gs): 0 .. Gs-1; U (f_Gs): Gs+1 .. NG-1
    const int s0 = kU ? 0 : Gs + 1, s1 = kU ? Gs : NG;
    // every partial's load in flight at once, then summed in source order
    double w[kMaxSrc];
#pragma unroll
    for (int p = 0; p < kMaxSrc; ++p) w[p] = s0 + p < s1 ? pp[size_t(s0 + p) * kVec + ev_e] : 0.0;
    double v = endv[ev_e];
#pragma unroll
    for (int p = 0; p < kMaxSrc; ++p)
      if (s0 + p < s1) v += w[p];
    if (!kU) {
      // f(t-1) of group Gs: record this CTA's slice, then combine per chain
      // column n(e):  f~ = [add] f(t-1) + [in = out(t')] scale * f(t')
      P.Fh[((size_t(t - 1) * P.nsets + set) * NG + Gs) * kVec + ev_e] = v;
      const int n = 8 * ((ev_e >> 5) & 1) + (ev_e & 7);
      const FastStep& st = sj[n];
      double f = st.in && st.add ? v : 0.0;
      const int ts = sinp[n];
      if (st.in && ts >= 0) f = fma(st.scale, ts == t - 1 ? v : fpre, f);
      v = f;
    }
    EV[ev_e] = v;
    const uint32_t loc = smem_u32(EV + ev_e);
#pragma unroll 1
    for (int pr = 1; pr < kCl; ++pr)
      asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(mapa_u32(loc, uint32_t((r + pr) % kCl))), "d"(v)
                   : "memory");
  }
  // the other direction's publish flags were last used by the previous
  // kernel (complete): reset them for its next launch
  if (tid < NG && r == 0 && G == 0) (kU ? P.flagL : P.flagU)[set * NG + tid] = 0u;
  if (tid == 0 && chain) {  // peer exchange buffers armed before anyone can send
    mbar_expect_tx(&xbar[0], kCl * kRows * kCs * 8);
    mbar_expect_tx(&xbar[1], kCl * kRows * kCs * 8);
  }
  cluster_sync_all();  // also: EV complete, every CTA's barriers armed
  if (tim) tim[2] = clock64();
  if (tlm) tlm[2] = gtime();

  // ---------------- the zero-inflow chain (warp-specialised) -----------------
  const uint32_t xb_base = smem_u32(&xbar[0]);  // xbar[1] at +8
  double* ybase = kU ? P.Xh + size_t(t) * hstep : P.Yt;
  if (warp < 4) {
    for (int q = 0; q < len; ++q) {
      const int J = rowQ(q);
      long long m0 = tim ? clock64() : 0, m1 = m0, m2 = m0;
      double y0 = 0.0, y1 = 0.0;
      if (q > 0) {
        const int u = q - 1;
        // refill: the slot of stage u-1 (row q-1, consumed last step) gets stage u+2
        if (tid == 0 && u >= 1) {
          mbar_wait(&sfreeC[(u - 1) % 3], uint32_t((u - 1) / 3) & 1u);
          issue_on(u + 2);
        }
        __syncwarp();  // warp 0 converged again before mma.sync
        mbar_wait(&tbarC[u % 3], uint32_t(u / 3) & 1u);
        if (tim) m1 = clock64();
        const int xb = (q - 1) & 1;
        mbar_wait_cluster(&xbar[xb], uint32_t((q - 1) >> 1) & 1u);
        if (tim) m2 = clock64();
        // re-arm for the next use (peers refill it only after receiving this
        // CTA's next slices, sent below after every chain warp read it)
        if (tid == 0) mbar_expect_tx(&xbar[xb], kCl * kRows * kCs * 8);
        warp_mma(ringC + (u % 3) * kSlice, X + xb * kVec, 0, 32, rt, ct, y0, y1);
        mbar_arrive(&sfreeC[u % 3]);
      }
      long long m3 = tim ? clock64() : 0;
      mbar_wait(&cready[q & 1], uint32_t(q >> 1) & 1u);
      long long m4 = tim ? clock64() : 0;
      y0 += Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2];
      y1 += Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2 + 1];
      mbar_arrive(&cfree[q & 1]);
      const int xi = vidx(krow, nch);
      {  // the last row too: every CTA gets the whole group-end vector (B below).
        // This CTA's own tiles go through st.async as well, so the exchange
        // barrier also orders the sibling warps' tiles before the next row reads them.
        const uint32_t loc = smem_u32(X + (q & 1) * kVec + xi);
#pragma unroll
        for (int pr = 0; pr < kCl; ++pr) {
          const uint32_t peer = (uint32_t(r) + pr) % kCl;
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                  mapa_u32(loc, peer)),
              "d"(y0), "d"(y1), "r"(mapa_u32(xb_base + 8u * uint32_t(q & 1), peer))
              : "memory");
        }
      }
      if (q + 1 == len) {
        // group-end value for the B phase: L -> last row J1, U -> first row J0
        double* ev = (kU ? P.Xend : P.Yend) + (size_t(set) * NG + G) * kVec + xi;
        *reinterpret_cast<double2*>(ev) = make_double2(y0, y1);
      }
      // the chain state in fragment layout (inactive chains and padded rows are 0)
      *reinterpret_cast<double2*>(frow(ybase, J) + xi) = make_double2(y0, y1);
      if (tim) {
        const long long m5 = clock64();
        tim[20] += m1 - m0;  // TMA ring wait
        tim[21] += m2 - m1;  // exchange wait
        tim[22] += m3 - m2;  // on-chain product
        tim[23] += m4 - m3;  // off-chain tile wait
        tim[24] += m5 - m4;  // stores + sends
        if (q < 12) tim[4 + q] = m5;
      }
    }
  } else {
    const int ot = tid - 128;  // 0..127
    // operand loads in fragment order: thread ot owns V[ot + 128u], u < 16,
    // i.e. chain vn and rows vk0 + 8u (conflict-free shared stores; a warp's
    // loads cover 8 chains x 4 consecutive rows, whole 32-byte sectors)
    const int vn = 8 * ((warp - 4) & 1) + (lane & 7), vk0 = 4 * ((warp - 4) >> 1) + ((lane >> 3) & 3);
    const FastStep vst = sj[vn];
    const bool vact = vst.in != nullptr;
    // L: b~ = in*scale + x~_{t-1} with in = x~_{t'} when it is an earlier
    // output (the rest of those outputs, Psi f, is in the combined f~ of EV)
    // or the gathered external plane; all in fragment order (contiguous).
    // U takes y~_J by TMA instead.
    const bool vadd = !kU && vact && vst.add != nullptr;
    const int vts = kU ? -1 : sinp[vn];
    const double* srcin = vts >= 0 ? P.Xh + size_t(vts) * hstep : P.Rin + size_t(t) * hstep;
    const double* srcad = vadd ? P.Xh + size_t(t - 1) * hstep : P.zeros;
    double xin[16], xad[16];
    auto load_v = [&](int J) {
      if (kU) return;
      const double* fi = srcin + (size_t(set) * P.ny + J) * kVec;
      const double* fa = vadd ? srcad + (size_t(set) * P.ny + J) * kVec : P.zeros;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = ot + 128 * u;  // == vidx(vk0 + 8u, vn)
        xin[u] = fi[e];
        xad[u] = fa[vadd ? e : 0];
      }
    };
    auto store_v = [&]() {
      if (kU) return;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = vk0 + 8 * u;
        const double v = fma(xin[u], vst.scale, xad[u]);
        V[ot + 128 * u] = (vact && k < P.nx) ? v : 0.0;  // == V[vidx(k, vn)]
      }
    };
    // per-chain scalars of this lane's chain pair
    double al[2] = {0.0, 0.0}, be[2] = {0.0, 0.0}, ga[2] = {0.0, 0.0};
    double addm[2] = {0.0, 0.0};
    const bool lacoef = !kU && P.coarse;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const FastStep& sw = sj[nch + w];
      // coefficient of the inflow term: (Ut Phi) e for every active chain (U);
      // L: the per-chain f~ is already combined in EV
      addm[w] = sw.in ? 1.0 : 0.0;
      // the two-level residual term, b -= (Shat y_c)_node / ms, after the
      // product: Li_J (Shat y_c) = al*Li a2 - be*Li a1 + ga*Li 1
      if (lacoef && sw.in && sw.node > 0) {
        const double gn = P.gam[sw.node], gp = P.gam[sw.node + 1];
        const bool d = sw.node != 1;
        const double gm = d ? P.gam[sw.node - 1] : 0.0;
        al[w] = gn * P.inv_ms;
        be[w] = (gp + gm) * P.inv_ms;
        ga[w] = d ? gn * P.inv_ms : 0.0;
      }
    }
    double la2 = 0.0, la1 = 0.0, la0 = 0.0;
    auto load_row = [&](int J) {  // per-lane row data: the LA terms
      const int kr = krow < P.nx ? krow : 0;
      if (lacoef) {
        const double* la = P.LA + size_t(J) * 3 * kN + kr;  // Li a2, Li a1, Li 1
        la2 = la[0];
        la1 = la[kN];
        la0 = la[2 * kN];
      }
    };
    load_v(rowQ(0));
    load_row(rowQ(0));
    store_v();
    if (len > 1) load_v(rowQ(1));
    named_bar_sync(1, 128);
    long long* otim = (P.tim && ot == 0) ? P.tim + (size_t(kU) * gridDim.x + blockIdx.x) * 32 : nullptr;
    for (int q = 0; q < len; ++q) {
      const int J = rowQ(q);
      const double cl2 = la2, cl1 = la1, cl0 = la0;
      if (q + 1 < len) load_row(rowQ(q + 1));
      long long n0 = otim ? clock64() : 0;
      mbar_wait(&tbarO[q & 1], uint32_t(q >> 1) & 1u);
      long long n1 = otim ? clock64() : 0;
      const double* so = ringO + (q & 1) * 3 * kSlice;
      double c0 = 0.0, c1 = 0.0;
      warp_mma(so, kU ? so + 2 * kSlice : V, okb, oke, rt, ct, c0, c1);  // Li_J b / Ut_J y~
      if (use_m1) {
        double m0v = 0.0, m1v = 0.0;
        warp_mma(so + kSlice, EV, 0, 32, rt, ct, m0v, m1v);  // (Li Psi)_J f / (Ut Phi)_J e
        c0 += addm[0] * m0v;
        c1 += addm[1] * m1v;
      }
      if (lacoef && krow < P.nx) {
        c0 -= al[0] * cl2 - be[0] * cl1 + ga[0] * cl0;
        c1 -= al[1] * cl2 - be[1] * cl1 + ga[1] * cl0;
      }
      long long n2 = otim ? clock64() : 0;
      if (q >= 2) mbar_wait(&cfree[q & 1], uint32_t((q >> 1) - 1) & 1u);
      long long n3 = otim ? clock64() : 0;
      Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2] = c0;
      Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2 + 1] = c1;
      mbar_arrive(&cready[q & 1]);
      named_bar_sync(1, 128);  // every off warp is done with V and off stage q
      if (ot == 0) {
        issue_off(q + 2);
        issue_off_v(q + 2);
      }
      long long n4 = otim ? clock64() : 0;
      if (!kU && q + 1 < len) {
        store_v();
        if (q + 2 < len) load_v(rowQ(q + 2));
        named_bar_sync(1, 128);  // V complete
      }
      if (otim) {
        const long long n5 = clock64();
        otim[25] += n1 - n0;  // off: ring wait
        otim[26] += n2 - n1;  // off: products
        otim[27] += n3 - n2;  // off: cfree wait
        otim[28] += n4 - n3;  // off: handoff + barrier + refill
        otim[29] += n5 - n4;  // off: operand stage
      }
    }
  }
  if (tim) tim[31] = clock64();

  // ---------------- B: products for the boundary values ---------------------
  //   L: e_G = y~_end(G) + sum_{i<G} TL_{G,i} y~_end(i)
  //   U: f_G = x~_first(G) + sum_{i>G} TU_{m(G),m(i)} x~_first(i),  m(x) = NG-1-x
  // The cluster of source group i computes the products with its own
  // group-end vector (in X after the last exchange) for its targets; pairs
  // i <-> NG-1-i share the work so no cluster computes more than
  // ceil((NG-1)/2) products (the borrowed ones wait for the partner's
  // published vector).  Results: one partial per (target, source).
  unsigned* flags = (kU ? P.flagU : P.flagL) + set * NG;
  const double* endv = (kU ? P.Xend : P.Yend) + size_t(set) * NG * kVec;
  if (tid == 0) __threadfence();  // this CTA's group-end slice before the flag
  __syncthreads();
  cluster_sync_all();
  if (tid == 0 && r == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(flags + G), "r"(1u) : "memory");
  const int half = NG / 2;  // ceil((NG-1)/2)
  const int pg = NG - 1 - G;
  // targets of source x: L -> x+1 .. NG-1, U -> 0 .. x-1 (count NG-1-x / x)
  auto ntarg = [&](int x) { return kU ? x : NG - 1 - x; };
  auto targ = [&](int x, int k) { return kU ? x - 1 - k : x + 1 + k; };
  const int nown = min(ntarg(G), half);
  const int nbor = (pg != G && ntarg(pg) > half) ? ntarg(pg) - half : 0;
  const double* T = kU ? P.TU : P.TL;
  auto tm = [&](int tg, int src) { return kU ? tri_idx(NG - 1 - tg, NG - 1 - src) : tri_idx(tg, src); };
  double* stage = sm;  // the rings are free now (9 slices)
  if (tid == 0) {
    for (int k = 0; k < nown + nbor; ++k) {
      const int src = k < nown ? G : pg;
      const int tg = k < nown ? targ(G, k) : targ(pg, half + (k - nown));
      mbar_expect_tx(&cbar[k], kSlice * 8 + (k == nown ? kVec * 8 : 0));
      bulk_g2s(stage + k * kSlice, T + (size_t(tm(tg, src)) * kCl + r) * kSlice, kSlice * 8, &cbar[k]);
    }
    if (nbor > 0) {  // the partner's vector, once it is published
      unsigned v = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flags + pg) : "memory");
      } while (v == 0u);
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      bulk_g2s(stage + 8 * kSlice, endv + size_t(pg) * kVec, kVec * 8, &cbar[nown]);
    }
  }
  const double* ownv = X + ((len - 1) & 1) * kVec;
  mbar_wait_cluster(&xbar[(len - 1) & 1], uint32_t((len - 1) >> 1) & 1u);  // last exchange complete
  for (int k = 0; k < nown + nbor; ++k) {
    const int src = k < nown ? G : pg;
    const int tg = k < nown ? targ(G, k) : targ(pg, half + (k - nown));
    mbar_wait(&cbar[k], 0u);
    double e0 = 0.0, e1 = 0.0;
    cta_mma(stage + k * kSlice, k < nown ? ownv : stage + 8 * kSlice, 0, 32, part, e0, e1);
    if (warp < 4) {
      double* out = (kU ? P.FP : P.EP) + ((size_t(set) * NG + tg) * NG + src) * kVec + vidx(krow, nch);
      *reinterpret_cast<double2*>(out) = make_double2(e0, e1);
    }
  }
  cluster_sync_all();  // no CTA exits while a peer may still address its shared memory
  if (tlm) tlm[3] = gtime();
}

// ---------------------------------------------------------------------------
// Per application, before the chains: insrc[c][t] = t' when the `in` plane of
// step t is the `out` plane of an earlier step t' of the same chain (the RASQ
// adjoint steps read the forward outputs), else -1; and the external `in`
// planes gathered into the block-vector fragment layout (Rin).
// ---------------------------------------------------------------------------
// live[c][t]: bit 0 out(t), bit 1 out2(t) is the final content of its plane
// (no later step of the chain writes the same plane), so the output pass can
// write every step in parallel.
__global__ void v4_insrc_kernel(const FastStep* __restrict__ jobs, int nchains, int nsteps, int* insrc,
                                int* live) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nchains * nsteps) return;
  const int c = i / nsteps, t = i - c * nsteps;
  const FastStep* J = jobs + int64_t(c) * nsteps;
  int src = -1;
  if (J[t].in)
    for (int tp = 0; tp < t; ++tp)
      if (J[tp].in && J[tp].out == J[t].in) src = tp;
  insrc[i] = src;
  int lv = 0;
  if (J[t].in) {
    bool o1 = J[t].out != nullptr, o2 = J[t].out2 != nullptr;
    if (o2 && J[t].out2 == J[t].out) o1 = false;
    for (int t2 = t + 1; t2 < nsteps; ++t2) {
      if (!J[t2].in) continue;
      if (o1 && (J[t2].out == J[t].out || J[t2].out2 == J[t].out)) o1 = false;
      if (o2 && (J[t2].out == J[t].out2 || J[t2].out2 == J[t].out2)) o2 = false;
    }
    lv = (o1 ? 1 : 0) | (o2 ? 2 : 0);
  }
  live[i] = lv;
}

__global__ void v4_gather_kernel(V4Params P) {
  const int J = blockIdx.x % P.ny;
  const int set = (blockIdx.x / P.ny) % P.nsets;
  const int t = blockIdx.x / (P.ny * P.nsets);
  double* dst = P.Rin + ((size_t(t) * P.nsets + set) * P.ny + J) * kVec;
  for (int e = threadIdx.x; e < kVec; e += blockDim.x) {
    const int k = 4 * (e >> 6) + ((e >> 3) & 3);
    const int n = 8 * ((e >> 5) & 1) + (e & 7);
    const int c = set * kCs + n;
    double v = 0.0;
    if (c < P.nchains && k < P.nx) {
      const FastStep st = P.jobs[int64_t(c) * P.nsteps + t];
      if (st.in && P.insrc[int64_t(c) * P.nsteps + t] < 0) v = st.in[size_t(J) * P.nx + k];
    }
    dst[e] = v;
  }
}

// ---------------------------------------------------------------------------
// After the chains: every step's output x_t = x~_t + Psi_J f_{G+1}(t) (Xh, Fh;
// f of the last step from the last U kernel's partials) to the job's out and
// out2 (+ gamma[node2]) where that write is live (v4_insrc_kernel), so the
// steps run in parallel: CTA (t, set, J, slice r), one tile per warp.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) v4_out_kernel(V4Params P) {
  pdl_wait();
  const int r = blockIdx.x % kCl;
  const int J = (blockIdx.x / kCl) % P.ny;
  const int set = (blockIdx.x / (kCl * P.ny)) % P.nsets;
  const int t = blockIdx.x / (kCl * P.ny * P.nsets);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rt = warp >> 1, ct = warp & 1;
  const int krow = r * kRows + rt * 8 + (lane >> 2);
  const int nch = ct * 8 + 2 * (lane & 3);
  // skip the CTA when no chain of the set has a live output at this step
  __shared__ int any_live;
  if (threadIdx.x == 0) any_live = 0;
  __syncthreads();
  if (threadIdx.x < kCs) {
    const int c = set * kCs + threadIdx.x;
    if (c < P.nchains && P.live[int64_t(c) * P.nsteps + t]) any_live = 1;
  }
  __syncthreads();
  if (!any_live) {
    pdl_launch();
    return;
  }
  const int G = J / P.g, NG = P.NG;
  const bool inflow = G < NG - 1;
  const int Gs = G + 1;
  double d0 = 0.0, d1 = 0.0;
  if (inflow) {
    const double* A = P.Psi + (size_t(J) * kCl + r) * kSlice + rt * 32 + lane;
    const int bo = ct * 32 + (lane & 3) * 8 + (lane >> 2);
    const double* fb = P.Fh + ((size_t(t) * P.nsets + set) * NG + Gs) * kVec + bo;
    const bool last = t + 1 == P.nsteps;  // f(last): group-end value + its sources' partials
    const double* ev = P.Xend + (size_t(set) * NG + Gs) * kVec + bo;
    const double* pp = P.FP + (size_t(set) * NG + Gs) * NG * kVec + bo;
    double e0 = 0.0, e1 = 0.0;
#pragma unroll 4
    for (int ks = 0; ks < 32; ks += 2) {
      double b0, b1;
      if (!last) {
        b0 = fb[ks * 64];
        b1 = fb[(ks + 1) * 64];
      } else {
        b0 = ev[ks * 64];
        b1 = ev[(ks + 1) * 64];
        for (int src = Gs + 1; src < NG; ++src) {
          b0 += pp[size_t(src) * kVec + ks * 64];
          b1 += pp[size_t(src) * kVec + (ks + 1) * 64];
        }
      }
      dmma4(d0, d1, A[ks * 64], b0);
      dmma4(e0, e1, A[(ks + 1) * 64], b1);
    }
    d0 += e0;
    d1 += e1;
  }
  if (krow < P.nx) {
    const size_t hstep = size_t(P.nsets) * P.ny * kVec;
    const double2 xv = *reinterpret_cast<const double2*>(
        P.Xh + size_t(t) * hstep + (size_t(set) * P.ny + J) * kVec + vidx(krow, nch));
    const int p = J * P.nx + krow;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int c = set * kCs + nch + w;
      if (c >= P.nchains) continue;
      const int lv = P.live[int64_t(c) * P.nsteps + t];
      if (!lv) continue;
      const FastStep st = P.jobs[int64_t(c) * P.nsteps + t];
      const double x = (w ? xv.y : xv.x) + (w ? d1 : d0);
      if (lv & 1) st.out[p] = x;
      if (lv & 2) st.out2[p] = x + ((st.node2 > 0 && P.gam) ? P.gam[st.node2] : 0.0);
    }
  }
  pdl_launch();
}

// ---------------------------------------------------------------------------
// setup: repack dense operators into fragment-ordered slices
//   mode 0: M'[a][b] = src[a*ld + b]                (a, b < n)
//   mode 1: M'[a][b] = src[b*ld + a] * dinv[b]      (Ut = Li^T D^{-1})
// ---------------------------------------------------------------------------
__global__ void frag_pack_kernel(const double* __restrict__ src, int64_t sstride, int ld, int n, int mode,
                                 const double* __restrict__ dinv, int dstride, double* __restrict__ dst) {
  const int m = blockIdx.y;
  const double* S = src + m * sstride;
  double* D = dst + int64_t(m) * kMat;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kMat; e += gridDim.x * blockDim.x) {
    const int r = e / kSlice, w = e % kSlice;
    const int ks = w / 64, rt = (w / 32) & 1, l = w & 31;
    const int a = r * kRows + rt * 8 + l / 4, b = ks * 4 + (l & 3);
    double v = 0.0;
    if (a < n && b < n) v = mode == 0 ? S[int64_t(a) * ld + b] : S[int64_t(b) * ld + a] * dinv[m * dstride + b];
    D[e] = v;
  }
}

// LA[J][j][a] = sum_b Li_J[a][b] v_j[J*nx + b], v = (a2, a1, 1), from the
// fragment-ordered Li (OffL)
__global__ void la_kernel(const double* __restrict__ OffL, const double* __restrict__ a1,
                          const double* __restrict__ a2, int nx, double* __restrict__ LA) {
  const int J = blockIdx.x, a = threadIdx.x;  // blockDim = kN
  const double* M = OffL + size_t(J) * kMat;
  double s2 = 0.0, s1 = 0.0, s0 = 0.0;
  if (a < nx) {
    const int r = a / kRows, rt = (a % kRows) / 8, li = (a % 8) * 4;
    for (int b = 0; b <= a; ++b) {
      const double m = M[r * kSlice + ((b / 4) * 2 + rt) * 32 + li + (b & 3)];
      s2 = fma(m, a2[J * nx + b], s2);
      s1 = fma(m, a1[J * nx + b], s1);
      s0 += m;
    }
  }
  LA[(size_t(J) * 3 + 0) * kN + a] = s2;
  LA[(size_t(J) * 3 + 1) * kN + a] = s1;
  LA[(size_t(J) * 3 + 2) * kN + a] = s0;
}

// C_J = A_J B_J (kN x kN, zero padded), A_J = Li_J (mode 0) or Li_J^T D_J^{-1}
// (mode 1) from the square inverse blocks (nx x nx), B_J dense kN x kN (setup)
__global__ void lmul_kernel(const double* __restrict__ Li, const double* __restrict__ dinv, int nx, int mode,
                            const double* __restrict__ B, double* __restrict__ C) {
  const int J = blockIdx.x;
  const double* L = Li + size_t(J) * nx * nx;
  const double* Bj = B + size_t(J) * kMat;
  for (int e = threadIdx.x; e < kMat; e += blockDim.x) {
    const int a = e / kN, b = e % kN;
    double acc = 0.0;
    if (a < nx) {
      if (mode == 0) {
        for (int k = 0; k <= a; ++k) acc = fma(L[a * nx + k], Bj[k * kN + b], acc);
      } else {
        for (int k = a; k < nx; ++k) acc = fma(L[k * nx + a] * dinv[J * nx + k], Bj[k * kN + b], acc);
      }
    }
    C[size_t(J) * kMat + e] = acc;
  }
}

void launch_ex(Ctx* c, const void* fn, int grid, size_t smem, bool cluster, void** args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThr4);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  // the A kernels wait across clusters (B tail): a cooperative launch makes
  // the driver guarantee that every CTA of the grid is co-resident when other
  // v4 contexts share the device (v4_register)
  if (c->v4_coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (cluster) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = kCl;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  KKT_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  c->launches++;
}

void launch_ex_threads(Ctx* c, const void* fn, int grid, int threads, void** args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KKT_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  c->launches++;
}

size_t smemA() { return sizeof(double) * (9 * size_t(kSlice) + 4 * size_t(kVec) + 3 * 4 * 32 * 2); }

}  // namespace

bool v4_supported(const Ctx* c) { return c->nx <= kN && c->ny >= 2 && !getenv("KKT_SWEEP_V3"); }

// Live v4 contexts per device (this process).  The A kernels wait across
// clusters, so a grid must not be starved of SMs by another such grid.  One
// non-cooperative grid alone is safe (cooperative grids are guaranteed their
// own residency and finish); every context after the first on a device
// launches cooperatively.  KKT_V4_COOP=0/1 forces the choice.
static std::atomic<int> g_live_v4[64];
void v4_register(Ctx* c) {
  const int d = c->device & 63;
  const int before = g_live_v4[d].fetch_add(1);
  c->v4_registered = true;
  c->v4_coop = before > 0;
  if (const char* e = getenv("KKT_V4_COOP")) c->v4_coop = atoi(e) != 0;
}
void v4_unregister(Ctx* c) {
  if (c->v4_registered) g_live_v4[c->device & 63].fetch_sub(1);
  c->v4_registered = false;
}

void set_v4_attributes() {
  static bool done = false;
  if (done) return;
  KKT_CUDA(cudaFuncSetAttribute(v4A_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemA())));
  KKT_CUDA(cudaFuncSetAttribute(v4A_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemA())));
  done = true;
}

// Group size for v4: every cluster of one chain set co-resident (one wave).
// An 8-CTA cluster must fit in one GPC, so fewer than 148/8 clusters fit at
// once (15 on B200 at one CTA per SM): ask the occupancy calculator.
int v4_group_size(const Ctx* c) {
  if (const char* e = getenv("KKT_V4_G")) return std::max(1, atoi(e));
  set_v4_attributes();
  const int nsets = std::max(1, (c->ndl + kCs - 1) / kCs);
  int max_clusters = kSmCount / kCl;
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kSmCount / kCl * kCl);
    cfg.blockDim = dim3(kThr4);
    cfg.dynamicSmemBytes = smemA();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(&v4A_kernel<false>), &cfg) ==
            cudaSuccess &&
        n > 0)
      max_clusters = n;
    cudaGetLastError();
  }
  const int max_groups = std::max(1, max_clusters / nsets);
  const int g = (c->ny + max_groups - 1) / max_groups;
  return std::max(g, 2);
}

// Repack G, H, Li, Ut, Phi, Psi, Tl, Tu (dense kMaxNx^2, built by
// build_group_operators with c->grp_g) into fragment-ordered operator slices.
void build_v4(Ctx* c, const double* G, const double* H, const double* Li, const double* dinv) {
  const int nx = c->nx, ny = c->ny, NG = c->grp_n;
  const int ntri = std::max(1, NG * (NG - 1) / 2);
  const size_t per = size_t(ny) * kMat;
  c->v4_ops.alloc(7 * per + 2 * size_t(ntri) * kMat);
  double* base = c->v4_ops.p;
  auto pack = [&](const double* src, int64_t sstride, int ld, int n, int mode, int count, double* dst) {
    const dim3 grid(16, count);
    KKT_LAUNCH(c, frag_pack_kernel, grid, 256, 0, src, sstride, ld, n, mode, dinv, nx, dst);
  };
  pack(G, kMat, kN, nx, 0, ny, base + 0 * per);                    // OnL  = G_J
  pack(Li, int64_t(nx) * nx, nx, nx, 0, ny, base + 1 * per);       // OffL = Li_J
  pack(H, kMat, kN, nx, 0, ny, base + 2 * per);                    // OnU  = H_J
  pack(Li, int64_t(nx) * nx, nx, nx, 1, ny, base + 3 * per);       // OffU = Li_J^T D_J^{-1}
  {
    // the inflow propagators as the other sweep sees them: Ut_J Phi_J, Li_J Psi_J
    DBuf<double> tmp(per);
    KKT_LAUNCH(c, lmul_kernel, ny, 256, 0, Li, dinv, nx, 1, c->Phi.p, tmp.p);
    pack(tmp.p, kMat, kN, nx, 0, ny, base + 4 * per);              // UPhi
    KKT_LAUNCH(c, lmul_kernel, ny, 256, 0, Li, dinv, nx, 0, c->Psi.p, tmp.p);
    pack(tmp.p, kMat, kN, nx, 0, ny, base + 6 * per);              // LPsi
    KKT_CUDA(cudaStreamSynchronize(c->stream));
  }
  pack(c->Psi.p, kMat, kN, nx, 0, ny, base + 5 * per);             // Psi
  if (NG > 1) {
    pack(c->grp_tl.p, kMat, kN, nx, 0, NG * (NG - 1) / 2, base + 7 * per);
    pack(c->grp_tu.p, kMat, kN, nx, 0, NG * (NG - 1) / 2, base + 7 * per + size_t(ntri) * kMat);
  }
  static_assert(kCMax <= 9, "the C slab aliases the 9 ring slices");
  c->v4_zero.alloc(kN);
  KKT_CUDA(cudaMemsetAsync(c->v4_zero.p, 0, sizeof(double) * kN, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  set_v4_attributes();
  v4_register(c);
}

// Run `nsteps` lock-step spatial solves of `nchains` chains (chain-major job
// table on the device): per step A_L, B_L, A_U, B_U, then the final C-part.
void v4_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms) {
  const int NG = c->grp_n;
  const int nsets = (nchains + kCs - 1) / kCs;
  if (nsets > c->v4_nsets) {
    // state for nsets chain sets: y~, x~ planes, group-end vectors, B partials.
    // Graphs captured against the old state are dropped.
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& e : c->graphs)
      if (e.exec) cudaGraphExecDestroy(e.exec);
    c->graphs.clear();
    const size_t nvec = size_t(nsets) * NG * kVec;
    c->v4_state.alloc(size_t(2 * nsets) * c->ny * kVec + 2 * nvec + 2 * nvec * NG);
    KKT_CUDA(cudaMemsetAsync(c->v4_state.p, 0, sizeof(double) * c->v4_state.n, c->stream));
    c->v4_flags.alloc(size_t(2) * nsets * NG);
    KKT_CUDA(cudaMemsetAsync(c->v4_flags.p, 0, sizeof(unsigned) * c->v4_flags.n, c->stream));
    c->v4_nsets = nsets;
  }
  const int nsets_alloc = c->v4_nsets;
  const size_t nveca = size_t(nsets_alloc) * NG * kVec;
  V4Params P;
  const size_t per = size_t(c->ny) * kMat;
  const int ntri = std::max(1, NG * (NG - 1) / 2);
  double* ops = c->v4_ops.p;
  P.OnL = ops;
  P.OffL = ops + per;
  P.OnU = ops + 2 * per;
  P.OffU = ops + 3 * per;
  P.UPhi = ops + 4 * per;
  P.Psi = ops + 5 * per;
  P.LPsi = ops + 6 * per;
  P.TL = ops + 7 * per;
  P.TU = ops + 7 * per + size_t(ntri) * kMat;
  double* st = c->v4_state.p;
  P.Yt = st;
  double* vb = st + size_t(2 * nsets_alloc) * c->ny * kVec;
  // per-step history (x~, gathered inputs, f) and the input-source table
  {
    const size_t hs = size_t(nsteps) * nsets * c->ny * kVec;
    const size_t fs = size_t(nsteps) * nsets * NG * kVec;
    const size_t need = 2 * hs + fs + size_t(nsets) * kCs * nsteps + 1;
    if (c->v4_hist.n < need) {
      KKT_CUDA(cudaStreamSynchronize(c->stream));
      for (auto& e : c->graphs)
        if (e.exec) cudaGraphExecDestroy(e.exec);
      c->graphs.clear();
      c->v4_hist.alloc(need);
      KKT_CUDA(cudaMemsetAsync(c->v4_hist.p, 0, sizeof(double) * need, c->stream));
    }
    P.Xh = c->v4_hist.p;
    P.Rin = c->v4_hist.p + hs;
    P.Fh = c->v4_hist.p + 2 * hs;
    P.insrc = reinterpret_cast<int*>(c->v4_hist.p + 2 * hs + fs);
    P.live = P.insrc + size_t(nsets) * kCs * nsteps;
  }
  P.Yend = vb;
  P.Xend = vb + nveca;
  P.EP = vb + 2 * nveca;
  P.FP = vb + 2 * nveca + nveca * NG;
  P.flagL = c->v4_flags.p;
  P.flagU = c->v4_flags.p + size_t(nsets_alloc) * NG;
  P.a1 = c->a1.p;
  P.a2 = c->a2.p;
  P.gam = c->gam.p;
  P.inv_ms = 1.0 / c->ms;
  P.nx = c->nx;
  P.ny = c->ny;
  P.nsp = c->nsp;
  P.g = c->grp_g;
  P.NG = NG;
  if (NG - 1 > kMaxSrc) throw Error(KKT_EINVAL, "sweep v4: too many groups for the inflow sum");
  P.nchains = nchains;
  P.nsets = nsets;
  P.jobs = jobs_dev;
  P.nsteps = nsteps;
  P.coarse = coarse_terms ? 1 : 0;
  P.zeros = c->v4_zero.p;
  if (coarse_terms && !c->v4_la.p) {
    c->v4_la.alloc(size_t(c->ny) * 3 * kN);
    KKT_LAUNCH(c, la_kernel, c->ny, kN, 0, P.OffL, c->a1.p, c->a2.p, c->nx, c->v4_la.p);
  }
  P.LA = c->v4_la.p;
  P.empty = getenv("KKT_V4_EMPTY") ? atoi(getenv("KKT_V4_EMPTY")) : 0;
  static const bool tim_on = getenv("KKT_V4_TIM") != nullptr;
  P.tim = nullptr;
  DBuf<long long> timbuf;
  if (tim_on) {
    timbuf.alloc(size_t(2) * nsets * NG * kCl * 32);
    KKT_CUDA(cudaMemsetAsync(timbuf.p, 0, sizeof(long long) * timbuf.n, c->stream));
    P.tim = timbuf.p;
  }
  const int gridA = nsets * NG * kCl;
  const size_t sA = smemA();
  static const bool tl_on = getenv("KKT_V4_TL") != nullptr;
  P.tl = nullptr;
  if (tl_on) {
    const size_t need = size_t(2) * nsteps * gridA * 4;
    if (c->v4_tl.n < need) c->v4_tl.alloc(need);
    P.tl = c->v4_tl.p;
  }
  auto sequence = [&]() {
    const int npairs = nchains * nsteps;
    KKT_LAUNCH(c, v4_insrc_kernel, (npairs + 127) / 128, 128, 0, jobs_dev, nchains, nsteps,
               const_cast<int*>(P.insrc), const_cast<int*>(P.live));
    KKT_LAUNCH(c, v4_gather_kernel, nsteps * nsets * c->ny, 256, 0, P);
    for (int t = 0; t < nsteps; ++t) {
      int zero = 0;
      {
        void* args[] = {&P, &t, &zero};
        launch_ex(c, reinterpret_cast<const void*>(&v4A_kernel<false>), gridA, sA, true, args);
      }
      {
        void* args[] = {&P, &t, &zero};
        launch_ex(c, reinterpret_cast<const void*>(&v4A_kernel<true>), gridA, sA, true, args);
      }
    }
    {
      void* args[] = {&P};
      launch_ex_threads(c, reinterpret_cast<const void*>(&v4_out_kernel), nsteps * nsets * c->ny * kCl, 128, args);
    }
  };
  static const bool no_graph = getenv("KKT_NO_GRAPH") != nullptr;
  if (no_graph || tim_on) {
    c->tbegin(3);
    sequence();
    c->tend(3);
    if (tim_on) {  // marks of the LAST launch of each A kernel (debug)
      std::vector<long long> h(timbuf.n);
      KKT_CUDA(cudaMemcpyAsync(h.data(), timbuf.p, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, c->stream));
      KKT_CUDA(cudaStreamSynchronize(c->stream));
      const int nb = nsets * NG * kCl;
      for (int u = 0; u < 2; ++u) {
        double acc[32] = {0};
        int cnt = 0;
        for (int b = 0; b < nb; ++b) {
          const long long* m = h.data() + (size_t(u) * nb + b) * 32;
          if (!m[0] || !m[31]) continue;
          ++cnt;
          long long prev = m[0];
          for (int i = 1; i < 32; ++i) {
            if (i >= 20 && i <= 29) {
              acc[i] += double(m[i]);
              continue;
            }
            if (m[i]) { acc[i] += double(m[i] - prev); prev = m[i]; }
          }
        }
        fprintf(stderr, "v4A<%d> cycles (avg over %d CTAs): pdl_wait %.0f | setup %.0f | Cpart %.0f | steps", u, cnt,
                acc[1] / cnt, acc[2] / cnt, acc[3] / cnt);
        for (int i = 4; i < 16; ++i)
          if (acc[i] > 0) fprintf(stderr, " %.0f", acc[i] / cnt);
        const double ns = 65.0 * 9.0 * cnt;  // per step (config-1 shape)
        fprintf(stderr, " | tail %.0f | per step: chain tma %.0f xwait %.0f on %.0f cwait %.0f send %.0f | off ring %.0f mma %.0f cfree %.0f hand %.0f stage %.0f\n",
                acc[31] / cnt, acc[20] / ns, acc[21] / ns, acc[22] / ns, acc[23] / ns, acc[24] / ns, acc[25] / ns,
                acc[26] / ns, acc[27] / ns, acc[28] / ns, acc[29] / ns);
      }
    }
    return;
  }
  Ctx::Graph* gr = nullptr;
  for (auto& e : c->graphs)
    if (e.jobs == jobs_dev && e.nchains == nchains && e.nsteps == nsteps && e.coarse == coarse_terms &&
        e.y == c->v4_state.p)
      gr = &e;
  if (!gr) {
    Ctx::Graph e;
    e.jobs = jobs_dev;
    e.nchains = nchains;
    e.nsteps = nsteps;
    e.coarse = coarse_terms;
    e.y = c->v4_state.p;
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
  if (tl_on) {  // kernel-boundary timeline of this application (debug)
    std::vector<unsigned long long> h(size_t(2) * nsteps * gridA * 4);
    KKT_CUDA(cudaMemcpyAsync(h.data(), P.tl, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                             c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    double gap[2] = {0, 0}, wspread[2] = {0, 0}, setup[2] = {0, 0}, body[2] = {0, 0}, prolog[2] = {0, 0};
    int cnt[2] = {0, 0};
    auto at = [&](int k, int b, int i) { return h[(size_t(k) * gridA + b) * 4 + i]; };
    for (int k = 1; k < 2 * nsteps; ++k) {
      unsigned long long end_prev = 0, wmin = ~0ull, wmax = 0, smax = 0, emax = 0, st_min = ~0ull;
      for (int b = 0; b < gridA; ++b) {
        end_prev = std::max(end_prev, at(k - 1, b, 3));
        wmin = std::min(wmin, at(k, b, 1));
        wmax = std::max(wmax, at(k, b, 1));
        smax = std::max(smax, at(k, b, 2));
        emax = std::max(emax, at(k, b, 3));
        st_min = std::min(st_min, at(k, b, 0));
      }
      const int u = k & 1;
      gap[u] += double(wmin) - double(end_prev);
      wspread[u] += double(wmax - wmin);
      setup[u] += double(smax) - double(wmax);
      body[u] += double(emax) - double(smax);
      prolog[u] += double(end_prev) - double(st_min);
      ++cnt[u];
    }
    for (int k = 2 * (nsteps / 2); k < 2 * (nsteps / 2) + 2; ++k) {  // one mid step, per cluster
      unsigned long long w0 = ~0ull;
      for (int b = 0; b < gridA; ++b) w0 = std::min(w0, at(k, b, 1));
      fprintf(stderr, "v4A<%d> step %d per cluster (ns from first wait return): wait / setup end / exit:", k & 1, k / 2);
      for (int cl = 0; cl < gridA / kCl; ++cl) {
        unsigned long long w = 0, se = 0, ex = 0;
        for (int b = cl * kCl; b < (cl + 1) * kCl; ++b) {
          w = std::max(w, at(k, b, 1));
          se = std::max(se, at(k, b, 2));
          ex = std::max(ex, at(k, b, 3));
        }
        fprintf(stderr, " [%d: %llu %llu %llu]", cl, w - w0, se - w0, ex - w0);
      }
      fprintf(stderr, "\n");
    }
    for (int u = 0; u < 2; ++u)
      fprintf(stderr,
              "v4A<%d> timeline (ns, avg over %d kernels): start-before-pred-end %.0f | pred end -> first wait return %.0f"
              " | wait-return spread %.0f | setup %.0f | rows+tail %.0f\n",
              u, cnt[u], prolog[u] / cnt[u], gap[u] / cnt[u], wspread[u] / cnt[u], setup[u] / cnt[u], body[u] / cnt[u]);
  }
}

}  // namespace kkt
