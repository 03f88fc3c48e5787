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
//  * A (the chain of g block steps of one group) runs on a cluster of 8 CTAs.
//    CTA r owns block rows 16r..16r+15 of every step and computes them for
//    ALL 16 chains of a chain set at once as 2x2 m8n8k4 fp64 DMMA tiles, so
//    each factor element read from shared memory serves 16 right-hand sides.
//    Matrix row slices arrive by TMA bulk copies (a 3-stage ring, fetched
//    steps ahead); the 16-row result slice of step q goes to the 7 peer CTAs
//    with st.async (DSMEM, mbarrier transaction counts), double-buffered.
//    The off-chain term (c_J or d_J) is computed before waiting for the
//    peers' slices, so it overlaps the exchange.
//  * The inflow correction of the previous sweep direction is folded into the
//    start of the next A kernel (C-part), so a time step is 4 kernels:
//    A_L(+C_U of the previous step) -> B_L -> A_U(+C_L) -> B_U.
//  * B (group-boundary values) is split into chunks of kBT propagator
//    products per CTA; the chunk partials are summed in a fixed order by the
//    consumer, so every result is deterministic.
//  * Kernels are chained with programmatic dependent launch and the whole
//    RASQ application (4*(2m+1)+1 launches) is replayed from a CUDA graph.
//
// Layouts.  Matrices (128x128, zero padded) are stored "fragment ordered":
// slice r (rows 16r..16r+15) = [ks 32][rt 2][lane 32] with element
// M[16r+8rt+lane/4][4ks+lane%4], the A operand of m8n8k4 read as 32
// consecutive doubles per warp.  A block vector of 128 rows x 16 chains is
// [ks 32][ct 2][kl 4][nl 8] (row 4ks+kl, chain 8ct+nl): the B operand reads
// 32 consecutive doubles, the D fragment writes chain pairs as double2, and
// the rows of CTA r are the contiguous doubles [256r, 256r+256).
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
constexpr int kRing = 3;
constexpr int kBT = 2;               // propagator products per B-phase CTA
constexpr int kCMax = 9;             // C-part operator slices in flight (the slab aliases ring + X + V)

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
__device__ __forceinline__ void l2_prefetch(const double* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
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
// k-steps [kb, ke), 4 independent accumulators.
__device__ __forceinline__ void warp_mma(const double* A, const double* B, int kb, int ke, int rt, int ct,
                                         double& d0, double& d1) {
  const int lane = threadIdx.x & 31;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
  const int boff = ct * 32 + (lane & 3) * 8 + (lane >> 2);
  int ks = kb;
  for (; ks + 4 <= ke; ks += 4) {
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
  for (; ks < ke; ++ks) dmma4(a0, a1, A[(ks * 2 + rt) * 32 + lane], B[ks * 64 + boff]);
  d0 += (a0 + b0) + (c0 + e0);
  d1 += (a1 + b1) + (c1 + e1);
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
  const double* Phi;   // L inflow propagators (C-part of the U kernel)
  const double* Psi;   // U inflow propagators (C-part of the L kernel)
  const double* TL;    // L boundary products
  const double* TU;    // U boundary products (mirrored indices)
  // state
  double* Yt;          // per chain n_sp: ytilde, then y (in place)
  double* Xt;          // per chain n_sp: xtilde
  double* Yend;        // [set][NG][kVec]: ytilde at each group's last row
  double* Xend;        // [set][NG][kVec]: xtilde at each group's first row
  double* EP;          // [set][NG][maxp][kVec]: partial sums of e_G - Yend(G)
  double* FP;          // [set][NG][maxp][kVec]: partial sums of f_G - Xend(G)
  const int2* bitemsL; // B-phase work items (G, part)
  const int2* bitemsU;
  int nitemsL, nitemsU, maxp;
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
  const double* zeros; // kN zeros: load target of masked-out lanes (branch-free loads)
  const double* LA;    // [J][3][kN]: Li_J a2, Li_J a1, Li_J 1 (two-level residual term)
  int empty;           // debug: KKT_V4_EMPTY=1 kernels return at once (launch floor)
  int no_l2pf;         // debug: KKT_V4_NO_L2PF disables the L2 prefetch of the next kernels' operators
};

__device__ __forceinline__ int nparts_L(int G) { return (G + kBT - 1) / kBT; }

// ---------------------------------------------------------------------------
// A kernel: [C-part of the other direction] then the zero-inflow chain.
//   L (kU = false), time step t:  C-part  x_{t-1,J} = xt_J + Psi_J f_{G+1}
//                                 (outputs of step t-1), then y~ chain.
//   U (kU = true):                C-part  y_J = y~_J + Phi_J e_{G-1} (in place),
//                                 then x~ chain.
// `final_only`: the C-part of the last step only (after the last U sweep).
// ---------------------------------------------------------------------------
template <bool kU>
__global__ void __launch_bounds__(kThr4, 1) v4A_kernel(V4Params P, int t, int final_only) {
  extern __shared__ __align__(128) double sm[];
  // [ring 3x2 slices | X 2 vectors | V] doubles as the C-part slab of up to
  // kCMax operator slices (all fetched at once); EV and part follow.
  double* ring = sm;                      // kRing stages x 2 slices
  double* X = ring + kRing * 2 * kSlice;  // 2 exchange buffers
  double* V = X + 2 * kVec;               // 2 off-chain operands (b_J or y_J)
  double* EV = V + 2 * kVec;              // inflow vector of the C-part
  double* part = EV + kVec;               // 4 tiles x 32 lanes x 2
  double* Cb = part + 4 * 32 * 2;         // 2 x (4 tiles x 32 lanes x 2): off-chain tiles
  double* cslab = sm;
  __shared__ __align__(8) uint64_t tbar[kRing];
  __shared__ __align__(8) uint64_t cbar[kCMax];
  __shared__ __align__(8) uint64_t xbar[2];
  __shared__ __align__(8) uint64_t cready[2], cfree[2], sfree[kRing];
  __shared__ FastStep sj[kCs];   // jobs of step t (chain)
  __shared__ FastStep sp[kCs];   // jobs of step t-1 (C-part of the L kernel)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = int(cta_rank());
  const int cid = blockIdx.x / kCl;
  const int G = cid % P.NG, set = cid / P.NG;
  const int J0 = G * P.g, J1 = min(P.ny, J0 + P.g) - 1, len = J1 - J0 + 1;
  const int NG = P.NG;
  const bool cpart = kU ? (!final_only) : (t > 0);
  const bool cinflow = kU ? (G > 0) : (G < NG - 1);
  const bool chain = !final_only;
  const double* Cm = kU ? P.Phi : P.Psi;
  const double* On = kU ? P.OnU : P.OnL;
  const double* Off = kU ? P.OffU : P.OffL;
  // off-chain triangle: Li lower (ks < 4r+4), Ut upper (ks >= 4r)
  const int okb = kU ? 4 * r : 0, oke = kU ? 32 : 4 * r + 4;
  auto rowC = [&](int i) { return J0 + i; };
  auto rowQ = [&](int q) { return kU ? J1 - q : J0 + q; };
  // chain stage q: on-chain slice (q > 0) and off-chain triangle
  auto issue_any = [&](int q) {  // by any one thread
    if (q >= len) return;
    double* dst = ring + (q % kRing) * 2 * kSlice;
    uint64_t* bar = &tbar[q % kRing];
    const int J = rowQ(q);
    const uint32_t offb = uint32_t(oke - okb) * 64 * 8;
    mbar_expect_tx(bar, (q > 0 ? kSlice * 8 : 0) + offb);
    if (q > 0) bulk_g2s(dst, On + (size_t(J) * kCl + r) * kSlice, kSlice * 8, bar);
    bulk_g2s(dst + kSlice + okb * 64, Off + (size_t(J) * kCl + r) * kSlice + okb * 64, offb, bar);
  };
  auto issue = [&](int q) {
    if (tid == 0) issue_any(q);
  };
  // C-part slices i0 .. i0+n-1, all in flight at once
  auto issue_c = [&](int i0, int n) {
    if (tid != 0) return;
    for (int i = 0; i < n; ++i) {
      mbar_expect_tx(&cbar[i], kSlice * 8);
      bulk_g2s(cslab + i * kSlice, Cm + (size_t(rowC(i0 + i)) * kCl + r) * kSlice, kSlice * 8, &cbar[i]);
    }
  };
  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&tbar[i], 1);
    for (int i = 0; i < kCMax; ++i) mbar_init(&cbar[i], 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&cready[i], 128);
      mbar_init(&cfree[i], 128);
    }
    for (int i = 0; i < kRing; ++i) mbar_init(&sfree[i], 256);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // the job table and the operators are constant during the graph: load them
  // before waiting for the predecessor kernel
  if (tid < kCs) {
    const int c = set * kCs + tid;
    FastStep z{nullptr, nullptr, nullptr, nullptr, 1.0, 0, 0};
    sj[tid] = (chain && c < P.nchains) ? P.jobs[int64_t(c) * P.nsteps + t] : z;
    sp[tid] = (!kU && cpart && c < P.nchains) ? P.jobs[int64_t(c) * P.nsteps + (t - 1)] : z;
  }
  __syncthreads();
  if (P.empty == 1) {  // debug: launch-overhead floor
    pdl_wait();
    pdl_launch();
    cluster_sync_all();
    return;
  }
  const bool use_slab = cpart && cinflow;
  if (use_slab) {
    issue_c(0, min(len, kCMax));
  } else if (chain) {
    issue(0);
    issue(1);
  }
  // Pull the operators of the next two kernels into L2 while this one runs
  // (the operator set of all four kernels exceeds the L2, so a cyclic sweep
  // would miss every time): the B kernel of this direction (its propagator
  // products of group G, slice r) and the A kernel of the other direction
  // (C-part, on- and off-chain slices of the same group and slice).
  if (warp == 1 && chain && !P.no_l2pf) {
    const double* Cn = kU ? P.Psi : P.Phi;
    const double* Onn = kU ? P.OnL : P.OnU;
    const double* Offn = kU ? P.OffL : P.OffU;
    const int nkb = kU ? 0 : 4 * r, nke = kU ? 4 * r + 4 : 32;  // the other triangle
    for (int i = lane; i < len; i += 32) {
      const size_t base = (size_t(J0 + i) * kCl + r) * kSlice;
      l2_prefetch(Cn + base, kSlice * 8);
      l2_prefetch(Onn + base, kSlice * 8);
      l2_prefetch(Offn + base + nkb * 64, uint32_t(nke - nkb) * 64 * 8);
    }
    const double* T = kU ? P.TU : P.TL;
    const int nterms = kU ? NG - 1 - G : G;
    for (int j = lane; j < nterms; j += 32) {
      const int m = kU ? tri_idx(NG - 1 - G, NG - 1 - (G + 1 + j)) : tri_idx(G, j);
      l2_prefetch(T + (size_t(m) * kCl + r) * kSlice, kSlice * 8);
    }
  }
  long long* tim = (P.tim && tid == 0) ? P.tim + (size_t(kU) * gridDim.x + blockIdx.x) * 32 : nullptr;
  if (tim) tim[0] = clock64();
  pdl_wait();  // everything below reads the predecessors' outputs
  pdl_launch();
  if (tim) tim[1] = clock64();

  const int t4 = warp & 3, rt = t4 >> 1, ct = t4 & 1;
  const bool owner = warp < 4;  // kh == 0 warps hold the reduced tiles
  const int krow = r * kRows + rt * 8 + (lane >> 2);  // this lane's block row
  const int nch = ct * 8 + 2 * (lane & 3);            // this lane's chain pair
  const int cpair = set * kCs + nch;                  // global chain of the pair's first

  // ---------------- C-part -------------------------------------------------
  // inflow vector e_{G-1} (U kernel) or f_{G+1} (L kernel): group-end value
  // plus the chunk partials, summed in a fixed order
  if (use_slab) {
    const int Gs = kU ? G - 1 : G + 1;
    const double* endv = (kU ? P.Yend : P.Xend) + (size_t(set) * NG + Gs) * kVec;
    const double* pp = (kU ? P.EP : P.FP) + (size_t(set) * NG + Gs) * P.maxp * kVec;
    const int np = kU ? nparts_L(Gs) : nparts_L(NG - 1 - Gs);
    constexpr int kU8 = kVec / kThr4;
    double v[kU8];
#pragma unroll
    for (int u = 0; u < kU8; ++u) v[u] = endv[tid + u * kThr4];
    for (int p0 = 0; p0 < np; p0 += 4) {  // 4 partials' loads in flight at once
      double w[4][kU8];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double* src = p0 + p < np ? pp + size_t(p0 + p) * kVec : P.zeros;
        const int stride = p0 + p < np ? kThr4 : 0;
#pragma unroll
        for (int u = 0; u < kU8; ++u) w[p][u] = src[(p0 + p < np ? tid : 0) + u * stride];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int u = 0; u < kU8; ++u) v[u] += w[p][u];
    }
#pragma unroll
    for (int u = 0; u < kU8; ++u) EV[tid + u * kThr4] = v[u];
  }
  // base values of the C-part rows (x~ for L, y~ for U), kCMax rows per batch
  double base0[kCMax], base1[kCMax];
  const bool rowok = owner && krow < P.nx;
  auto load_base = [&](int i0) {
    const double* src = kU ? P.Yt : P.Xt;
    const int kr = krow < P.nx ? krow : 0;
#pragma unroll
    for (int u = 0; u < kCMax; ++u) {
      const int ii = i0 + u < len ? i0 + u : 0;
      const size_t p = size_t(rowC(ii)) * P.nx + kr;
      base0[u] = src[size_t(cpair) * P.nsp + p];
      base1[u] = src[size_t(cpair + 1) * P.nsp + p];
    }
  };
  if (cpart) load_base(0);
  // peer exchange buffers are armed before anyone can send (cluster barrier)
  if (tid == 0 && chain) {
    mbar_expect_tx(&xbar[0], (kCl - 1) * kRows * kCs * 8);
    mbar_expect_tx(&xbar[1], (kCl - 1) * kRows * kCs * 8);
  }
  cluster_sync_all();
  if (tim) tim[2] = clock64();

  if (cpart) {
    double g2[2] = {0.0, 0.0};
    if (!kU && P.gam) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (sp[nch + u].out2 && sp[nch + u].node2 > 0) g2[u] = P.gam[sp[nch + u].node2];
    }
    uint32_t cph = 0;
    for (int i0 = 0; i0 < len; i0 += kCMax) {
      if (i0 > 0) {
        load_base(i0);
        if (use_slab) issue_c(i0, min(len - i0, kCMax));  // the previous batch's reads are done
      }
#pragma unroll
      for (int u = 0; u < kCMax; ++u) {
        const int i = i0 + u;
        if (i >= len) break;
        const int J = rowC(i);
        double d0 = base0[u], d1 = base1[u];
        if (use_slab) {
          mbar_wait(&cbar[u], cph);
          cta_mma(cslab + u * kSlice, EV, 0, 32, part, d0, d1);
        }
        if (rowok) {
          const int p = J * P.nx + krow;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const double x = w ? d1 : d0;
            if (kU) {
              if (cinflow && sj[nch + w].in) P.Yt[size_t(cpair + w) * P.nsp + p] = x;
            } else {
              const FastStep& st = sp[nch + w];
              if (st.in) {
                if (st.out) st.out[p] = x;
                if (st.out2) st.out2[p] = x + g2[w];
              }
            }
          }
        }
      }
      cph ^= 1u;
    }
    // the slab is free (cta_mma ends with __syncthreads): start the chain's ring
    if (use_slab && chain) {
      issue(0);
      issue(1);
    }
    cluster_sync_all();  // the group's rows are complete for every CTA of the cluster
  }
  if (tim) tim[3] = clock64();
  if (!chain) return;

  // ---------------- the zero-inflow chain (warp-specialised) -----------------
  // warps 0-3: the dependent chain, one output tile each:
  //     wait for the peers' slices of the previous row, + G_J y_{J-1}
  //     (H_J x_{J+1}), + the off-chain tile, send the slice to the peers.
  // warps 4-7: the off-chain term of the rows ahead, c_J = Li_J b_J
  //     (d_J = Ut_J y_J), one tile each, handed over through Cb[q&1]
  //     (cready/cfree), plus the operand loads and the TMA ring refills.
  // Ring stage q (on slice + off triangle) is freed by all 256 threads (sfree).
  const uint32_t xb_base = smem_u32(&xbar[0]);  // xbar[1] at +8
  double* ybase = kU ? P.Xt : P.Yt;
  if (warp < 4) {
    for (int q = 0; q < len; ++q) {
      const int J = rowQ(q);
      const int st = q % kRing;
      long long m0 = tim ? clock64() : 0;
      mbar_wait(&tbar[st], uint32_t(q / kRing) & 1u);
      double y0 = 0.0, y1 = 0.0;
      long long m1 = tim ? clock64() : 0, m2 = m1;
      if (q > 0) {
        const int xb = (q - 1) & 1;
        mbar_wait_cluster(&xbar[xb], uint32_t((q - 1) >> 1) & 1u);
        if (tim) m2 = clock64();
        // re-arm for the next use (peers refill it only after receiving this
        // CTA's next slices, sent below after every chain warp read it)
        if (tid == 0) mbar_expect_tx(&xbar[xb], (kCl - 1) * kRows * kCs * 8);
        warp_mma(ring + st * 2 * kSlice, X + xb * kVec, 0, 32, rt, ct, y0, y1);
      }
      mbar_arrive(&sfree[st]);
      long long m3 = tim ? clock64() : 0;
      mbar_wait(&cready[q & 1], uint32_t(q >> 1) & 1u);
      long long m4 = tim ? clock64() : 0;
      y0 += Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2];
      y1 += Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2 + 1];
      mbar_arrive(&cfree[q & 1]);
      const int xi = vidx(krow, nch);
      if (q + 1 < len) {
        double* xs = X + (q & 1) * kVec + xi;
        *reinterpret_cast<double2*>(xs) = make_double2(y0, y1);
        const uint32_t loc = smem_u32(xs);
#pragma unroll
        for (int pr = 1; pr < kCl; ++pr) {
          const uint32_t peer = (uint32_t(r) + pr) % kCl;
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                  mapa_u32(loc, peer)),
              "d"(y0), "d"(y1), "r"(mapa_u32(xb_base + 8u * uint32_t(q & 1), peer))
              : "memory");
        }
      } else {
        // group-end value for the B phase: L -> last row J1, U -> first row J0
        double* ev = (kU ? P.Xend : P.Yend) + (size_t(set) * NG + G) * kVec + xi;
        *reinterpret_cast<double2*>(ev) = make_double2(y0, y1);
      }
      if (krow < P.nx) {
        const int p = J * P.nx + krow;
        if (sj[nch].in) ybase[size_t(cpair) * P.nsp + p] = y0;
        if (sj[nch + 1].in) ybase[size_t(cpair + 1) * P.nsp + p] = y1;
      }
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
    // operand loads: warp (w-4) -> chains 4(w-4) + lane/8, rows (lane&7) + 8u
    const int vn = 4 * (warp - 4) + (lane >> 3), vk0 = lane & 7;
    const FastStep vst = sj[vn];
    const bool vact = vst.in != nullptr;
    double xin[16], xad[16];
    auto load_v = [&](int J) {
      // every address valid (masked lanes read `zeros`), so all loads issue at once
      const double* pin;
      const double* padd;
      if (kU) {
        pin = vact ? P.Yt + size_t(set * kCs + vn) * P.nsp + size_t(J) * P.nx : P.zeros;
        padd = P.zeros;
      } else {
        pin = vact ? vst.in + size_t(J) * P.nx : P.zeros;
        padd = (vact && vst.add) ? vst.add + size_t(J) * P.nx : P.zeros;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = vk0 + 8 * u < P.nx ? vk0 + 8 * u : 0;
        xin[u] = pin[k];
        if (!kU) xad[u] = padd[k];
      }
    };
    auto store_v = [&](int b) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = vk0 + 8 * u;
        const double v = kU ? xin[u] : fma(xin[u], vst.scale, xad[u]);
        V[b * kVec + vidx(k, vn)] = (vact && k < P.nx) ? v : 0.0;
      }
    };
    // the two-level residual term of the L right-hand side, b -= (Shat y_c)_node / ms,
    // enters after the product: Li_J (Shat y_c) = al*Li a2 - be*Li a1 + ga*Li 1
    // with per-chain scalars from the coarse values gamma (sweep.cu jobs, node)
    const bool lacoef = !kU && P.coarse;
    double al[2] = {0.0, 0.0}, be[2] = {0.0, 0.0}, ga[2] = {0.0, 0.0};
    if (lacoef) {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const FastStep& sw = sj[nch + w];
        if (sw.in && sw.node > 0) {
          const double gn = P.gam[sw.node], gp = P.gam[sw.node + 1];
          const bool d = sw.node != 1;
          const double gm = d ? P.gam[sw.node - 1] : 0.0;
          al[w] = gn * P.inv_ms;
          be[w] = (gp + gm) * P.inv_ms;
          ga[w] = d ? gn * P.inv_ms : 0.0;
        }
      }
    }
    double la2 = 0.0, la1 = 0.0, la0 = 0.0;
    auto load_la = [&](int J) {
      if (!lacoef) return;
      const double* la = P.LA + size_t(J) * 3 * kN + (krow < kN ? krow : 0);  // Li a2, Li a1, Li 1
      la2 = la[0];
      la1 = la[kN];
      la0 = la[2 * kN];
    };
    load_v(rowQ(0));
    load_la(rowQ(0));
    store_v(0);
    if (len > 1) load_v(rowQ(1));
    named_bar_sync(1, 128);
    for (int q = 0; q < len; ++q) {
      const int st = q % kRing;
      const double cl2 = la2, cl1 = la1, cl0 = la0;
      if (q + 1 < len) load_la(rowQ(q + 1));
      mbar_wait(&tbar[st], uint32_t(q / kRing) & 1u);
      double c0 = 0.0, c1 = 0.0;
      warp_mma(ring + st * 2 * kSlice + kSlice, V + (q & 1) * kVec, okb, oke, rt, ct, c0, c1);
      mbar_arrive(&sfree[st]);
      if (lacoef && krow < P.nx) {
        c0 -= al[0] * cl2 - be[0] * cl1 + ga[0] * cl0;
        c1 -= al[1] * cl2 - be[1] * cl1 + ga[1] * cl0;
      }
      if (q >= 2) mbar_wait(&cfree[q & 1], uint32_t((q >> 1) - 1) & 1u);
      Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2] = c0;
      Cb[(q & 1) * 256 + (t4 * 32 + lane) * 2 + 1] = c1;
      mbar_arrive(&cready[q & 1]);
      // refill: stage q+kRing-1 goes to the slot of stage q-1 once both
      // groups are done with it
      if (ot == 0 && q + kRing - 1 < len) {
        if (q >= 1) mbar_wait(&sfree[(q - 1) % kRing], uint32_t((q - 1) / kRing) & 1u);
        issue_any(q + kRing - 1);
      }
      if (q + 1 < len) {
        named_bar_sync(1, 128);  // every off warp is done reading V[(q+1)&1] (row q-1)
        store_v((q + 1) & 1);
        if (q + 2 < len) load_v(rowQ(q + 2));
        named_bar_sync(1, 128);  // V[(q+1)&1] complete
      }
    }
  }
  if (tim) tim[31] = clock64();
  cluster_sync_all();  // no CTA exits while a peer may still address its shared memory
}

// ---------------------------------------------------------------------------
// B kernel: chunk partials of the boundary values
//   L: e_G - Yend(G) = sum_{i<G} TL_{G,i} Yend(i)
//   U: f_G - Xend(G) = sum_{i>G} TU_{m(G),m(i)} Xend(i),  m(x) = NG-1-x
// one CTA per (set, item = (G, chunk), row slice r); up to kBT products.
// ---------------------------------------------------------------------------
template <bool kU>
__global__ void __launch_bounds__(kThr4) v4B_kernel(V4Params P) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                 // 2 stages x (T slice + vector)
  double* part = ring + 2 * (kSlice + kVec);
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, lane = tid & 31;
  const int nitems = kU ? P.nitemsU : P.nitemsL;
  const int r = blockIdx.x % kCl;
  const int it = (blockIdx.x / kCl) % nitems;
  const int set = blockIdx.x / (kCl * nitems);
  const int2 item = (kU ? P.bitemsU : P.bitemsL)[it];
  const int G = item.x, chunk = item.y;
  const int NG = P.NG;
  const int nterms = kU ? NG - 1 - G : G;
  const int i0 = chunk * kBT, i1 = min(nterms, i0 + kBT);
  const double* T = kU ? P.TU : P.TL;
  const double* endv = (kU ? P.Xend : P.Yend) + size_t(set) * NG * kVec;
  auto src_group = [&](int j) { return kU ? G + 1 + j : j; };
  auto tmat = [&](int j) { return kU ? tri_idx(NG - 1 - G, NG - 1 - src_group(j)) : tri_idx(G, j); };
  if (P.empty) {  // debug: launch-overhead floor
    pdl_wait();
    pdl_launch();
    return;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue_T = [&](int j) {  // operator slice: independent of the predecessors
    if (tid == 0 && j < i1) {
      double* dst = ring + ((j - i0) & 1) * (kSlice + kVec);
      mbar_expect_tx(&bar[(j - i0) & 1], (kSlice + kVec) * 8);
      bulk_g2s(dst, T + (size_t(tmat(j)) * kCl + r) * kSlice, kSlice * 8, &bar[(j - i0) & 1]);
    }
  };
  auto issue_v = [&](int j) {
    if (tid == 0 && j < i1) {
      double* dst = ring + ((j - i0) & 1) * (kSlice + kVec) + kSlice;
      bulk_g2s(dst, endv + size_t(src_group(j)) * kVec, kVec * 8, &bar[(j - i0) & 1]);
    }
  };
  issue_T(i0);
  issue_T(i0 + 1);
  pdl_wait();
  pdl_launch();

  issue_v(i0);
  issue_v(i0 + 1);
  double d0 = 0.0, d1 = 0.0;
  uint32_t ph = 0;
  for (int j = i0; j < i1; ++j) {
    const int b = (j - i0) & 1;
    mbar_wait(&bar[b], (ph >> b) & 1u);
    ph ^= 1u << b;
    const double* st = ring + b * (kSlice + kVec);
    cta_mma(st, st + kSlice, 0, 32, part, d0, d1);  // ends with __syncthreads: stage free
    issue_T(j + 2);
    issue_v(j + 2);
  }
  if (threadIdx.x < 128) {
    const int warp = threadIdx.x >> 5, t4 = warp & 3, rt = t4 >> 1, ct = t4 & 1;
    const int krow = r * kRows + rt * 8 + (lane >> 2);
    const int nch = ct * 8 + 2 * (lane & 3);
    double* out = (kU ? P.FP : P.EP) + ((size_t(set) * NG + G) * P.maxp + chunk) * kVec + vidx(krow, nch);
    *reinterpret_cast<double2*>(out) = make_double2(d0, d1);
  }
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

void launch_ex(Ctx* c, const void* fn, int grid, size_t smem, bool cluster, void** args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThr4);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
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

size_t smemA() { return sizeof(double) * (size_t(kRing) * 2 * kSlice + 5 * size_t(kVec) + 3 * 4 * 32 * 2); }
size_t smemB() { return sizeof(double) * (2 * size_t(kSlice + kVec) + 4 * 32 * 2); }

}  // namespace

bool v4_supported(const Ctx* c) { return c->nx <= kN && c->ny >= 2 && !getenv("KKT_SWEEP_V3"); }

void set_v4_attributes() {
  static bool done = false;
  if (done) return;
  KKT_CUDA(cudaFuncSetAttribute(v4A_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemA())));
  KKT_CUDA(cudaFuncSetAttribute(v4A_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemA())));
  KKT_CUDA(cudaFuncSetAttribute(v4B_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemB())));
  KKT_CUDA(cudaFuncSetAttribute(v4B_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemB())));
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
  c->v4_ops.alloc(6 * per + 2 * size_t(ntri) * kMat);
  double* base = c->v4_ops.p;
  auto pack = [&](const double* src, int64_t sstride, int ld, int n, int mode, int count, double* dst) {
    const dim3 grid(16, count);
    KKT_LAUNCH(c, frag_pack_kernel, grid, 256, 0, src, sstride, ld, n, mode, dinv, nx, dst);
  };
  pack(G, kMat, kN, nx, 0, ny, base + 0 * per);                    // OnL
  pack(Li, int64_t(nx) * nx, nx, nx, 0, ny, base + 1 * per);       // OffL
  pack(H, kMat, kN, nx, 0, ny, base + 2 * per);                    // OnU
  pack(Li, int64_t(nx) * nx, nx, nx, 1, ny, base + 3 * per);       // OffU = Li^T D^{-1}
  pack(c->Phi.p, kMat, kN, nx, 0, ny, base + 4 * per);
  pack(c->Psi.p, kMat, kN, nx, 0, ny, base + 5 * per);
  if (NG > 1) {
    pack(c->grp_tl.p, kMat, kN, nx, 0, NG * (NG - 1) / 2, base + 6 * per);
    pack(c->grp_tu.p, kMat, kN, nx, 0, NG * (NG - 1) / 2, base + 6 * per + size_t(ntri) * kMat);
  }
  static_assert(kCMax * kSlice <= kRing * 2 * kSlice + 3 * kVec, "C slab exceeds ring + X + V");
  // The operators are re-read every time step (131 MB at config 1, more than
  // the L2 holds, so a cyclic sweep would miss every time): mark as much of
  // them as the persisting carve-out allows as L2-persisting.
  if (!getenv("KKT_NO_L2PIN")) {
    int max_persist = 0, max_window = 0;
    KKT_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device));
    KKT_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device));
    if (max_persist > 0 && max_window > 0) {
      const size_t bytes = std::min(sizeof(double) * c->v4_ops.n, size_t(max_window));
      const size_t carve = std::min(bytes, size_t(max_persist));
      KKT_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = c->v4_ops.p;
      attr.accessPolicyWindow.num_bytes = bytes;
      attr.accessPolicyWindow.hitRatio = float(std::min(1.0, double(carve) / double(bytes)));
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      KKT_CUDA(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr));
      if (getenv("KKT_V4_TIM"))
        fprintf(stderr, "v4: L2 persisting carve %zu of window %zu (max persist %d, max window %d)\n", carve, bytes,
                max_persist, max_window);
    }
  }
  // B-phase work items
  std::vector<int2> iL, iU;
  int maxp = 1;
  for (int Gg = 0; Gg < NG; ++Gg) {
    const int nl = (Gg + kBT - 1) / kBT, nu = (NG - 1 - Gg + kBT - 1) / kBT;
    for (int p = 0; p < nl; ++p) iL.push_back(make_int2(Gg, p));
    for (int p = 0; p < nu; ++p) iU.push_back(make_int2(Gg, p));
    maxp = std::max(maxp, std::max(nl, nu));
  }
  c->v4_maxp = maxp;
  c->v4_zero.alloc(kN);
  KKT_CUDA(cudaMemsetAsync(c->v4_zero.p, 0, sizeof(double) * kN, c->stream));
  c->v4_nitemsL = int(iL.size());
  c->v4_nitemsU = int(iU.size());
  c->v4_items.alloc(iL.size() + iU.size() + 1);
  if (!iL.empty())
    KKT_CUDA(cudaMemcpyAsync(c->v4_items.p, iL.data(), sizeof(int2) * iL.size(), cudaMemcpyHostToDevice, c->stream));
  if (!iU.empty())
    KKT_CUDA(cudaMemcpyAsync(c->v4_items.p + iL.size(), iU.data(), sizeof(int2) * iU.size(),
                             cudaMemcpyHostToDevice, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  set_v4_attributes();
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
    c->v4_state.alloc(size_t(2 * nsets * kCs) * c->nsp + 2 * nvec * (1 + c->v4_maxp));
    KKT_CUDA(cudaMemsetAsync(c->v4_state.p, 0, sizeof(double) * c->v4_state.n, c->stream));
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
  P.Phi = ops + 4 * per;
  P.Psi = ops + 5 * per;
  P.TL = ops + 6 * per;
  P.TU = ops + 6 * per + size_t(ntri) * kMat;
  double* st = c->v4_state.p;
  P.Yt = st;
  P.Xt = st + size_t(nsets_alloc * kCs) * c->nsp;
  double* vb = st + size_t(2 * nsets_alloc * kCs) * c->nsp;
  P.Yend = vb;
  P.Xend = vb + nveca;
  P.EP = vb + 2 * nveca;
  P.FP = vb + 2 * nveca + nveca * c->v4_maxp;
  P.bitemsL = c->v4_items.p;
  P.bitemsU = c->v4_items.p + c->v4_nitemsL;
  P.nitemsL = c->v4_nitemsL;
  P.nitemsU = c->v4_nitemsU;
  P.maxp = c->v4_maxp;
  P.a1 = c->a1.p;
  P.a2 = c->a2.p;
  P.gam = c->gam.p;
  P.inv_ms = 1.0 / c->ms;
  P.nx = c->nx;
  P.ny = c->ny;
  P.nsp = c->nsp;
  P.g = c->grp_g;
  P.NG = NG;
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
  P.no_l2pf = getenv("KKT_V4_NO_L2PF") ? 1 : 0;
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
  const size_t sA = smemA(), sB = smemB();
  auto sequence = [&]() {
    for (int t = 0; t <= nsteps; ++t) {
      int fin = t == nsteps ? 1 : 0;
      {
        void* args[] = {&P, &t, &fin};
        launch_ex(c, reinterpret_cast<const void*>(&v4A_kernel<false>), gridA, sA, true, args);
      }
      if (fin) break;
      if (P.nitemsL > 0) {
        void* args[] = {&P};
        launch_ex(c, reinterpret_cast<const void*>(&v4B_kernel<false>), nsets * P.nitemsL * kCl, sB, false, args);
      }
      {
        int zero = 0;
        void* args[] = {&P, &t, &zero};
        launch_ex(c, reinterpret_cast<const void*>(&v4A_kernel<true>), gridA, sA, true, args);
      }
      if (P.nitemsU > 0) {
        void* args[] = {&P};
        launch_ex(c, reinterpret_cast<const void*>(&v4B_kernel<true>), nsets * P.nitemsU * kCl, sB, false, args);
      }
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
            if (i >= 20 && i <= 25) {
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
        fprintf(stderr, " | tail %.0f | sums: tma %.0f xwait %.0f on %.0f cwait %.0f send %.0f (unused %.0f)\n", acc[31] / cnt,
                acc[20] / cnt, acc[21] / cnt, acc[22] / cnt, acc[23] / cnt, acc[24] / cnt, acc[25] / cnt);
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
}

}  // namespace kkt
