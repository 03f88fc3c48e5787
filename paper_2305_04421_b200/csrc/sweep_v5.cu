// sweep_v5.cu — FAST spatial-solve chains for large grids (128 < nx <= 511:
// configs 2 and 3), cluster-cooperative block substitution with the chains
// batched into fp64 tensor-core tiles.
//
// The method is the reference's LU solve (BandedLU::solve_in_place /
// solve_transpose_in_place, linalg.cpp:127-162) in the block form of
// sweep_fast.cu, on the block-recursion factors of factor_block.cu
// (Li_J = L_JJ^{-1}, Ui_J = U_JJ^{-1}):
//     L sweep  y_J = Li_J b_J + G_J y_{J-1},   G_J = cy Li_J Ui_{J-1}
//     U sweep  x_J = Ui_J y_J + H_J x_{J+1},   H_J = cy Ui_J Li_J
// i.e. sweep_fast.cu's  y_J = Li_J (b_J + cy Ui_{J-1} y_{J-1})  and
// x_J = Ui_J (y_J + cy Li_J x_{J+1})  with the two dependent triangular
// products of a block step pre-multiplied (same factors, re-associated:
// rounding-level differences, gated like the rest of FAST).
//
// Mapping.  Chains (time subdomains) are independent, so each set of 8
// chains runs its whole job list — every step, both sweep directions —
// inside ONE cluster of kN/32 CTAs with no inter-cluster traffic at all; one
// launch per RASQ application.  CTA r owns block rows 32r..32r+31 of every
// block step and computes them for the 8 chains of its set as four 8x8 fp64
// DMMA tiles (m8n8k4), so every operator element read serves 8 chains.
//   * warps 0-3 (chain): y_J tile = G_J[rows] * y_{J-1} + c_J tile; the
//     32-row slice of the result goes to every CTA of the cluster (itself
//     included) by st.async into DSMEM, completing on the receivers'
//     mbarrier (double-buffered), so the next block step can start as soon
//     as the last slice lands.
//   * warps 4-7 (off-chain): c_J = Li_J b_J (L) / d_J = Ui_J y_J (U) for the
//     rows ahead, over the nonzero 64-column chunks of the triangle only;
//     they build the operand b_J = in*scale + add - (Shat y_c)/ms (the fused
//     two-level residual, schur.cpp:435-437, analytically as sweep_fast.cu)
//     from the reference-layout planes, one block row ahead in registers.
//   * warp 8 / warp 9 (producers): keep the on-chain / off-chain operator
//     rings full with cp.async.bulk copies of 16 KB chunks (32 rows x 64
//     columns, fragment ordered), mbarrier transaction counts.
//   * between sweep directions the cluster synchronises once (release /
//     acquire at cluster scope): the U sweep's operand y_J and the next L
//     sweep's operand x_{t-1} are global rows written by the other CTAs.
//
// Layouts.  Operators: per block row J, per CTA r, per 64-column chunk c a
// contiguous 16 KB chunk [ks 16][rt 4][lane 32] holding
// M[32r + 8rt + lane/4][64c + 4ks + lane%4] (the A operand of m8n8k4 read as
// 32 consecutive doubles per warp), zero padded to kN.  Block vectors of kN
// rows x 8 chains: [k][n] (the B operand reads 32 consecutive doubles; the
// D fragment writes a chain pair as one double2).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sweep_tma.cuh"

namespace kkt {
namespace {
using namespace tma;

constexpr int kS = 8;           // chains per set (the n of m8n8k4)
constexpr int kRowsV5 = 32;     // block rows per CTA
constexpr int kChunk = 2048;    // doubles per operator chunk: 32 rows x 64 columns
constexpr int kThr5 = 320;      // 4 chain + 4 off-chain + 2 producer warps

template <int kN> struct V5Cfg {
  static constexpr int CL = kN / kRowsV5;     // CTAs per cluster
  static constexpr int NCH = kN / 64;         // chunks per row slice
  // a bulk copy costs ~420 cycles of the SM's TMA unit whatever its size up
  // to 32 KB (scripts/mb_tma.cu), so the on-chain stream moves CC chunks per copy
  static constexpr int CC = kN == 512 ? 2 : 1;  // chunks per on-chain copy
  static constexpr int NC = kN == 512 ? 2 : 4;  // on-chain ring slots (CC chunks each)
  static constexpr int NO = kN == 512 ? 3 : 4;  // off-chain ring slots (1 chunk each)
  static constexpr int NOP = NCH / CC;          // on-chain copies per row slice
  // resident operators: the whole row slice in the ring regions (kN = 256)
  static constexpr bool kRes = NC * CC >= NCH && NO >= NCH;
  static constexpr int VEC = kN * kS;         // doubles per block vector
  static constexpr int PER = VEC / 128;       // operand elements per off-chain thread
  static constexpr size_t smem = sizeof(double) * (size_t(NC * CC + NO) * kChunk + 3 * size_t(VEC) + 2 * 256);
};

struct V5Params {
  const double* OnL;   // G_J
  const double* OffL;  // Li_J
  const double* OnU;   // H_J
  const double* OffU;  // Ui_J
  double* Y;           // [set][J][VEC]: the L sweep's y_J
  const double* LA;    // [J][3][kN]: Li_J a2, Li_J a1, Li_J 1 (two-level residual term)
  const double* gam;
  double inv_ms;
  int nx, ny, nchains, nsteps, coarse;
  const FastStep* jobs;
  int jstar;          // block rows J >= jstar use the resident operators of row jstar
  long long* tim;      // debug (KKT_V5_TIM): per-CTA clock64 sums, null in production
};

__device__ __forceinline__ uint32_t cta_rank5() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa5(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void expect_tx5(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void arrive5(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void wait_cluster5(uint64_t* b, uint32_t par) {
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
__device__ __forceinline__ void g2s5(double* dst, const double* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void dmma5(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// One warp: tile rt (8 rows) x 8 chains += chunk (32 rows x 64 columns) x B (64 x 8).
// The operands of the next 4 k-steps are loaded while the current 4 DMMAs are
// in the pipe (a lone warp otherwise waits for shared memory every 4 DMMAs:
// scripts/mb_dmma_smem.cu).
__device__ __forceinline__ void chunk_mma(const double* A, const double* B, int rt, double (&acc)[4][2]) {
  const int lane = threadIdx.x & 31;
  const double* Ap = A + rt * 32 + lane;
  const double* Bp = B + (lane & 3) * 8 + (lane >> 2);
  double av[4], bv[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    av[u] = Ap[u * 128];
    bv[u] = Bp[u * 32];
  }
#pragma unroll
  for (int ks = 4; ks < 16; ks += 4) {
    double an[4], bn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      an[u] = Ap[(ks + u) * 128];
      bn[u] = Bp[(ks + u) * 32];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma5(acc[u][0], acc[u][1], av[u], bv[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      av[u] = an[u];
      bv[u] = bn[u];
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) dmma5(acc[u][0], acc[u][1], av[u], bv[u]);
}

// nonzero 64-column chunks of CTA r's triangle slice: Li lower (k <= 32r+31),
// Ui upper (k >= 32r)
__device__ __forceinline__ void tri_range(bool up, int r, int nch, int& cb, int& ce) {
  if (up) {
    cb = (32 * r) / 64;
    ce = nch;
  } else {
    cb = 0;
    ce = (32 * r + 31) / 64 + 1;
  }
}

template <int kN>
__global__ void __launch_bounds__(kThr5, 1) v5_kernel(V5Params P) {
  using C = V5Cfg<kN>;
  constexpr int CL = C::CL, NCH = C::NCH, NC = C::NC, NO = C::NO, VEC = C::VEC, PER = C::PER;
  constexpr int CC = C::CC, NOP = C::NOP;
  extern __shared__ __align__(128) double sm[];
  double* ringC = sm;
  double* ringO = ringC + NC * CC * kChunk;
  double* X = ringO + NO * kChunk;   // 2 x VEC exchange buffers
  double* V = X + 2 * VEC;           // off-chain operand
  double* Cb = V + VEC;              // 2 x 256 off-chain tiles
  __shared__ __align__(8) uint64_t fullC[NC], freeC[NC], fullO[NO], freeO[NO], xbar[2], cready[2], cfree[2];
  __shared__ __align__(8) uint64_t resFullA, resFreeA, resFullB, resFreeB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = int(cta_rank5());
  const int set = blockIdx.x / CL;
  const int ny = P.ny, nx = P.nx, nsteps = P.nsteps;
  const int nsweeps = 2 * nsteps;
  constexpr uint32_t kSliceBytes = kRowsV5 * kS * 8;  // one CTA's rows of a block vector

  if (P.tim && tid == 0) P.tim[size_t(blockIdx.x) * 16 + 15] = clock64();
  if (tid == 0) {
    for (int i = 0; i < NC; ++i) {
      mbar_init(&fullC[i], 1);
      mbar_init(&freeC[i], 128);
    }
    for (int i = 0; i < NO; ++i) {
      mbar_init(&fullO[i], 1);
      mbar_init(&freeO[i], 128);
    }
    // exchange barriers, one per buffer: every CTA's slice (this one's too)
    // arrives by st.async and completes transaction bytes
    for (int i = 0; i < 2; ++i) {
      mbar_init(&xbar[i], 1);
      mbar_init(&cready[i], 128);
      mbar_init(&cfree[i], 128);
    }
    mbar_init(&resFullA, 1);
    mbar_init(&resFreeA, 128);
    mbar_init(&resFullB, 1);
    mbar_init(&resFreeB, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int i = 0; i < 2; ++i) expect_tx5(&xbar[i], CL * kSliceBytes);
  }
  cl_arrive();
  cl_wait();

  auto rowJ = [&](bool up, int q) { return up ? ny - 1 - q : q; };
  const size_t mat = size_t(kN) * kN;

  if (warp < 4) {
    // ------------------------------------------------------------ chain warps
    const int rt = warp;
    const int a = kRowsV5 * r + 8 * rt + (lane >> 2);  // this lane's row within the block
    const int n0 = 2 * (lane & 3);                      // this lane's chain pair
    const uint32_t xb0 = smem_u32(X);
    uint32_t sc = 0, gq = 0, cres_n = 0;
    bool cres = false;
    long long* tim = (P.tim && tid == 0) ? P.tim + size_t(blockIdx.x) * 16 : nullptr;
    long long m0 = 0, m1 = 0;
    for (int k = 0; k < nsweeps; ++k) {
      const int t = k >> 1;
      const bool up = k & 1;
      FastStep st[2];
      double g2[2] = {0.0, 0.0};
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int ch = set * kS + n0 + w;
        st[w] = ch < P.nchains ? P.jobs[size_t(ch) * nsteps + t]
                               : FastStep{nullptr, nullptr, nullptr, nullptr, 1.0, 0, 0};
        if (up && st[w].in && st[w].out2 && st[w].node2 > 0 && P.gam) g2[w] = P.gam[st[w].node2];
      }
      for (int q = 0; q < ny; ++q, ++gq) {
        const int J = rowJ(up, q);
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        if (tim) m0 = clock64();
        if (gq > 0) {
          // the previous row, chunk by chunk as its slices land: this CTA's
          // own chunk first, then the others in rotated order (fixed per CTA)
          const uint32_t pb = (gq - 1) & 1u, par = ((gq - 1) >> 1) & 1u;
          auto wait_all = [&]() {
            wait_cluster5(&xbar[pb], par);
            if (tid == 0) expect_tx5(&xbar[pb], CL * kSliceBytes);  // its next use
          };
          if (q > 0) {
            const double* xv = X + pb * VEC;
            const bool res = J >= P.jstar;
            // every slice first: per-chunk cluster-scope acquires inside the
            // product loop measured slower than one pass here
            if (tim) m0 = clock64();
            wait_all();
            if (tim) { m1 = clock64(); tim[0] += m1 - m0; }
            if (res && !cres) {
              mbar_wait(&resFullA, cres_n & 1u);
              cres = true;
              ++cres_n;
            }
#pragma unroll 1
            for (int i = 0; i < NOP; ++i) {
              const int o = ((r >> 1) / CC + i) % NOP;
              const double* A;
              uint32_t slot = 0;
              if (res) {
                A = ringC + size_t(o) * CC * kChunk;
              } else {
                slot = sc % NC;
                if (tim) m0 = clock64();
                mbar_wait(&fullC[slot], (sc / NC) & 1u);
                if (tim) { m1 = clock64(); tim[1] += m1 - m0; }
                A = ringC + size_t(slot) * CC * kChunk;
              }
#pragma unroll
              for (int u = 0; u < CC; ++u) {
                const int c = o * CC + u;
                if (tim) m0 = clock64();
                chunk_mma(A + u * kChunk, xv + c * 64 * kS, rt, acc);
                if (tim) { m1 = clock64(); tim[2] += m1 - m0; }
              }
              if (!res) {
                arrive5(&freeC[slot]);
                ++sc;
              }
            }
            if (res && (q + 1 == ny || rowJ(up, q + 1) < P.jstar)) {  // end of the resident phase
              arrive5(&resFreeA);
              cres = false;
            }
          } else {
            wait_all();
            if (tim) { m1 = clock64(); tim[0] += m1 - m0; m0 = m1; }
          }
        }
        const uint32_t cb = gq & 1u;
        if (tim) m0 = clock64();
        mbar_wait(&cready[cb], (gq >> 1) & 1u);
        if (tim) { m1 = clock64(); tim[3] += m1 - m0; m0 = m1; }
        double y0 = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
        double y1 = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
        y0 += Cb[cb * 256 + (rt * 32 + lane) * 2];
        y1 += Cb[cb * 256 + (rt * 32 + lane) * 2 + 1];
        arrive5(&cfree[cb]);
        // the slice to every CTA of the cluster (itself included) by st.async
        {
          const uint32_t loc = xb0 + cb * uint32_t(VEC * 8) + uint32_t((a * kS + n0) * 8);
          const uint32_t bar = smem_u32(&xbar[cb]);
#pragma unroll 1
          for (int pr = 0; pr < CL; ++pr) {
            const uint32_t peer = uint32_t((r + pr) % CL);
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                    mapa5(loc, peer)),
                "d"(y0), "d"(y1), "r"(mapa5(bar, peer))
                : "memory");
          }
        }
        if (!up) {
          double* yw = P.Y + (size_t(set) * ny + J) * VEC + a * kS + n0;
          *reinterpret_cast<double2*>(yw) = make_double2(y0, y1);
        } else if (a < nx) {
          const size_t p = size_t(J) * nx + a;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const double v = w ? y1 : y0;
            if (st[w].in) {
              if (st[w].out) st[w].out[p] = v;
              if (st[w].out2) st[w].out2[p] = v + g2[w];
            }
          }
        }
        if (tim) { m1 = clock64(); tim[4] += m1 - m0; }
      }
      if (k > 0) cl_wait();
      cl_arrive();
    }
    // the last exchange has landed before this CTA can exit
    wait_cluster5(&xbar[(gq - 1) & 1u], ((gq - 1) >> 1) & 1u);
    cl_wait();
    if (tim) tim[14] = clock64();
  } else if (warp < 8) {
    // ------------------------------------------------------- off-chain warps
    const int ot = tid - 128, rt = warp - 4;
    const int vn = lane & 7, vk0 = ot >> 3;  // operand element ot + 128u: row vk0 + 16u, chain vn
    const int ch = set * kS + vn;
    uint32_t so = 0, gq = 0, ores_n = 0;
    bool ores = false;
    double xin[PER], xad[PER];
    long long* tim = (P.tim && ot == 0) ? P.tim + size_t(blockIdx.x) * 16 : nullptr;
    long long m0 = 0, m1 = 0;
    for (int k = 0; k < nsweeps; ++k) {
      const int t = k >> 1;
      const bool up = k & 1;
      const FastStep st = ch < P.nchains ? P.jobs[size_t(ch) * nsteps + t]
                                         : FastStep{nullptr, nullptr, nullptr, nullptr, 1.0, 0, 0};
      const bool act = st.in != nullptr;
      // the two-level residual term of the tile's chain pair, after the
      // product: Li_J (Shat y_c)_node / ms = al Li a2 - be Li a1 + ga Li 1
      const int pn0 = 2 * (lane & 3);
      double al[2] = {0.0, 0.0}, be[2] = {0.0, 0.0}, ga[2] = {0.0, 0.0};
      const bool lacoef = !up && P.coarse;
      if (lacoef) {
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int cw = set * kS + pn0 + w;
          if (cw >= P.nchains) continue;
          const FastStep& sw = P.jobs[size_t(cw) * nsteps + t];
          if (!sw.in || sw.node <= 0) continue;
          const double gn = P.gam[sw.node], gp = P.gam[sw.node + 1];
          const bool d = sw.node != 1;
          const double gm = d ? P.gam[sw.node - 1] : 0.0;
          al[w] = gn * P.inv_ms;
          be[w] = (gp + gm) * P.inv_ms;
          ga[w] = d ? gn * P.inv_ms : 0.0;
        }
      }
      const int ta = kRowsV5 * r + 8 * rt + (lane >> 2);  // the tile row of this lane
      double la2 = 0.0, la1 = 0.0, la0 = 0.0;
      auto load_la = [&](int J) {
        if (lacoef) {
          const double* la = P.LA + size_t(J) * 3 * kN + ta;
          la2 = la[0];
          la1 = la[kN];
          la0 = la[2 * kN];
        }
      };
      const double* ysrc = P.Y + size_t(set) * ny * VEC;
      auto load = [&](int J) {
        if (up) {
          const double* src = ysrc + size_t(J) * VEC + ot;
#pragma unroll
          for (int u = 0; u < PER; ++u) xin[u] = src[128 * u];
        } else {
          const size_t base = size_t(J) * nx;
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int kk = vk0 + 16 * u;
            const bool ok = act && kk < nx;
            xin[u] = ok ? st.in[base + kk] : 0.0;
            xad[u] = (ok && st.add) ? st.add[base + kk] : 0.0;
          }
        }
      };
      int cbeg, cend;
      tri_range(up, r, NCH, cbeg, cend);
      load(rowJ(up, 0));
      load_la(rowJ(up, 0));
      for (int q = 0; q < ny; ++q, ++gq) {
        const int J = rowJ(up, q);
        if (tim) m0 = clock64();
        bar_named(1, 128);  // every off warp is done reading V
        if (up) {
#pragma unroll
          for (int u = 0; u < PER; ++u) V[ot + 128 * u] = xin[u];
        } else {
#pragma unroll
          for (int u = 0; u < PER; ++u) V[ot + 128 * u] = fma(xin[u], st.scale, xad[u]);
        }
        const double cl2 = la2, cl1 = la1, cl0 = la0;
        bar_named(1, 128);  // V complete
        if (tim) { m1 = clock64(); tim[5] += m1 - m0; m0 = m1; }
        if (q + 1 < ny) {
          load(rowJ(up, q + 1));
          load_la(rowJ(up, q + 1));
        }
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        const bool res = J >= P.jstar;
        if (res && !ores) {
          mbar_wait(&resFullB, ores_n & 1u);
          ores = true;
          ++ores_n;
        }
#pragma unroll 1
        for (int c = cbeg; c < cend; ++c) {
          const double* A;
          uint32_t slot = 0;
          if (res) {
            A = ringO + size_t(c) * kChunk;
          } else {
            slot = so % NO;
            if (tim) m0 = clock64();
            mbar_wait(&fullO[slot], (so / NO) & 1u);
            if (tim) { m1 = clock64(); tim[6] += m1 - m0; }
            A = ringO + size_t(slot) * kChunk;
          }
          if (tim) m0 = clock64();
          chunk_mma(A, V + c * 64 * kS, rt, acc);
          if (tim) { m1 = clock64(); tim[7] += m1 - m0; }
          if (!res) {
            arrive5(&freeO[slot]);
            ++so;
          }
        }
        if (res && (q + 1 == ny || rowJ(up, q + 1) < P.jstar)) {
          arrive5(&resFreeB);
          ores = false;
        }
        const uint32_t cb = gq & 1u;
        if (tim) m0 = clock64();
        if (gq >= 2) mbar_wait(&cfree[cb], ((gq >> 1) - 1) & 1u);
        if (tim) { m1 = clock64(); tim[8] += m1 - m0; }
        double c0 = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
        double c1 = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
        if (lacoef) {
          c0 -= al[0] * cl2 - be[0] * cl1 + ga[0] * cl0;
          c1 -= al[1] * cl2 - be[1] * cl1 + ga[1] * cl0;
        }
        Cb[cb * 256 + (rt * 32 + lane) * 2] = c0;
        Cb[cb * 256 + (rt * 32 + lane) * 2 + 1] = c1;
        arrive5(&cready[cb]);
      }
      if (tim) m0 = clock64();
      cl_arrive();
      cl_wait();  // the other CTAs' rows of this sweep are visible
      if (tim) tim[9] += clock64() - m0;
    }
  } else {
    // ------------------------------------------------------------ producers
    const bool onc = warp == 8;
    const int nslot = onc ? NC : NO;
    uint64_t* fullb = onc ? fullC : fullO;
    uint64_t* freeb = onc ? freeC : freeO;
    uint64_t* rfull = onc ? &resFullA : &resFullB;
    uint64_t* rfree = onc ? &resFreeA : &resFreeB;
    double* ring = onc ? ringC : ringO;
    const uint32_t opbytes = uint32_t((onc ? CC : 1) * kChunk * 8);
    uint32_t cnt = 0, nres = 0;
    bool inres = false;
    for (int k = 0; k < nsweeps; ++k) {
      const bool up = k & 1;
      if (lane == 0) {
        const double* M = onc ? (up ? P.OnU : P.OnL) : (up ? P.OffU : P.OffL);
        int cbeg = 0, cend = NCH;
        if (!onc) tri_range(up, r, NCH, cbeg, cend);
        inres = false;  // a sweep's resident operators are its own (G/Li vs H/Ui)
        for (int q = onc ? 1 : 0; q < ny; ++q) {
          const int J = rowJ(up, q);
          const bool res = J >= P.jstar;
          if (res && !inres) {
            // every streamed copy consumed, the previous resident phase over
            for (int j = 1; j <= nslot; ++j)
              if (cnt >= uint32_t(j)) {
                const uint32_t n = cnt - j;
                mbar_wait(&freeb[n % nslot], (n / nslot) & 1u);
              }
            if (nres > 0) mbar_wait(rfree, (nres - 1) & 1u);
            const double* src = M + size_t(P.jstar) * mat + size_t(r) * NCH * kChunk + size_t(cbeg) * kChunk;
            const uint32_t bytes = uint32_t((cend - cbeg) * kChunk * 8);
            expect_tx5(rfull, bytes);
            g2s5(ring + size_t(cbeg) * kChunk, src, bytes, rfull);
            inres = true;
            ++nres;
          }
          if (!res && inres) {
            mbar_wait(rfree, (nres - 1) & 1u);
            inres = false;
          }
          if (res) continue;
          const double* src = M + size_t(J) * mat + size_t(r) * NCH * kChunk;
          const int nops = onc ? NOP : cend - cbeg;
          for (int i = 0; i < nops; ++i, ++cnt) {
            // on-chain: the chain's rotated order, CC chunks per copy
            const int c0 = onc ? (((r >> 1) / CC + i) % NOP) * CC : cbeg + i;
            const uint32_t slot = cnt % nslot;
            if (cnt >= uint32_t(nslot)) mbar_wait(&freeb[slot], ((cnt / nslot) - 1) & 1u);
            expect_tx5(&fullb[slot], opbytes);
            g2s5(ring + size_t(slot) * (opbytes / 8), src + size_t(c0) * kChunk, opbytes, &fullb[slot]);
          }
        }
      }
      __syncwarp();
      if (k > 0) cl_wait();
      cl_arrive();
    }
    cl_wait();
  }
}

// dst[J][r][c][ks][rt][lane] = scale * src[J][a][k] (zero padded), J < nJ
__global__ void v5_pack_kernel(const double* __restrict__ src, int nx, int kN, int nJ, double scale,
                               double* __restrict__ dst) {
  const int64_t mat = int64_t(kN) * kN;
  const int nch = kN / 64;
  const int64_t total = mat * nJ;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t J = e / mat;
    const int f = int(e - J * mat);
    const int ln = f & 31, rt = (f >> 5) & 3, ks = (f >> 7) & 15, rest = f >> 11;
    const int c = rest % nch, r = rest / nch;
    const int a = 32 * r + 8 * rt + (ln >> 2), k = 64 * c + 4 * ks + (ln & 3);
    dst[e] = (a < nx && k < nx) ? scale * src[J * int64_t(nx) * nx + int64_t(a) * nx + k] : 0.0;
  }
}

// LA[J][.][a] = (Li_J a2)[a], (Li_J a1)[a], (Li_J 1)[a] from the row-major Li
__global__ void v5_la_kernel(const double* __restrict__ Li, const double* __restrict__ a1,
                             const double* __restrict__ a2, int nx, int kN, double* __restrict__ LA) {
  const int J = blockIdx.x;
  const double* M = Li + size_t(J) * nx * nx;
  for (int a = threadIdx.x; a < kN; a += blockDim.x) {
    double s2 = 0.0, s1 = 0.0, s0 = 0.0;
    if (a < nx)
      for (int b = 0; b <= a; ++b) {
        const double m = M[size_t(a) * nx + b];
        s2 = fma(m, a2[size_t(J) * nx + b], s2);
        s1 = fma(m, a1[size_t(J) * nx + b], s1);
        s0 += m;
      }
    LA[(size_t(J) * 3 + 0) * kN + a] = s2;
    LA[(size_t(J) * 3 + 1) * kN + a] = s1;
    LA[(size_t(J) * 3 + 2) * kN + a] = s0;
  }
}

// dev[2J + m] = max |M_J - M_{ny-1}|, mag[2J + m] = max |M_J|, M = Li (m = 0), Ui (m = 1)
__global__ void v5_conv_kernel(const double* __restrict__ Li, const double* __restrict__ Ui, int nx, int ny,
                               double* __restrict__ dev, double* __restrict__ mag) {
  __shared__ double sd[2][256], sm_[2][256];
  const int J = blockIdx.x;
  const size_t nn = size_t(nx) * nx;
  double d[2] = {0.0, 0.0}, g[2] = {0.0, 0.0};
  for (size_t e = threadIdx.x; e < nn; e += blockDim.x) {
    const double a0 = Li[size_t(J) * nn + e], b0 = Li[size_t(ny - 1) * nn + e];
    const double a1 = Ui[size_t(J) * nn + e], b1 = Ui[size_t(ny - 1) * nn + e];
    d[0] = fmax(d[0], fabs(a0 - b0));
    d[1] = fmax(d[1], fabs(a1 - b1));
    g[0] = fmax(g[0], fabs(a0));
    g[1] = fmax(g[1], fabs(a1));
  }
  for (int m = 0; m < 2; ++m) {
    sd[m][threadIdx.x] = d[m];
    sm_[m][threadIdx.x] = g[m];
  }
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w)
      for (int m = 0; m < 2; ++m) {
        sd[m][threadIdx.x] = fmax(sd[m][threadIdx.x], sd[m][threadIdx.x + w]);
        sm_[m][threadIdx.x] = fmax(sm_[m][threadIdx.x], sm_[m][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 2) {
    dev[2 * J + threadIdx.x] = sd[threadIdx.x][0];
    mag[2 * J + threadIdx.x] = sm_[threadIdx.x][0];
  }
}

template <int kN>
void v5_launch(Ctx* c, const V5Params& P, int nsets) {
  using Cf = V5Cfg<kN>;
  static bool attr_done = false;
  if (!attr_done) {
    KKT_CUDA(cudaFuncSetAttribute(v5_kernel<kN>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cf::smem)));
    if (Cf::CL > 8) KKT_CUDA(cudaFuncSetAttribute(v5_kernel<kN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nsets * Cf::CL);
  cfg.blockDim = dim3(kThr5);
  cfg.dynamicSmemBytes = Cf::smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cf::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  V5Params p = P;
  void* args[] = {&p};
  KKT_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(&v5_kernel<kN>), args));
  c->launches++;
}

}  // namespace

bool v5_supported(const Ctx* c) {
  static const bool off = std::getenv("KKT_SWEEP_V5_OFF") != nullptr;  // testing: sweep_fast.cu chains
  return !off && c->mode == KKT_MODE_FAST && c->nx > 128 && c->nx <= 511 && c->ny >= 2 && c->Li.p && c->Ui.p;
}

void build_v5(Ctx* c) {
  const int nx = c->nx, ny = c->ny;
  const int kN = nx <= 255 ? 256 : 512;
  const size_t mat = size_t(kN) * kN, nn = size_t(nx) * nx;
  c->v5_kn = kN;
  c->v5_ops.alloc(4 * size_t(ny) * mat);
  double* OnL = c->v5_ops.p;
  double* OffL = OnL + ny * mat;
  double* OnU = OffL + ny * mat;
  double* OffU = OnU + ny * mat;
  const int pg = kSmCount * 8;
  KKT_LAUNCH(c, v5_pack_kernel, pg, 256, 0, c->Li.p, nx, kN, ny, 1.0, OffL);
  KKT_LAUNCH(c, v5_pack_kernel, pg, 256, 0, c->Ui.p, nx, kN, ny, 1.0, OffU);
  KKT_CUDA(cudaMemsetAsync(OnL, 0, sizeof(double) * mat, c->stream));                          // G_0: unused
  KKT_CUDA(cudaMemsetAsync(OnU + size_t(ny - 1) * mat, 0, sizeof(double) * mat, c->stream));  // H_{ny-1}
  const int Jb = std::min(ny - 1, 64);
  DBuf<double> T(size_t(Jb) * nn);
  for (int J0 = 1; J0 < ny; J0 += Jb) {  // G_J = cy Li_J Ui_{J-1}
    const int nb = std::min(Jb, ny - J0);
    GemmArgs g{c->Li.p + J0 * nn, c->Ui.p + (J0 - 1) * nn, T.p, nx, nx, nx,
               int64_t(nn), int64_t(nn), int64_t(nn), nx, nx, nx};
    gemm_f64(c, g, nb);
    KKT_LAUNCH(c, v5_pack_kernel, pg, 256, 0, T.p, nx, kN, nb, c->cy, OnL + J0 * mat);
  }
  for (int J0 = 0; J0 < ny - 1; J0 += Jb) {  // H_J = cy Ui_J Li_J
    const int nb = std::min(Jb, ny - 1 - J0);
    GemmArgs g{c->Ui.p + J0 * nn, c->Li.p + J0 * nn, T.p, nx, nx, nx,
               int64_t(nn), int64_t(nn), int64_t(nn), nx, nx, nx};
    gemm_f64(c, g, nb);
    KKT_LAUNCH(c, v5_pack_kernel, pg, 256, 0, T.p, nx, kN, nb, c->cy, OnU + J0 * mat);
  }
  // The block recursion D_J = T - cy^2 D_{J-1}^{-1} converges geometrically
  // (factor_block.cu), so from some row on the factors equal the last row's
  // to rounding: rows J >= jstar then use row jstar's operators, kept
  // resident in shared memory (kN = 256).  jstar is the first row from which
  // Li and Ui (and so G, H) stay within tol * max|M| of the last row's; a
  // rounding-level substitution like the rest of FAST.  No such row: ny.
  c->v5_jstar = ny;
  const bool res_ok = kN == 256;
  static const char* jt = std::getenv("KKT_V5_JTOL");
  const double tol = jt ? std::atof(jt) : 1e-15;
  if (res_ok && tol > 0.0 && ny >= 3) {
    DBuf<double> dev(2 * size_t(ny)), mag(2 * size_t(ny));
    KKT_LAUNCH(c, v5_conv_kernel, ny, 256, 0, c->Li.p, c->Ui.p, nx, ny, dev.p, mag.p);
    std::vector<double> hd(2 * ny), hm(2 * ny);
    KKT_CUDA(cudaMemcpyAsync(hd.data(), dev.p, sizeof(double) * 2 * ny, cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaMemcpyAsync(hm.data(), mag.p, sizeof(double) * 2 * ny, cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    int first = ny - 1;  // rows first .. ny-1 all within tol
    while (first > 0 && hd[2 * (first - 1)] <= tol * hm[2 * (ny - 1)] &&
           hd[2 * (first - 1) + 1] <= tol * hm[2 * (ny - 1) + 1])
      --first;
    const int js = first + 1;  // G_J needs Li_J and Ui_{J-1}
    if (js <= ny - 2) c->v5_jstar = js;
    if (std::getenv("KKT_V5_TIM")) {
      for (int J = 0; J < ny; J += std::max(1, ny / 24))
        std::fprintf(stderr, "v5 conv J=%4d  dLi %.3e  dUi %.3e\n", J, hd[2 * J] / hm[2 * (ny - 1)],
                     hd[2 * J + 1] / hm[2 * (ny - 1) + 1]);
      std::fprintf(stderr, "v5 jstar %d of ny %d (tol %.1e)\n", c->v5_jstar, ny, tol);
    }
  }
  KKT_CUDA(cudaStreamSynchronize(c->stream));  // T is freed on return
}

void v5_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms) {
  const int kN = c->v5_kn, ny = c->ny;
  const size_t mat = size_t(kN) * kN;
  const int nsets = (nchains + kS - 1) / kS;
  const size_t need = size_t(nsets) * ny * kN * kS;
  if (c->v5_y.n < need) {
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    c->v5_y.alloc(need);
  }
  V5Params P;
  P.OnL = c->v5_ops.p;
  P.OffL = P.OnL + ny * mat;
  P.OnU = P.OffL + ny * mat;
  P.OffU = P.OnU + ny * mat;
  P.Y = c->v5_y.p;
  if (coarse_terms && !c->v5_la.p) {
    c->v5_la.alloc(size_t(ny) * 3 * kN);
    KKT_LAUNCH(c, v5_la_kernel, ny, 256, 0, c->Li.p, c->a1.p, c->a2.p, c->nx, kN, c->v5_la.p);
  }
  P.LA = c->v5_la.p;
  P.gam = c->gam.p;
  P.inv_ms = 1.0 / c->ms;
  P.nx = c->nx;
  P.ny = ny;
  P.nchains = nchains;
  P.nsteps = nsteps;
  P.coarse = coarse_terms ? 1 : 0;
  P.jobs = jobs_dev;
  P.jstar = c->v5_jstar;
  static const bool dbg = std::getenv("KKT_V5_TIM") != nullptr;
  DBuf<long long> tim;
  P.tim = nullptr;
  if (dbg) {
    tim.alloc(size_t(nsets) * (kN / kRowsV5) * 16);
    KKT_CUDA(cudaMemsetAsync(tim.p, 0, sizeof(long long) * tim.n, c->stream));
    P.tim = tim.p;
  }
  c->tbegin(3);
  if (kN == 256)
    v5_launch<256>(c, P, nsets);
  else
    v5_launch<512>(c, P, nsets);
  c->tend(3);
  if (dbg) {
    std::vector<long long> h(tim.n);
    KKT_CUDA(cudaMemcpyAsync(h.data(), tim.p, sizeof(long long) * tim.n, cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    const int ncta = int(tim.n / 16);
    const long long rows = (long long)ny * 2 * nsteps;
    long long t0 = h[15];
    for (int b = 0; b < ncta; ++b) t0 = std::min(t0, h[size_t(b) * 16 + 15]);
    for (int b = 0; b < ncta; ++b) {
      const long long* x = &h[size_t(b) * 16];
      std::fprintf(stderr,
                   "v5 cta %3d start %8lld end %10lld | chain/row: xbar %5lld ring %5lld mma %5lld cready %5lld send %5lld"
                   " | off/row: V %5lld ring %5lld mma %5lld cfree %5lld | off sweepbar/sweep %lld\n",
                   b, x[15] - t0, x[14] - t0, x[0] / rows, x[1] / rows, x[2] / rows, x[3] / rows, x[4] / rows,
                   x[5] / rows, x[6] / rows, x[7] / rows, x[8] / rows, x[9] / (2 * nsteps));
    }
    int ncl = 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nsets * (kN / kRowsV5));
    cfg.blockDim = dim3(kThr5);
    cfg.dynamicSmemBytes = kN == 256 ? V5Cfg<256>::smem : V5Cfg<512>::smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim = {unsigned(kN / kRowsV5), 1, 1};
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = kN == 256 ? cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(&v5_kernel<256>), &cfg)
                              : cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(&v5_kernel<512>), &cfg);
    std::fprintf(stderr, "v5: kN %d sets %d max active clusters %d (%s)\n", kN, nsets, ncl, cudaGetErrorString(e));
  }
}

}  // namespace kkt
