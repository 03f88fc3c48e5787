// sweep_v6.cu — FAST RASQ sweeps for the large grids (128 < nx <= 1023:
// BASELINE configs 2, 3 and 4), device-wide block substitution; block size
// KN = 256 (nx <= 255), 512 (nx <= 511) or 1024.
//
// Same block recursion as sweep v5 (the reference's LU solve
// BandedLU::solve_in_place, linalg.cpp:127-145, on the block factors of
// factor_block.cu, with the two dependent triangular products of a block step
// pre-multiplied):
//     L:  y_J = Li_J b_J + G_J y_{J-1},   G_J = cy Li_J Ui_{J-1}
//     U:  x_J = Ui_J y_J + H_J x_{J+1},   H_J = cy Ui_J Li_J
// At nx = 1023 a block row is 1024 x 1024 doubles (8 MB): one cluster cannot
// hold a row slice next to its vectors (v5's layout); at nx = 511 v5's 16-CTA
// clusters fit only 7 of 8 chain sets at once and wait on their triangle
// imbalance.  v6 spreads every block step over the whole device instead:
//   * off-chain terms first, for all J at once: c_J = Li_J b_J (d_J = Ui_J y_J)
//     is a batched triangular product with no dependency (v6_off2_kernel, or
//     v6_off_kernel at KN = 256), the triangle streamed once per spatial
//     solve for all local chains;
//   * then the dependent chain y_J = c_J + G_J y_{J-1} (v6_chain_kernel): a
//     co-resident grid of KN/16 row slices x chain groups; CTA (s, g) owns rows
//     16s..16s+15 for the 8 chains of group g, stages its slice of G_J (the
//     next row's during this row's barrier) and y_{J-1} by bulk copies,
//     multiplies them as fp64 DMMA (m8n8k4) tiles split over 8 warps along k,
//     and publishes y_J with a release counter per chain group (one
//     grid-wide barrier per block row).
// Block vectors are chain-interleaved, W[g][J][k][8] (KN rows, zero padded), so the DMMA B operand of a k-step is 256 contiguous bytes.
// Operators are packed in fragment order, [J][s][ks][mt][lane] =
// M[16s + 8mt + lane/4][4ks + lane%4], so each warp's A operand is 32
// consecutive doubles.  Chains, steps and the fused two-level residual follow
// fast_chain_kernel (sweep_fast.cu) exactly; only the operation order differs
// (FAST mode, rounding level).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sweep.cuh"
#include "sweep_tma.cuh"

namespace kkt {
namespace {
using tma::mbar_init;
using tma::mbar_wait;
using tma::tma_load;

// KN: padded block size, 1024 (511 < nx <= 1023) or 512 (255 < nx <= 511)
constexpr int kThr6 = 256;            // 8 warps
constexpr int kG = 8;                 // chains per group (the n of m8n8k4)
#define V6_DIMS                                                                          \
  constexpr int kSl = KN / 16; /* row slices per block row */                           \
  constexpr int kKS = KN / 4;  /* k-steps of a full row */                              \
  constexpr int kKW = kKS / 8; /* k-steps per warp (chain kernel) */                    \
  (void)kSl;                                                                             \
  (void)kKW;

__device__ __forceinline__ void dmma6(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr unsigned long long kLLEmpty = 0xFFFFFFFFFFFFFFFFull;  // handoff slot not yet written

struct V6Params {
  const double* Lp;  // packed Li_J
  const double* Up;  // packed Ui_J
  const double* Gp;  // packed G_J (J >= 1)
  const double* Hp;  // packed H_J (J <= ny-2)
  double* W0;        // [g][J][kN][8]: b, then y, then x
  double* W1;        // [g][J][kN][8]: c, then d
  const FastStep* jobs;
  int nsteps, t;
  int nx, ny, nchains, ngroups;
  const double* a1;
  const double* a2;
  const double* gam;
  double inv_ms;
  int coarse;
  unsigned* cnt;     // per chain group: row-completion counter (chain kernels)
  int g0;            // first chain group of this chain-kernel wave
  int jstar;         // block rows J >= jstar use row jstar's operators (ny: none)
  // k-row grouping of the chain: the ny block rows form ngr groups of k rows (L: from row 0 up,
  // U: from row ny-1 down); a group's rows all depend on the previous group's LAST row only,
  //   y_{g k + i} = c'_{g k + i} + Phi_{g k + i} y_{g k - 1},  Phi_{g k + i} = G_{g k + i} ... G_{g k},
  // with c' the zero-inflow chain inside the group (v6_inner_kernel), so one row handoff serves
  // k rows.  k == 1: Phi = G, the plain recurrence.
  const double* Phi;  // packed propagators of the L groups (k == 1: Gp)
  const double* Psi;  // packed propagators of the U groups (k == 1: Hp)
  int k, ngr;
  int nind;           // L: groups [0, nind) have their own Phi rows, the rest share one converged set
  int gconv;          // U: groups [0, gconv) (from the top) share the converged set, the rest have their own
  int pass;           // v6_inner_kernel: row i of every group
  // Low-latency row handoff (kLL): the last row of a group is published as bare 8-byte values, one
  // per (row, chain), in a slot per (chain group, group step) that the host pre-fills with a
  // sentinel bit pattern (all ones: a NaN no arithmetic produces) before every chain launch.
  // Consumers spin on the slots of exactly the values they need until none is the sentinel, so a
  // handoff is one L2 write and one L2 read: no release / acquire counter, no separate copy of y.
  // Only 64-bit store atomicity is assumed.  Slots are not reused inside a launch.
  unsigned long long* ll;
  size_t nll;               // slots
  int nopoll;               // KKT_V6_NOPOLL (timing experiment only: WRONG results): take the slots as they are
  // Numerical band of the propagators: per (packed operator row, 16-row slice) the window of
  // k-steps {first, per-warp count} outside which every entry is below KKT_V6_BTOL (1e-17) times
  // the operator's largest entry.  The inverted blocks decay exponentially away from the diagonal
  // (half-bandwidth ~144 of 511 at config 2); the chain multiplies only the window.
  const int2* bandPhi;
  const int2* bandPsi;
  // raw {first k-step, one past the last} per (operator row, slice) of Li, Ui, G, H: the off-chain
  // triangles and the in-group products skip the k-steps outside (null: none skipped)
  const int2* rawL;
  const int2* rawU;
  const int2* rawG;
  const int2* rawH;
  long long* tim;    // KKT_V6_TIM: per-row clock64 phase sums of CTA 0 (6 per direction)
  // Two-sided (twisted) elimination, ny odd (build_twist_middle, factor_block.cu): block rows
  // 0..M-1 (downward) and nyA-1..M+1 (upward, the mirror image: the same operators) are two
  // half-length "virtual" chains per real chain, M = (nyA-1)/2 rows each; ny above is then M and
  // ngroups counts virtual chain groups: gv = g + h*nreal is half h (0: top, 1: bottom) of real
  // group g, its row j is block row j (top) or nyA-1-j (bottom).  The two eliminations meet in
  // row M (v6_mid_kernel), and the back substitution runs outward from it.  A chain CTA serves
  // both halves of its group in turn, so each half's handoff latency hides behind the other's
  // product and the dependent chain is half as long.
  int twist, nyA, nreal;
  int wmax;          // v6_chainw_kernel: the widest window's k-steps per warp (shared-memory extent)
  int spin_ns;       // KKT_V6_SPIN_NS: pause between failed poll rounds (0: none)
  int stagger;       // v6_chainw_kernel: cycles by which the upper half of the chain groups starts late
  // Inverse-block ("Thomas") form of the twisted elimination (k == 1, slot handoff): with
  // H_J = cy D_J^{-1} the forward elimination is z_J = H_J (b_J/cy + z_{J-1}) and the back
  // substitution x_J = z_J + H_J x_{J+1} = H_J (y_J + x_{J+1}), y_J = b_J/cy + z_{J-1}.  Both map
  // onto the chain recurrences with H as the only operator set and NO off-chain products:
  //   L chain:  y_0 = c_0,  y_J = c_J + H_{J-1} y_{J-1},  c = b/cy (written by v6_form_b_kernel)
  //   middle:   x_M = Dm^{-1} b_M + E2 (y_{M-1} + y'_{M+1}),  E2 = cy Dm^{-1} H_{M-1}
  //   U chain:  X_{M-1} = y_{M-1} + x_M,  X_J = y_J + H_{J+1} X_{J+1};  the product is x_{J+1}
  //   last:     x_0 = H_0 X_0  (v6_mid_kernel, mode 2)
  int thomas;
  double inv_cy;
  int nohold;        // KKT_V6_NOHOLD (testing): fetch the operator window for every row, also an unchanged one
  double* Wm;        // [2][nreal][kN][8]: b_M, then x_M
  const double* Dm;  // packed Dm^{-1}
  const double* Em;  // packed cy Dm^{-1} Ui_{M-1}
};

// Operator row of block row J, and its load: rows past jstar share one
// operator set, which stays in L2 (default caching); the others stream
// (evict-first).
__device__ __forceinline__ int oprow(int J, int jstar) { return J < jstar ? J : jstar; }
__device__ __forceinline__ double ldop(const double* p, bool res) { return res ? __ldg(p) : __ldcs(p); }

template <int KN>
__device__ __forceinline__ size_t widx(int g, int J, int ny) { return (size_t(g) * ny + J) * KN * kG; }

// b = in*scale + add - (Shat y_c)_node / ms, chain-interleaved (fast_chain_kernel's b).
// One CTA per (virtual chain group, block row, 256-row chunk): the 8 chains' plane rows are read
// coalesced (consecutive threads = consecutive grid points of one chain) into a padded shared
// tile and written out chain-interleaved, again coalesced.  (One thread per output element read
// the 8 planes 32 bytes at a time: 177 us per step at config 2 against ~70 us of traffic.)
constexpr int kFbChunk = 256;
template <int KN>
__global__ void __launch_bounds__(kFbChunk) v6_form_b_kernel(V6Params P) {
  __shared__ double tile[kFbChunk][kG + 1];
  constexpr int kChunks = KN / kFbChunk;
  const int chunk = blockIdx.x % kChunks;
  const int rb = blockIdx.x / kChunks;             // row block: (gv, j), then the middle rows (g)
  const int nrb = P.ngroups * P.ny;
  int J, g;
  double* dst;
  if (rb < nrb) {
    const int j = rb % P.ny, gv = rb / P.ny;
    const int h = gv >= P.nreal ? 1 : 0;
    g = gv - h * P.nreal;
    J = h ? P.nyA - 1 - j : j;
    dst = (P.thomas ? P.W1 : P.W0) + size_t(rb) * KN * kG;  // Thomas form: c = b / cy, straight to the chain
  } else {
    g = rb - nrb;
    J = P.ny;  // the middle row of the twisted elimination
    dst = P.Wm + size_t(g) * KN * kG;
  }
  const int k = chunk * kFbChunk + threadIdx.x;
  const int p = J * P.nx + k;
#pragma unroll
  for (int c = 0; c < kG; ++c) {
    const int ch = g * kG + c;
    double v = 0.0;
    if (k < P.nx && ch < P.nchains) {
      const FastStep st = P.jobs[size_t(ch) * P.nsteps + P.t];
      if (st.in) {
        v = st.in[p] * st.scale;
        if (st.add) v += st.add[p];
        if (P.coarse && st.node > 0) {
          const double gn = P.gam[st.node], gm = P.gam[st.node - 1], gp = P.gam[st.node + 1];
          double sh = gn * P.a2[p] - gp * P.a1[p];
          if (st.node != 1) sh += gn - gm * P.a1[p];
          v -= sh * P.inv_ms;
        }
      }
    }
    tile[threadIdx.x][c] = (P.thomas && rb < nrb) ? v * P.inv_cy : v;
  }
  __syncthreads();
  double* o = dst + size_t(chunk) * kFbChunk * kG;
#pragma unroll
  for (int r = 0; r < kG; ++r) {
    const int e = threadIdx.x + kFbChunk * r;
    o[e] = tile[e >> 3][e & 7];
  }
}

// Partials of 8 warps -> 16 x 8 slice (fixed order): thread t < 128 owns
// D[m][n], m = 8mt + lane/4, n = 2(lane%4) + e with t = (mt*32 + lane)*2 + e.
__device__ __forceinline__ double reduce8(const double* red, int t) {
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w * 128 + t];
  return s;
}
__device__ __forceinline__ void slice_coords(int t, int& m, int& n) {
  const int e = t & 1, q = t >> 1, mt = q >> 5, lane = q & 31;
  m = 8 * mt + (lane >> 2);
  n = 2 * (lane & 3) + e;
}

// k-step range of slice s of a triangle (lower: Li, upper: Ui), cut to the operator's numerical band
__device__ __forceinline__ void tri_range(bool upper, int s, int kKS, const int2* raw, int row, int kSl, int& ks0, int& ks1) {
  ks0 = upper ? 4 * s : 0;
  ks1 = upper ? kKS : 4 * s + 4;
  if (raw) {
    const int2 b = raw[size_t(row) * kSl + s];
    ks0 = max(ks0, b.x);
    ks1 = min(ks1, b.y);
  }
}
// the same with the table entry fetched one slice ahead (b = this slice's entry)
__device__ __forceinline__ void tri_range_b(bool upper, int s, int kKS, bool have, int2 b, int& ks0, int& ks1) {
  ks0 = upper ? 4 * s : 0;
  ks1 = upper ? kKS : 4 * s + 4;
  if (have) {
    ks0 = max(ks0, b.x);
    ks1 = min(ks1, b.y);
  }
}

// Batched triangular products for every block row: Out[g][J] = T_J In[g][J]
// over the nonzero k-steps of the triangle (lower: Li, upper: Ui).  One CTA
// per block row J; chain groups in pairs, their block vectors In[g][J] staged
// in shared memory (2 x 64 KB); each warp owns whole row slices (zig-zag
// pairs s, 15-s of every 16, so the triangle work is balanced) and streams
// them from HBM in fragment order, the next 16 k-steps in flight while the
// current 16 are multiplied.  A warp accumulates a slice over all its k-steps
// itself, so no cross-warp reduction is needed.
constexpr int kOffChunk = 16;
template <int KN>
constexpr size_t off_smem() { return sizeof(double) * 2 * KN * kG; }

template <int KN, bool kUpper>
__global__ void __launch_bounds__(kThr6, 1) v6_off_kernel(V6Params P) {
  V6_DIMS
  extern __shared__ double Bs[];  // [2][kN][8]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bo = (lane & 3) * kG + (lane >> 2);  // B fragment offset within a k-step
  for (int J = blockIdx.x; J < P.ny; J += gridDim.x) {
    for (int gp = 0; gp < P.ngroups; gp += 2) {
      __syncthreads();  // the previous pair's readers are done with Bs
      for (int i = threadIdx.x; i < KN * kG; i += kThr6) {  // double2 units over both groups
        const int gi = i / (KN * kG / 2), r = i - gi * (KN * kG / 2);
        double2 v = make_double2(0.0, 0.0);
        if (gp + gi < P.ngroups) v = __ldcg(reinterpret_cast<const double2*>(P.W0 + widx<KN>(gp + gi, J, P.ny)) + r);
        reinterpret_cast<double2*>(Bs)[i] = v;
      }
      __syncthreads();
      for (int i = 0; i < kSl / 8; ++i) {
        const int s = (i >> 1) * 16 + ((i & 1) ? 15 - warp : warp);
        int ks0, ks1;
        tri_range(kUpper, s, kKS, kUpper ? P.rawU : P.rawL, oprow(J, P.jstar), kSl, ks0, ks1);
        const bool res = J >= P.jstar;
        const double* A = (kUpper ? P.Up : P.Lp) + (size_t(oprow(J, P.jstar)) * kSl + s) * kKS * 64 + lane;
        double d[2][2][2] = {};
        double ac[kOffChunk][2], an[kOffChunk][2];
#pragma unroll
        for (int u = 0; u < kOffChunk; ++u) {
          const bool ok = ks0 + u < ks1;
          ac[u][0] = ok ? ldop(A + size_t(ks0 + u) * 64, res) : 0.0;
          ac[u][1] = ok ? ldop(A + size_t(ks0 + u) * 64 + 32, res) : 0.0;
        }
        for (int ks = ks0; ks < ks1; ks += kOffChunk) {
#pragma unroll
          for (int u = 0; u < kOffChunk; ++u) {
            const bool ok = ks + kOffChunk + u < ks1;
            an[u][0] = ok ? ldop(A + size_t(ks + kOffChunk + u) * 64, res) : 0.0;
            an[u][1] = ok ? ldop(A + size_t(ks + kOffChunk + u) * 64 + 32, res) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kOffChunk; ++u) {
            if (ks + u < ks1) {
              const double b0 = Bs[(4 * (ks + u)) * kG + bo];
              const double b1 = Bs[KN * kG + (4 * (ks + u)) * kG + bo];
              dmma6(d[0][0][0], d[0][0][1], ac[u][0], b0);
              dmma6(d[0][1][0], d[0][1][1], ac[u][1], b0);
              dmma6(d[1][0][0], d[1][0][1], ac[u][0], b1);
              dmma6(d[1][1][0], d[1][1][1], ac[u][1], b1);
            }
          }
#pragma unroll
          for (int u = 0; u < kOffChunk; ++u) {
            ac[u][0] = an[u][0];
            ac[u][1] = an[u][1];
          }
        }
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (gp + g >= P.ngroups) break;
          double* O = P.W1 + widx<KN>(gp + g, J, P.ny) + size_t(16 * s + (lane >> 2)) * kG + 2 * (lane & 3);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
            *reinterpret_cast<double2*>(O + mt * 8 * kG) = make_double2(d[g][mt][0], d[g][mt][1]);
        }
      }
    }
  }
}

// TMA-streamed batched triangular products (default for KN >= 512; KKT_V6_OFF=1
// selects v6_off_kernel above; measured P^-1: config 2 181.5 -> 176.3 ms,
// config-4 slab 174.9 -> 165.9 ms; at KN = 256 the plain kernel stays, 308 vs 312 ms).  The plain loads of v6_off_kernel are bounded by the
// SM's outstanding misses (~3.2 TB/s over the device); here one producer warp
// streams each slice's nonzero k-steps in 32 KB bulk copies through a 2-slot
// ring, and 8 consumer warps split every chunk along k, accumulate the slice
// in registers and reduce it through shared memory (double-buffered by slice
// parity, one named barrier per slice) in a fixed order.
constexpr int kOffRing = 2;      // ring slots
constexpr int kOffThr = 288;     // 8 consumer warps + 1 producer warp
// NG chain groups share one pass over the triangle (their block vectors staged side by side), so
// 8 chain groups (config 2) stream it twice instead of four times; the ring chunk shrinks to keep
// the CTA under the shared-memory limit.
template <int NG>
constexpr int off_ck() { return NG == 2 ? 64 : 32; }  // k-steps per chunk (32 KB / 16 KB)
template <int KN, int NG>
constexpr size_t off2_smem() {
  return sizeof(double) * (NG * KN * kG + kOffRing * off_ck<NG>() * 64 + 2 * 8 * NG * 128) + 8 * sizeof(uint64_t);
}

template <int KN, bool kUpper, int NG>
__global__ void __launch_bounds__(kOffThr, 1) v6_off2_kernel(V6Params P) {
  V6_DIMS
  constexpr int CK = off_ck<NG>();
  extern __shared__ __align__(128) double so[];
  double* Bs = so;                               // [NG][KN][8]
  double* ring = Bs + NG * KN * kG;              // [slot][CK][64]
  double* red = ring + kOffRing * CK * 64;       // [slice parity 2][warp 8][NG * 128]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * 8 * NG * 128);
  uint64_t* empty = full + kOffRing;
  uint64_t* barB = empty + kOffRing;
  uint64_t* bfree = barB + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kOffRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    mbar_init(barB, 1);
    mbar_init(bfree, 8);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const double* T = kUpper ? P.Up : P.Lp;
  if (warp == 8) {  // producer
    if (lane == 0) {
      int it = 0, item = 0;
      // items (block row, pass of NG chain groups) dealt round-robin: the CTAs that work on one row's
      // passes run side by side (its triangle is fetched from HBM once), and no CTA gets a whole row more
      const int npass = (P.ngroups + NG - 1) / NG;
      for (int gitem = blockIdx.x; gitem < P.ny * npass; gitem += gridDim.x, ++item) {
        const int J = gitem / npass, gp = (gitem % npass) * NG;
        const double* TJ = T + size_t(oprow(J, P.jstar)) * kSl * kKS * 64;
        {
          if (item > 0) mbar_wait(bfree, uint32_t(item - 1) & 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tma::smem_u32(barB)),
                       "r"(uint32_t(sizeof(double) * NG * KN * kG))
                       : "memory");
          const uint32_t vb = uint32_t(sizeof(double) * KN * kG);
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            const int gs = gp + g < P.ngroups ? gp + g : gp;  // a missing group reads gp (its outputs are not written)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             tma::smem_u32(Bs + size_t(g) * KN * kG)), "l"(P.W0 + widx<KN>(gs, J, P.ny)), "r"(vb),
                         "r"(tma::smem_u32(barB))
                         : "memory");
          }
          const int2* rawrow = (kUpper ? P.rawU : P.rawL) ? (kUpper ? P.rawU : P.rawL) + size_t(oprow(J, P.jstar)) * kSl : nullptr;
          int2 rb = rawrow ? rawrow[0] : make_int2(0, 0);
          for (int s = 0; s < kSl; ++s) {
            int ks0, ks1;
            const int2 cur = rb;
            if (rawrow && s + 1 < kSl) rb = rawrow[s + 1];  // one slice ahead: off the critical path
            tri_range_b(kUpper, s, kKS, rawrow != nullptr, cur, ks0, ks1);
            for (int kb = ks0; kb < ks1; kb += CK, ++it) {
              const int slot = it % kOffRing, len = min(CK, ks1 - kb);
              if (it >= kOffRing) mbar_wait(&empty[slot], uint32_t(it / kOffRing - 1) & 1u);
              tma_load(ring + size_t(slot) * CK * 64, TJ + (size_t(s) * kKS + kb) * 64,
                       uint32_t(sizeof(double) * 64 * len), &full[slot]);
            }
          }
        }
      }
    }
    return;
  }
  const int bo = (lane & 3) * kG + (lane >> 2);
  int it = 0, item = 0, sl = 0;
  const int npass = (P.ngroups + NG - 1) / NG;
  for (int gitem = blockIdx.x; gitem < P.ny * npass; gitem += gridDim.x, ++item) {
    const int J = gitem / npass, gp = (gitem % npass) * NG;
    {
      mbar_wait(barB, uint32_t(item) & 1u);
      const int2* rawrow = (kUpper ? P.rawU : P.rawL) ? (kUpper ? P.rawU : P.rawL) + size_t(oprow(J, P.jstar)) * kSl : nullptr;
      int2 rb = rawrow ? rawrow[0] : make_int2(0, 0);
      for (int s = 0; s < kSl; ++s, ++sl) {
        int ks0, ks1;
        const int2 cur = rb;
        if (rawrow && s + 1 < kSl) rb = rawrow[s + 1];
        tri_range_b(kUpper, s, kKS, rawrow != nullptr, cur, ks0, ks1);
        double d[NG][2][2] = {};
        for (int kb = ks0; kb < ks1; kb += CK, ++it) {
          const int slot = it % kOffRing, len = min(CK, ks1 - kb);
          mbar_wait(&full[slot], uint32_t(it / kOffRing) & 1u);
          const double* R = ring + size_t(slot) * CK * 64 + lane;
#pragma unroll
          for (int q = 0; q < CK / 8; ++q) {
            const int u = warp + 8 * q;
            if (u < len) {
              const double a0 = R[u * 64], a1 = R[u * 64 + 32];
#pragma unroll
              for (int g = 0; g < NG; ++g) {
                const double bg = Bs[size_t(g) * KN * kG + (4 * (kb + u)) * kG + bo];
                dmma6(d[g][0][0], d[g][0][1], a0, bg);
                dmma6(d[g][1][0], d[g][1][1], a1, bg);
              }
            }
          }
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma::smem_u32(&empty[slot])) : "memory");
        }
        double* rw = red + size_t(sl & 1) * 8 * NG * 128 + warp * NG * 128;
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) rw[g * 128 + (mt * 32 + lane) * 2 + e] = d[g][mt][e];
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
#pragma unroll
        for (int h = 0; h < NG / 2; ++h) {
          const int t = threadIdx.x, g = 2 * h + (t >> 7), r = t & 127;
          int m, n;
          slice_coords(r, m, n);
          const double* rr = red + size_t(sl & 1) * 8 * NG * 128 + g * 128 + r;
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) v += rr[w * NG * 128];
          if (gp + g < P.ngroups) P.W1[widx<KN>(gp + g, J, P.ny) + size_t(16 * s + m) * kG + n] = v;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma::smem_u32(bfree)) : "memory");
    }
  }
}

// Batched triangular products without a cross-warp reduction (the default for KN >= 512).
// v6_off2_kernel splits every chunk along k over its 8 warps and reduces each 16-row slice through
// shared memory behind a CTA barrier; once the triangles are cut to the operators' numerical band a
// slice has only ~34 k-steps (config 2), so that kernel spends more time in barriers and reductions
// than in DMMAs (40% of its DMMA-issue bound).  Here the slices are taken four at a time and warp w
// owns one 8-row tile of the quad (slice 4q + w/2, tile w%2) over the slice's WHOLE k-range, so each
// warp keeps its accumulators in registers from the first k-step to the store.  One producer lane
// streams the four slices' k-steps through four small rings (kOff3R slots of kOff3CK k-steps each);
// the two warps of a slice share a ring.  The block vectors of NG chain groups are staged once per
// (block row, pass) item by bulk copies, as in v6_off2_kernel.
constexpr int kOff3CK = 16;  // k-steps per ring slot (8 KB)
constexpr int kOff3R = 3;    // slots per ring
template <int KN, int NG>
constexpr size_t off3_smem() {
  return sizeof(double) * (size_t(NG) * KN * kG + size_t(4) * kOff3R * kOff3CK * 64) + (2 * 4 * kOff3R + 2) * sizeof(uint64_t);
}

template <int KN, bool kUpper, int NG>
__global__ void __launch_bounds__(kOffThr, 1) v6_off3_kernel(V6Params P) {
  V6_DIMS
  constexpr int CK = kOff3CK, R = kOff3R;
  extern __shared__ __align__(128) double so[];
  double* Bs = so;                           // [NG][KN][8]
  double* ring = Bs + size_t(NG) * KN * kG;  // [slice of the quad 4][slot R][CK][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + size_t(4) * R * CK * 64);  // [4][R]
  uint64_t* empty = full + 4 * R;                                               // [4][R]
  uint64_t* barB = empty + 4 * R;
  uint64_t* bfree = barB + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4 * R; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 2);
    }
    mbar_init(barB, 1);
    mbar_init(bfree, 8);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const double* T = kUpper ? P.Up : P.Lp;
  const int2* raw = kUpper ? P.rawU : P.rawL;
  const int npass = (P.ngroups + NG - 1) / NG;
  const int nitems = P.ny * npass;
  if (warp == 8) {  // producer
    if (lane == 0) {
      int itr[4] = {0, 0, 0, 0};
      int item = 0;
      for (int gitem = blockIdx.x; gitem < nitems; gitem += gridDim.x, ++item) {
        const int J = gitem / npass, gp = (gitem % npass) * NG;
        const int orow = oprow(J, P.jstar);
        const double* TJ = T + size_t(orow) * kSl * kKS * 64;
        if (item > 0) mbar_wait(bfree, uint32_t(item - 1) & 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tma::smem_u32(barB)),
                     "r"(uint32_t(sizeof(double) * NG * KN * kG))
                     : "memory");
        const uint32_t vb = uint32_t(sizeof(double) * KN * kG);
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const int gs = gp + g < P.ngroups ? gp + g : gp;  // a missing group reads gp (its outputs are not written)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                           tma::smem_u32(Bs + size_t(g) * KN * kG)), "l"(P.W0 + widx<KN>(gs, J, P.ny)), "r"(vb),
                       "r"(tma::smem_u32(barB))
                       : "memory");
        }
        for (int q = 0; q < kSl / 4; ++q) {
          int k0[4], k1[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) tri_range(kUpper, 4 * q + i, kKS, raw, orow, kSl, k0[i], k1[i]);
          bool any = true;
          while (any) {  // one chunk per slice in turn, so the four rings fill evenly
            any = false;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (k0[i] < k1[i]) {
                const int slot = itr[i] % R, len = min(CK, k1[i] - k0[i]);
                if (itr[i] >= R) mbar_wait(&empty[i * R + slot], uint32_t(itr[i] / R - 1) & 1u);
                tma_load(ring + (size_t(i) * R + slot) * CK * 64, TJ + (size_t(4 * q + i) * kKS + k0[i]) * 64,
                         uint32_t(sizeof(double) * 64 * len), &full[i * R + slot]);
                k0[i] += len;
                ++itr[i];
                any = true;
              }
            }
          }
        }
      }
    }
    return;
  }
  const int sl = warp >> 1, mt = warp & 1;
  const int bo = (lane & 3) * kG + (lane >> 2);
  int it = 0, item = 0;
  for (int gitem = blockIdx.x; gitem < nitems; gitem += gridDim.x, ++item) {
    const int J = gitem / npass, gp = (gitem % npass) * NG;
    const int orow = oprow(J, P.jstar);
    mbar_wait(barB, uint32_t(item) & 1u);
    for (int q = 0; q < kSl / 4; ++q) {
      const int s = 4 * q + sl;
      int ks0, ks1;
      tri_range(kUpper, s, kKS, raw, orow, kSl, ks0, ks1);
      double d[2][NG][2] = {};
      for (int kb = ks0; kb < ks1; kb += CK, ++it) {
        const int slot = it % R, len = min(CK, ks1 - kb);
        mbar_wait(&full[sl * R + slot], uint32_t(it / R) & 1u);
        const double* A = ring + (size_t(sl) * R + slot) * CK * 64 + mt * 32 + lane;
        const double* B = Bs + size_t(4 * kb) * kG + bo;
        int u = 0;
#pragma unroll 2
        for (; u + 1 < len; u += 2) {  // two k-steps on separate accumulators
          const double a0 = A[u * 64], a1 = A[(u + 1) * 64];
          double b0[NG], b1[NG];
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            b0[g] = B[size_t(g) * KN * kG + u * 4 * kG];
            b1[g] = B[size_t(g) * KN * kG + (u + 1) * 4 * kG];
          }
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            dmma6(d[0][g][0], d[0][g][1], a0, b0[g]);
            dmma6(d[1][g][0], d[1][g][1], a1, b1[g]);
          }
        }
        if (u < len) {
          const double a0 = A[u * 64];
#pragma unroll
          for (int g = 0; g < NG; ++g) dmma6(d[0][g][0], d[0][g][1], a0, B[size_t(g) * KN * kG + u * 4 * kG]);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma::smem_u32(&empty[sl * R + slot])) : "memory");
      }
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        if (gp + g < P.ngroups) {
          double* O = P.W1 + widx<KN>(gp + g, J, P.ny) + size_t(16 * s + 8 * mt + (lane >> 2)) * kG + 2 * (lane & 3);
          *reinterpret_cast<double2*>(O) = make_double2(d[0][g][0] + d[1][g][0], d[0][g][1] + d[1][g][1]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma::smem_u32(bfree)) : "memory");
  }
}

// Row of the group-local numbering: group gr, row i of the group (L: rows ascend from 0, U: descend
// from ny-1); -1 when the (ragged, last) group has no such row.
__device__ __forceinline__ int grow(bool upper, int gr, int i, int k, int ny) {
  const int J = upper ? ny - 1 - gr * k - i : gr * k + i;
  return (J >= 0 && J < ny) ? J : -1;
}
// Packed propagator index of (group gr, row i): see V6Params.
__device__ __forceinline__ int propidx(bool upper, int gr, int i, int J, const V6Params& P) {
  if (P.k == 1) return P.thomas ? oprow(upper ? J + 1 : (J > 0 ? J - 1 : 0), P.jstar) : oprow(J, P.jstar);  // Thomas: H_{J+1} / H_{J-1}
  if (upper) return gr < P.gconv ? i : P.k + (gr - P.gconv) * P.k + i;
  return gr < P.nind ? gr * P.k + i : P.nind * P.k + i;
}

// Zero-inflow chains inside the groups, pass i = P.pass (1 .. k-1), every group at once:
//   L: c'_J = c_J + G_J c'_{J-1},  J = g k + i;   U: d'_J = d_J + H_J d'_{J+1},  J = ny-1 - g k - i
// in place in W1.  One CTA per (group, pair of chain groups); the two chain groups' c'_{J-+1} are
// staged in shared memory; each warp owns whole 16-row slices and streams its operator slice from
// L2 / HBM in fragment order, 16 k-steps in flight (as v6_off_kernel, full rows instead of triangles).
template <int KN, bool kUpper, bool kBand>
__global__ void __launch_bounds__(kThr6, 1) v6_inner_kernel(V6Params P) {
  V6_DIMS
  extern __shared__ double Bs[];  // [2][kN][8]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bo = (lane & 3) * kG + (lane >> 2);
  const int npairs = (P.ngroups + 1) / 2;
  const int gr = blockIdx.x / npairs, gp = 2 * (blockIdx.x % npairs);
  const int J = grow(kUpper, gr, P.pass, P.k, P.ny);
  if (J < 0) return;
  const int Jp = kUpper ? J + 1 : J - 1;
  for (int i = threadIdx.x; i < KN * kG; i += kThr6) {  // double2 units over both groups
    const int gi = i / (KN * kG / 2), r = i - gi * (KN * kG / 2);
    double2 v = make_double2(0.0, 0.0);
    if (gp + gi < P.ngroups) v = __ldcg(reinterpret_cast<const double2*>(P.W1 + widx<KN>(gp + gi, Jp, P.ny)) + r);
    reinterpret_cast<double2*>(Bs)[i] = v;
  }
  __syncthreads();
  // the row's operator: G_J / H_J, or in the inverse-block form H_{J-1} / H_{J+1} (V6Params::thomas)
  const int Jop = P.thomas ? Jp : J;
  const bool useH = kUpper || P.thomas;
  const bool res = Jop >= P.jstar;
  for (int s = warp; s < kSl; s += 8) {
    const double* A = (useH ? P.Hp : P.Gp) + (size_t(oprow(Jop, P.jstar)) * kSl + s) * kKS * 64 + lane;
    double d[2][2][2] = {};
    double ac[kOffChunk][2], an[kOffChunk][2];
    int ks0 = 0, ks1 = kKS;  // compile-time constants without the band
    if constexpr (kBand) {
      const int2 b = (useH ? P.rawH : P.rawG)[size_t(oprow(Jop, P.jstar)) * kSl + s];
      ks0 = b.x;
      ks1 = b.y;
    }
#pragma unroll
    for (int u = 0; u < kOffChunk; ++u) {
      const bool ok = ks0 + u < ks1;
      ac[u][0] = ok ? ldop(A + size_t(ks0 + u) * 64, res) : 0.0;
      ac[u][1] = ok ? ldop(A + size_t(ks0 + u) * 64 + 32, res) : 0.0;
    }
    for (int ks = ks0; ks < ks1; ks += kOffChunk) {
#pragma unroll
      for (int u = 0; u < kOffChunk; ++u) {
        const bool ok = ks + kOffChunk + u < ks1;
        an[u][0] = ok ? ldop(A + size_t(ks + kOffChunk + u) * 64, res) : 0.0;
        an[u][1] = ok ? ldop(A + size_t(ks + kOffChunk + u) * 64 + 32, res) : 0.0;
      }
      if (ks + kOffChunk <= ks1) {  // a whole chunk: no per-step guard
#pragma unroll
        for (int u = 0; u < kOffChunk; ++u) {
          const double b0 = Bs[(4 * (ks + u)) * kG + bo];
          const double b1 = Bs[KN * kG + (4 * (ks + u)) * kG + bo];
          dmma6(d[0][0][0], d[0][0][1], ac[u][0], b0);
          dmma6(d[0][1][0], d[0][1][1], ac[u][1], b0);
          dmma6(d[1][0][0], d[1][0][1], ac[u][0], b1);
          dmma6(d[1][1][0], d[1][1][1], ac[u][1], b1);
        }
      } else {
#pragma unroll
        for (int u = 0; u < kOffChunk; ++u) {
          if (ks + u < ks1) {
            const double b0 = Bs[(4 * (ks + u)) * kG + bo];
            const double b1 = Bs[KN * kG + (4 * (ks + u)) * kG + bo];
            dmma6(d[0][0][0], d[0][0][1], ac[u][0], b0);
            dmma6(d[0][1][0], d[0][1][1], ac[u][1], b0);
            dmma6(d[1][0][0], d[1][0][1], ac[u][0], b1);
            dmma6(d[1][1][0], d[1][1][1], ac[u][1], b1);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kOffChunk; ++u) {
        ac[u][0] = an[u][0];
        ac[u][1] = an[u][1];
      }
    }
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      if (gp + g >= P.ngroups) break;
      double* O = P.W1 + widx<KN>(gp + g, J, P.ny) + size_t(16 * s + (lane >> 2)) * kG + 2 * (lane & 3);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        double2* o2 = reinterpret_cast<double2*>(O + mt * 8 * kG);
        const double2 c0 = *o2;
        *o2 = make_double2(c0.x + d[g][mt][0], c0.y + d[g][mt][1]);
      }
    }
  }
}

// The dependent chain of one sweep direction for chain groups g0 .. g0 + gridDim.x/kSl - 1:
//   L: y_J = c_J + G_J y_{J-1}  (J = 0 .. ny-1; c in W1, y to W0)
//   U: x_J = d_J + H_J x_{J+1}  (J = ny-1 .. 0; d in W1, x to W0 and the job's outputs)
// CTA (s, g) owns rows 16s..16s+15 of the 8 chains of group g.  Its operator
// slice (128 KB) and y_{J-1} (64 KB) arrive by bulk copies into shared memory:
// plain loads were bounded by the SM's outstanding-miss limit (~15 B/clk/SM
// measured with the operands replaced by constants: the operator stream, not
// the DMMA, set the row time), the copy engine is not.  The next row's slice
// is copied while this row's reduction, outputs and row barrier run.  Each
// output warp publishes its own stores (release after __syncwarp), 4 counts
// per CTA and row, so no CTA barrier sits between the stores and the count.
template <int KN>
constexpr size_t chain_smem() { return sizeof(double) * (16 * KN + KN * kG + 2 * 8 * 128) + 3 * sizeof(uint64_t); }

__device__ __forceinline__ ulonglong2 ld_slots(const unsigned long long* p) {  // two adjacent slots
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];\n" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_slot(unsigned long long* p, double val) {
  unsigned long long b = (unsigned long long)__double_as_longlong(val);
  if (b == kLLEmpty) b = 0x7FF8000000000000ull;  // a NaN with the sentinel's bits: publish the canonical one
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(b) : "memory");
}

// co-resident CTAs per SM the register budget must allow (shared memory would allow 3 / 2 / 1 at
// KN = 256 / 512 / 1024); without it the KN = 512 packet-handoff kernel takes 130 registers, one
// CTA per SM, and config 2's 256 CTAs run in two waves (measured: P^-1 170 -> 200 ms)
template <int KN>
constexpr int chain_min_blocks() { return KN <= 512 ? 2 : 1; }  // 3 at KN = 256 spills (80 registers)

template <int KN, bool kUpper, bool kLL, bool kWin>
__global__ void __launch_bounds__(kThr6, chain_min_blocks<KN>()) v6_chain_kernel(V6Params P) {
  V6_DIMS
  extern __shared__ __align__(128) double sm6[];
  double* As = sm6;                 // [ks KN/4][mt 2][lane 32]
  double* Bs = As + 16 * KN;       // [k KN][8]
  double* red = Bs + KN * kG;      // [2][warp 8][128]: alternating, so one CTA barrier per product
  uint64_t* barA = reinterpret_cast<uint64_t*>(red + 2 * 8 * 128);
  uint64_t* barB = barA + 1;  // [2]: the halves of y_{J-1} (warps 0-3 use k < KN/2, warps 4-7 the rest)
  // CTA (sigma, g): sigma = i * kSl + s is slice s of row i of every group; g is the REAL chain
  // group (with the twisted elimination the CTA serves its two virtual groups g, g + nreal in turn)
  const int rows_per_g = kSl * P.k;
  const int sig = blockIdx.x % rows_per_g, g = P.g0 + blockIdx.x / rows_per_g;
  const int s = sig % kSl, gi = sig / kSl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ny = P.ny;
  const int nh = (kLL && P.twist) ? 2 : 1;
  const double* Mbase = (kUpper ? P.Psi : P.Phi) + size_t(s) * kKS * 64;
  const size_t mstride = size_t(kSl) * kKS * 64;
  unsigned* cnt = P.cnt + g;
  const bool last_row = gi == P.k - 1;  // the row the next group waits for
  int m = 0, n = 0;
  const bool outt = threadIdx.x < 128;
  if (outt) slice_coords(threadIdx.x, m, n);
  const int row = 16 * s + m, ch = g * kG + n;
  double* out = nullptr;
  double* out2 = nullptr;
  double g2 = 0.0;
  if (kUpper && outt && row < P.nx && ch < P.nchains) {
    const FastStep st = P.jobs[size_t(ch) * P.nsteps + P.t];
    if (st.in) {
      out = st.out;
      out2 = st.out2;
      if (st.out2 && st.node2 > 0 && P.gam) g2 = P.gam[st.node2];
    }
  }
  auto Jof = [&](int gr) { return grow(kUpper, gr, gi, P.k, ny); };  // this CTA's row of group gr
  // v: the chain value of row J (slot, W0); pv: the product alone.  Thomas form, U: the product is
  // x_{J+1} (the start row has none)
  auto emit = [&](int h, int gr, int J, double v, double pv, double yv) {
    const int gv = g + h * P.nreal;
    if (kLL && last_row)
      st_slot(P.ll + (size_t(gv) * P.ngr + gr) * (KN * kG) + size_t(row) * kG + n, v);
    // Thomas form, U, grouped rows: the chain value is X_J = y_J + x_{J+1}; yv = y_J was read from W0
    // (this same element) before this store, at the start of the product
    P.W0[widx<KN>(gv, J, ny) + size_t(row) * kG + n] = v;
    if (kUpper && P.thomas && J == ny - 1) return;  // X_{M-1} = y_{M-1} + x_M: the start row has no output
    const int Jo = P.thomas ? J + 1 : J;
    const double ov = P.thomas ? (P.k == 1 ? pv : v - yv) : v;
    const int Ja = h ? P.nyA - 1 - Jo : Jo;  // the block row of the grid (bottom half: mirrored)
    if (out) out[size_t(Ja) * P.nx + row] = ov;
    if (out2) out2[size_t(Ja) * P.nx + row] = ov + g2;
  };
  // each output warp publishes its own stores (release after __syncwarp), so
  // no CTA-wide barrier sits between the stores and the count; 4 per CTA and row
  auto signal = [&]() {
    if (!kLL && outt && last_row) {
      __syncwarp();
      if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(cnt) : "memory");
    }
  };
  // windows only in the <kWin> instantiation (slot handoff; the counter path copies y in fixed halves)
  const int2* band = kWin ? (kUpper ? P.bandPsi : P.bandPhi) : nullptr;
  auto window = [&](int pidx) { return band ? band[size_t(pidx) * kSl + s] : make_int2(0, kKW); };
  auto copy_a = [&](int gr, int J, int2 wn) {  // thread 0: this slice's window of the operator row
    const int pidx = propidx(kUpper, gr, gi, J, P);
    tma_load(As + size_t(wn.x) * 64, Mbase + size_t(pidx) * mstride + size_t(wn.x) * 64,
             uint32_t(sizeof(double) * 64 * 8 * wn.y), barA);
  };
  // the window of the next group step is fetched one step ahead, off the row's critical path
  int2 wn_next = make_int2(0, kKW);
  if (threadIdx.x == 0) {
    mbar_init(barA, 1);
    mbar_init(barB, 1);
    mbar_init(barB + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  {  // group 0 has no inflow: its rows are the zero-inflow chain values
    const int J = Jof(0);
    if (J < 0) return;
    if (outt)
      for (int h = 0; h < nh; ++h) {
        const size_t e = widx<KN>(g + h * P.nreal, J, ny) + size_t(row) * kG + n;
        const double y0 = (kUpper && P.thomas && P.k > 1) ? __ldcg(P.W0 + e) : 0.0;
        emit(h, 0, J, __ldcg(P.W1 + e), 0.0, y0);
      }
    signal();
    if (P.ngr > 1 && Jof(1) >= 0) {
      wn_next = window(propidx(kUpper, 1, gi, Jof(1), P));
      if (threadIdx.x == 0) copy_a(1, Jof(1), wn_next);
    }
  }
  const int bo = (lane & 3) * kG + (lane >> 2);
  const bool tm = P.tim && blockIdx.x == kSl / 2 && threadIdx.x == 0;  // a middle slice: the full band window
  long long ts[7] = {0, 0, 0, 0, 0, 0, 0}, acc[6] = {0, 0, 0, 0, 0, 0};
  int rb = 0;  // reduction buffer in use
  for (int idx = 1; idx < P.ngr; ++idx) {
    const int J = Jof(idx);
    if (J < 0) break;  // the ragged last group has no such row (and no successor waits for it)
    const int Jp = kUpper ? ny - idx * P.k : idx * P.k - 1;  // the previous group's last row
    const int2 wn = wn_next;  // {first k-step, k-steps per warp}
    const bool more = idx + 1 < P.ngr && Jof(idx + 1) >= 0;
    if (more) wn_next = window(propidx(kUpper, idx + 1, gi, Jof(idx + 1), P));
    const uint32_t par = uint32_t(idx - 1) & 1u;
    for (int h = 0; h < nh; ++h) {
      const int gv = g + h * P.nreal;
      if (tm) ts[0] = clock64();
      double cval = 0.0;
      double yv = 0.0;  // Thomas form, U, grouped rows: y_J, still in W0 until this row's emit overwrites it
      if (outt) {
        const size_t e = widx<KN>(gv, J, ny) + size_t(row) * kG + n;
        cval = __ldcg(((kUpper && P.thomas && P.k == 1) ? P.W0 : P.W1) + e);
        if (kUpper && P.thomas && P.k > 1) yv = __ldcg(P.W0 + e);
      }
      if (!kLL) {
        if (threadIdx.x == 0) {
          const unsigned target = unsigned(idx) * kSl * 4;
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
          } while (v < target);
          if (tm) ts[1] = clock64();
          // y_{J-1} was written by other CTAs through the generic proxy; the copy reads it through the async proxy
          asm volatile("fence.proxy.async.global;\n" ::: "memory");
          const double* ysrc = P.W0 + widx<KN>(gv, Jp, ny);
          tma_load(Bs, ysrc, sizeof(double) * KN * kG / 2, barB);
          tma_load(Bs + KN * kG / 2, ysrc + KN * kG / 2, sizeof(double) * KN * kG / 2, barB + 1);
        }
        __syncthreads();
      }
      if (kLL) {
        // this warp's k-steps of the previous group's last row: 32 values per k-step, loaded as
        // pairs (16 bytes), up to 8 loads in flight; re-issue only the pairs not yet complete.
        // A warp reads and writes only its own k-range of Bs, so no CTA barrier guards Bs here.
        (void)Jp;
        const size_t voff = size_t(wn.x + warp * wn.y) * 32 + 2 * lane;
        const unsigned long long* src = P.ll + (size_t(gv) * P.ngr + (idx - 1)) * (KN * kG) + voff;
        double* dstB = Bs + voff;
        if (!kWin) {  // full row: compile-time batches
          constexpr int kPairs = KN / 64;  // 16-byte loads per lane
          constexpr int kBatch = kPairs < 8 ? kPairs : 8;
#pragma unroll 1
          for (int q0 = 0; q0 < kPairs; q0 += kBatch) {
            ulonglong2 v[kBatch];
            unsigned pending = (1u << kBatch) - 1u;
            while (pending) {
#pragma unroll
              for (int u = 0; u < kBatch; ++u)
                if ((pending >> u) & 1u) v[u] = ld_slots(src + (q0 + u) * 64);
#pragma unroll
              for (int u = 0; u < kBatch; ++u)
                if (((pending >> u) & 1u) && ((v[u].x != kLLEmpty && v[u].y != kLLEmpty) || P.nopoll)) {
                  *reinterpret_cast<double2*>(dstB + (q0 + u) * 64) =
                      make_double2(__longlong_as_double((long long)v[u].x), __longlong_as_double((long long)v[u].y));
                  pending &= ~(1u << u);
                }
              if (pending && P.spin_ns) __nanosleep(P.spin_ns);
            }
          }
        } else {
          const int npairs = wn.y >> 1;
#pragma unroll 1
          for (int q0 = 0; q0 < npairs; q0 += 8) {
            ulonglong2 v[8];
            unsigned pending = npairs - q0 >= 8 ? 0xffu : (1u << (npairs - q0)) - 1u;
            while (pending) {
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if ((pending >> u) & 1u) v[u] = ld_slots(src + (q0 + u) * 64);
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (((pending >> u) & 1u) && ((v[u].x != kLLEmpty && v[u].y != kLLEmpty) || P.nopoll)) {
                  *reinterpret_cast<double2*>(dstB + (q0 + u) * 64) =
                      make_double2(__longlong_as_double((long long)v[u].x), __longlong_as_double((long long)v[u].y));
                  pending &= ~(1u << u);
                }
              if (pending && P.spin_ns) __nanosleep(P.spin_ns);
            }
          }
        }
        __syncwarp();
        if (tm) ts[1] = ts[2] = clock64();
        if (h == 0) mbar_wait(barA, par);  // the operator slice serves both halves
        if (tm) ts[3] = clock64();
      } else {
        mbar_wait(barA, par);
        if (tm) ts[2] = clock64();
        mbar_wait(barB + (warp >> 2), par);  // this warp's half only: the other half may still be landing
        if (tm) ts[3] = clock64();
      }
      double d[2][2][2] = {};
      const double* Aw = As + size_t(wn.x + warp * wn.y) * 64 + lane;
      const double* Bw = Bs + size_t(wn.x + warp * wn.y) * 4 * kG + bo;
      if (!kWin) {  // full row: the fixed, fully unrolled product
#pragma unroll
        for (int i0 = 0; i0 < kKW; i0 += 8) {
          double a0[8], a1[8], b[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            a0[u] = Aw[(i0 + u) * 64];
            a1[u] = Aw[(i0 + u) * 64 + 32];
            b[u] = Bw[(i0 + u) * 4 * kG];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            dmma6(d[u & 1][0][0], d[u & 1][0][1], a0[u], b[u]);
            dmma6(d[u & 1][1][0], d[u & 1][1][1], a1[u], b[u]);
          }
        }
      } else
#pragma unroll 1
      for (int i0 = 0; i0 < wn.y; i0 += 8) {
        double a0[8], a1[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ok = i0 + u < wn.y;
          a0[u] = ok ? Aw[(i0 + u) * 64] : 0.0;
          a1[u] = ok ? Aw[(i0 + u) * 64 + 32] : 0.0;
          b[u] = ok ? Bw[(i0 + u) * 4 * kG] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0 + u < wn.y) {
            dmma6(d[u & 1][0][0], d[u & 1][0][1], a0[u], b[u]);
            dmma6(d[u & 1][1][0], d[u & 1][1][1], a1[u], b[u]);
          }
        }
      }
      double* redw = red + rb * (8 * 128);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) redw[warp * 128 + (mt * 32 + lane) * 2 + e] = d[0][mt][e] + d[1][mt][e];
      if (tm) ts[4] = clock64();
      // As / Bs consumed by every warp, red[rb] complete.  The other buffer is written next, after
      // this barrier, which every reader of its previous contents has passed: one barrier per product.
      __syncthreads();
      if (outt) {
        const double pv = reduce8(redw, threadIdx.x);
        emit(h, idx, J, cval + pv, pv, yv);
      }
      rb ^= 1;
      if (tm) {
        ts[5] = ts[6] = clock64();
        for (int q = 0; q < 6; ++q) acc[q] += ts[q + 1] - ts[q];
      }
    }
    signal();
    if (more && threadIdx.x == 0) copy_a(idx + 1, Jof(idx + 1), wn_next);
  }
  if (tm)
    for (int q = 0; q < 6; ++q) atomicAdd(reinterpret_cast<unsigned long long*>(P.tim + (kUpper ? 6 : 0) + q),
                                          (unsigned long long)acc[q]);
}

// The windowed chain (slot handoff + numerical band, config 2's case) with the NEXT product's slots
// prefetched: shared memory holds only the band window (As: 8 wmax k-steps, two Bs buffers of the
// same extent), and each warp copies its k-range of the next product's slots global -> shared with
// cp.async.cg (L2, no registers) before (same row, other half) or right after (next row) the
// current product's DMMA loop, so the slot loads -- ~1.6k cycles per product when issued and
// awaited in place, even with every value already published (KKT_V6_NOPOLL) -- overlap the
// product, its reduction and its stores.  On arrival the warp checks its own pairs for the
// sentinel and polls the (rare) missing ones synchronously, exactly as v6_chain_kernel does.
template <int KN>
constexpr size_t chainw_smem(int wmax) {
  return sizeof(double) * (size_t(8) * wmax * 64 + 2 * size_t(8) * wmax * 32 + 2 * 8 * 128) + 3 * sizeof(uint64_t);
}

template <int KN, bool kUpper>
__global__ void __launch_bounds__(kThr6, chain_min_blocks<KN>()) v6_chainw_kernel(V6Params P) {
  V6_DIMS
  extern __shared__ __align__(128) double sm6[];
  const int wmax = P.wmax;
  double* As = sm6;                          // [8 wmax k-steps][mt 2][lane 32], window-relative
  double* Bs0 = As + size_t(8) * wmax * 64;  // [2][warp 8][wmax k-steps][4][8], window-relative
  const size_t bsz = size_t(8) * wmax * 32;
  double* red = Bs0 + 2 * bsz;               // [2][warp 8][128]
  uint64_t* barA = reinterpret_cast<uint64_t*>(red + 2 * 8 * 128);
  const int rows_per_g = kSl * P.k;
  const int sig = blockIdx.x % rows_per_g, g = P.g0 + blockIdx.x / rows_per_g;
  const int s = sig % kSl, gi = sig / kSl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ny = P.ny;
  const int nh = P.twist ? 2 : 1;
  const double* Mbase = (kUpper ? P.Psi : P.Phi) + size_t(s) * kKS * 64;
  const size_t mstride = size_t(kSl) * kKS * 64;
  const bool last_row = gi == P.k - 1;
  int m = 0, n = 0;
  const bool outt = threadIdx.x < 128;
  if (outt) slice_coords(threadIdx.x, m, n);
  const int row = 16 * s + m, ch = g * kG + n;
  double* out = nullptr;
  double* out2 = nullptr;
  double g2 = 0.0;
  if (kUpper && outt && row < P.nx && ch < P.nchains) {
    const FastStep st = P.jobs[size_t(ch) * P.nsteps + P.t];
    if (st.in) {
      out = st.out;
      out2 = st.out2;
      if (st.out2 && st.node2 > 0 && P.gam) g2 = P.gam[st.node2];
    }
  }
  auto Jof = [&](int gr) { return grow(kUpper, gr, gi, P.k, ny); };
  auto emit = [&](int h, int gr, int J, double v, double pv, double yv) {  // as in v6_chain_kernel
    const int gv = g + h * P.nreal;
    if (last_row) st_slot(P.ll + (size_t(gv) * P.ngr + gr) * (KN * kG) + size_t(row) * kG + n, v);
    // Thomas form, U, grouped rows: the chain value is X_J = y_J + x_{J+1}; yv = y_J was read from W0
    // (this same element) before this store, at the start of the product
    P.W0[widx<KN>(gv, J, ny) + size_t(row) * kG + n] = v;
    if (kUpper && P.thomas && J == ny - 1) return;  // X_{M-1} = y_{M-1} + x_M: the start row has no output
    const int Jo = P.thomas ? J + 1 : J;
    const double ov = P.thomas ? (P.k == 1 ? pv : v - yv) : v;
    const int Ja = h ? P.nyA - 1 - Jo : Jo;
    if (out) out[size_t(Ja) * P.nx + row] = ov;
    if (out2) out2[size_t(Ja) * P.nx + row] = ov + g2;
  };
  const int2* band = kUpper ? P.bandPsi : P.bandPhi;
  auto window = [&](int pidx) { return band[size_t(pidx) * kSl + s]; };
  // This slice's window of the operator row of (group step gr, block row J) -> As, unless As holds
  // it already: the rows past jstar share one converged operator set (70% of config 2's rows), so
  // the chain keeps that window in shared memory instead of fetching it again for every row.
  // Every thread keeps the bookkeeping (held row, copies issued, one in flight); thread 0 copies.
  int held = -1;
  uint32_t ncopy = 0;
  bool inflight = false;
  auto copy_a = [&](int gr, int J, int2 wn) {
    const int pidx = propidx(kUpper, gr, gi, J, P);
    if (pidx == held && !P.nohold) return;
    held = pidx;
    ++ncopy;
    inflight = true;
    if (threadIdx.x == 0)
      tma_load(As, Mbase + size_t(pidx) * mstride + size_t(wn.x) * 64, uint32_t(sizeof(double) * 64 * 8 * wn.y), barA);
  };
  // this warp's k-range of the slots of (virtual group gv, group step st) -> its part of Bs[buf]
  // (handing the whole window to the bulk-copy engine from one thread instead measured slower:
  // the copies land later than the per-lane cp.async ones, 113.5 vs 100.8 ms on the same box)
  auto prefetch = [&](int buf, int gv, int st, int2 wn) {
    const unsigned long long* src = P.ll + (size_t(gv) * P.ngr + st) * (KN * kG) + size_t(wn.x + warp * wn.y) * 32 + 2 * lane;
    const uint32_t dst = tma::smem_u32(Bs0 + buf * bsz + size_t(warp) * wmax * 32 + 2 * lane);
    const int npairs = wn.y >> 1;
    for (int q = 0; q < npairs; ++q)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + uint32_t(q) * 512),
                   "l"(__cvta_generic_to_global(src + q * 64))
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // the prefetched pairs have landed: those that still hold the sentinel are polled as in
  // v6_chain_kernel (up to 8 loads in flight per lane, only the incomplete pairs re-issued)
  auto complete = [&](int buf, int gv, int st, int2 wn) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    const unsigned long long* src = P.ll + (size_t(gv) * P.ngr + st) * (KN * kG) + size_t(wn.x + warp * wn.y) * 32 + 2 * lane;
    double* dstB = Bs0 + buf * bsz + size_t(warp) * wmax * 32 + 2 * lane;
    const int npairs = wn.y >> 1;
#pragma unroll 1
    for (int q0 = 0; q0 < npairs; q0 += 4) {
      unsigned pending = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u < npairs) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(dstB + (q0 + u) * 64);
          if (v.x == kLLEmpty || v.y == kLLEmpty) pending |= 1u << u;
        }
      if (P.nopoll) pending = 0;
      while (pending) {
        ulonglong2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((pending >> u) & 1u) v[u] = ld_slots(src + (q0 + u) * 64);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (((pending >> u) & 1u) && v[u].x != kLLEmpty && v[u].y != kLLEmpty) {
            *reinterpret_cast<ulonglong2*>(dstB + (q0 + u) * 64) = v[u];
            pending &= ~(1u << u);
          }
      }
    }
    __syncwarp();
  };
  int2 wn_next = make_int2(0, 2);
  if (threadIdx.x == 0) {
    mbar_init(barA, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // Two chain CTAs share an SM (CTA b with b + 148 under the usual placement, i.e. a group of the
  // lower half with one of the upper half).  Chains of different groups are independent, so
  // starting the upper half of the groups half a product late puts the two CTAs' DMMA loops in
  // anti-phase: each then has the SM's fp64 pipe to itself, and the other's slot loads, reduction
  // and stores run under it.  Nothing restores or destroys the offset (both CTAs are delayed
  // alike where they do overlap), so it holds along the whole chain.
  if (P.tim && threadIdx.x == 0 && blockIdx.x < 1024) {  // KKT_V6_TIM: which SM this CTA runs on
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    P.tim[12 + blockIdx.x] = (long long)smid;
  }
  if (P.stagger > 0 && 2 * (blockIdx.x / rows_per_g) >= gridDim.x / rows_per_g) {
    const long long t0 = clock64();
    while (clock64() - t0 < P.stagger) {
    }
  }
  {  // group 0 has no inflow: its rows are the zero-inflow chain values
    const int J = Jof(0);
    if (J < 0) return;
    if (outt)
      for (int h = 0; h < nh; ++h) {
        const size_t e = widx<KN>(g + h * P.nreal, J, ny) + size_t(row) * kG + n;
        const double y0 = (kUpper && P.thomas && P.k > 1) ? __ldcg(P.W0 + e) : 0.0;
        emit(h, 0, J, __ldcg(P.W1 + e), 0.0, y0);
      }
    if (P.ngr > 1 && Jof(1) >= 0) {
      wn_next = window(propidx(kUpper, 1, gi, Jof(1), P));
      copy_a(1, Jof(1), wn_next);
      prefetch(0, g, 0, wn_next);
    }
  }
  const int bo = (lane & 3) * kG + (lane >> 2);
  const bool tm = P.tim && blockIdx.x == kSl / 2 && threadIdx.x == 0;
  long long ts[7] = {0, 0, 0, 0, 0, 0, 0}, acc[6] = {0, 0, 0, 0, 0, 0};
  int rb = 0, buf = 0;
  for (int idx = 1; idx < P.ngr; ++idx) {
    const int J = Jof(idx);
    if (J < 0) break;
    const int2 wn = wn_next;
    const bool more = idx + 1 < P.ngr && Jof(idx + 1) >= 0;
    if (more) wn_next = window(propidx(kUpper, idx + 1, gi, Jof(idx + 1), P));
    for (int h = 0; h < nh; ++h) {
      const int gv = g + h * P.nreal;
      if (tm) ts[0] = clock64();
      double cval = 0.0;
      double yv = 0.0;  // Thomas form, U, grouped rows: y_J, still in W0 until this row's emit overwrites it
      if (outt) {
        const size_t e = widx<KN>(gv, J, ny) + size_t(row) * kG + n;
        cval = __ldcg(((kUpper && P.thomas && P.k == 1) ? P.W0 : P.W1) + e);
        if (kUpper && P.thomas && P.k > 1) yv = __ldcg(P.W0 + e);
      }
      complete(buf, gv, idx - 1, wn);
      if (tm) ts[1] = ts[2] = clock64();
      // the other half of this row was published a whole product ago: fetch it under this product
      const bool early = h + 1 < nh;
      if (early) prefetch(buf ^ 1, g + (h + 1) * P.nreal, idx - 1, wn);
      if (inflight) {  // the operator slice serves both halves
        mbar_wait(barA, (ncopy - 1u) & 1u);
        inflight = false;
      }
      if (tm) ts[3] = clock64();
      double d[2][2][2] = {};
      const double* Aw = As + size_t(warp * wn.y) * 64 + lane;
      const double* Bw = Bs0 + buf * bsz + size_t(warp) * wmax * 32 + bo;
#pragma unroll 1
      for (int i0 = 0; i0 < wn.y; i0 += 8) {
        double a0[8], a1[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ok = i0 + u < wn.y;
          a0[u] = ok ? Aw[(i0 + u) * 64] : 0.0;
          a1[u] = ok ? Aw[(i0 + u) * 64 + 32] : 0.0;
          b[u] = ok ? Bw[(i0 + u) * 4 * kG] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0 + u < wn.y) {
            dmma6(d[u & 1][0][0], d[u & 1][0][1], a0[u], b[u]);
            dmma6(d[u & 1][1][0], d[u & 1][1][1], a1[u], b[u]);
          }
        }
      }
      // the next row's first half was published during this row: fetch it under the reduction and the
      // stores (issued before the DMMA loop instead it measured no faster: 100.9 vs 100.5 ms)
      if (!early && more) prefetch(buf ^ 1, g, idx, wn_next);
      double* redw = red + rb * (8 * 128);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) redw[warp * 128 + (mt * 32 + lane) * 2 + e] = d[0][mt][e] + d[1][mt][e];
      if (tm) ts[4] = clock64();
      __syncthreads();  // As consumed by every warp (last half), red[rb] complete
      // the next row's operator window, as soon as As is free (before this half's stores)
      if (h + 1 == nh && more) copy_a(idx + 1, Jof(idx + 1), wn_next);
      if (outt) {
        const double pv = reduce8(redw, threadIdx.x);
        emit(h, idx, J, cval + pv, pv, yv);
      }
      rb ^= 1;
      buf ^= 1;
      if (tm) {
        ts[5] = ts[6] = clock64();
        for (int q = 0; q < 6; ++q) acc[q] += ts[q + 1] - ts[q];
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (tm)
    for (int q = 0; q < 6; ++q) atomicAdd(reinterpret_cast<unsigned long long*>(P.tim + (kUpper ? 6 : 0) + q),
                                          (unsigned long long)acc[q]);
}

// The middle row of the twisted elimination: one dense block product per real chain group with
// packed operator rows, CTA (s, g) = 16 rows x 8 chains, 8 warps split along k (fixed-order sum).
//   mode 0 (between the inward and the outward chains):
//     x_M = Dm^{-1} b_M + E (y_{M-1} + y'_{M+1})  ->  Wm (x_M) and the job's out planes at row M
//   mode 1 (after the outward off-chain products d_j = Ui_j y_j):
//     d_{M-1} += H_{M-1} x_M for both halves: the inflow of the first outward row
template <int KN>
__global__ void __launch_bounds__(kThr6) v6_mid_kernel(V6Params P, int mode) {
  V6_DIMS
  __shared__ double red[8 * 128];
  const int s = blockIdx.x % kSl;
  const int gq = blockIdx.x / kSl;                 // mode 2: a virtual chain group; else a real one
  const int h2 = (mode == 2 && gq >= P.nreal) ? 1 : 0;
  const int g = gq - h2 * P.nreal;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bo = (lane & 3) * kG + (lane >> 2);
  const int M = P.ny;  // rows per half chain = the middle block row
  const size_t vec = size_t(KN) * kG;
  double* xm = P.Wm + size_t(P.nreal) * vec + size_t(g) * vec;
  double d[2][2] = {};
  auto prod = [&](const double* A, const double* in1, const double* in2) {
    const double* Aw = A + size_t(s) * kKS * 64 + lane;
#pragma unroll 4
    for (int i = 0; i < kKW; ++i) {
      const int ks = warp * kKW + i;
      const double a0 = __ldg(Aw + size_t(ks) * 64), a1 = __ldg(Aw + size_t(ks) * 64 + 32);
      double b = __ldcg(in1 + size_t(4 * ks) * kG + bo);
      if (in2) b += __ldcg(in2 + size_t(4 * ks) * kG + bo);
      dmma6(d[0][0], d[0][1], a0, b);
      dmma6(d[1][0], d[1][1], a1, b);
    }
  };
  if (mode == 0) {
    prod(P.Dm, P.Wm + size_t(g) * vec, nullptr);
    prod(P.Em, P.W0 + widx<KN>(g, M - 1, M), P.W0 + widx<KN>(g + P.nreal, M - 1, M));
  } else if (mode == 2) {  // Thomas form, after the outward chains: x_0 = H_0 X_0 of this half
    prod(P.Hp, P.W0 + widx<KN>(gq, 0, M), nullptr);
  } else if (!P.thomas) {
    prod(P.Hp + size_t(oprow(M - 1, P.jstar)) * kSl * kKS * 64, xm, nullptr);
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) red[warp * 128 + (mt * 32 + lane) * 2 + e] = d[mt][e];
  __syncthreads();
  if (threadIdx.x < 128) {
    int m, n;
    slice_coords(threadIdx.x, m, n);
    const int row = 16 * s + m, ch = g * kG + n;
    const double v = reduce8(red, threadIdx.x);
    if (mode == 0) {
      xm[size_t(row) * kG + n] = v;
      if (row < P.nx && ch < P.nchains) {
        const FastStep st = P.jobs[size_t(ch) * P.nsteps + P.t];
        if (st.in) {
          if (st.out) st.out[size_t(M) * P.nx + row] = v;
          if (st.out2) {
            double g2 = 0.0;
            if (st.node2 > 0 && P.gam) g2 = P.gam[st.node2];
            st.out2[size_t(M) * P.nx + row] = v + g2;
          }
        }
      }
    } else if (mode == 2) {
      if (row < P.nx && ch < P.nchains) {
        const FastStep st = P.jobs[size_t(ch) * P.nsteps + P.t];
        if (st.in) {
          const int Ja = h2 ? P.nyA - 1 : 0;
          if (st.out) st.out[size_t(Ja) * P.nx + row] = v;
          if (st.out2) {
            double g2 = 0.0;
            if (st.node2 > 0 && P.gam) g2 = P.gam[st.node2];
            st.out2[size_t(Ja) * P.nx + row] = v + g2;
          }
        }
      }
    } else if (P.thomas) {  // the start of the outward chains: X_{M-1} = y_{M-1} + x_M, both halves
      const double x = xm[size_t(row) * kG + n];
      const size_t a = widx<KN>(g, M - 1, M) + size_t(row) * kG + n, b = widx<KN>(g + P.nreal, M - 1, M) + size_t(row) * kG + n;
      P.W1[a] = P.W0[a] + x;
      P.W1[b] = P.W0[b] + x;
    } else {
      P.W1[widx<KN>(g, M - 1, M) + size_t(row) * kG + n] += v;
      P.W1[widx<KN>(g + P.nreal, M - 1, M) + size_t(row) * kG + n] += v;
    }
  }
}

// dev[2J + m] = max |M_J - M_{ny-1}|, mag[2J + m] = max |M_J|, M = Li (m = 0), Ui (m = 1)
__global__ void __launch_bounds__(256) v6_conv_kernel(const double* __restrict__ Li, const double* __restrict__ Ui,
                                                      int nx, int ny, double* __restrict__ dev,
                                                      double* __restrict__ mag) {
  __shared__ double sh[4][256];
  const int J = blockIdx.x;
  const size_t nn = size_t(nx) * nx;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (size_t e = threadIdx.x; e < nn; e += blockDim.x) {
    const double l = Li[size_t(J) * nn + e], u = Ui[size_t(J) * nn + e];
    v[0] = fmax(v[0], fabs(l - Li[size_t(ny - 1) * nn + e]));
    v[1] = fmax(v[1], fabs(u - Ui[size_t(ny - 1) * nn + e]));
    v[2] = fmax(v[2], fabs(l));
    v[3] = fmax(v[3], fabs(u));
  }
  for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = v[q];
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w)
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = fmax(sh[q][threadIdx.x], sh[q][threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x < 2) {
    dev[2 * J + threadIdx.x] = sh[threadIdx.x][0];
    mag[2 * J + threadIdx.x] = sh[2 + threadIdx.x][0];
  }
}

// Window table of a packed operator set (see V6Params::bandPhi): one CTA per operator row.
template <int KN>
__global__ void __launch_bounds__(256) v6_band_kernel(const double* __restrict__ packed, double tol, int2* __restrict__ band,
                                                      int2* __restrict__ raw) {
  V6_DIMS
  __shared__ double smax[256];
  __shared__ int slo[kSl], shi[kSl];
  const double* M = packed + size_t(blockIdx.x) * KN * KN;
  double m = 0.0;
  for (int e = threadIdx.x; e < KN * KN; e += 256) m = fmax(m, fabs(M[e]));
  smax[threadIdx.x] = m;
  for (int i = threadIdx.x; i < kSl; i += 256) {
    slo[i] = kKS;
    shi[i] = -1;
  }
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + w]);
    __syncthreads();
  }
  const double thr = tol * smax[0];
  for (int e = threadIdx.x; e < KN * KN; e += 256) {
    if (fabs(M[e]) > thr) {
      const int ks = (e >> 6) % kKS, sl = (e >> 6) / kKS;
      atomicMin(&slo[sl], ks);
      atomicMax(&shi[sl], ks);
    }
  }
  __syncthreads();
  for (int sl = threadIdx.x; sl < kSl; sl += 256) {
    const int lo = slo[sl], hi = shi[sl];
    int cnt = 2, w0 = 0;
    if (hi >= lo) {
      cnt = min(kKW, 2 * ((hi - lo + 1 + 15) / 16));  // k-steps per warp, even
      w0 = max(0, min(lo, kKS - 8 * cnt));
    }
    if (band) band[size_t(blockIdx.x) * kSl + sl] = make_int2(w0, cnt);
    if (raw) raw[size_t(blockIdx.x) * kSl + sl] = hi >= lo ? make_int2(lo, hi + 1) : make_int2(0, 0);
  }
}

// Fragment-order pack: dst[J][s][ks][mt][lane] = scale * src[J][16s+8mt+lane/4][4ks+lane%4]
template <int KN>
__global__ void v6_pack_kernel(const double* __restrict__ src, int nx, int nJ, double scale,
                               double* __restrict__ dst) {
  V6_DIMS
  const size_t per = size_t(KN) * KN, total = size_t(nJ) * per, nn = size_t(nx) * nx;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t J = e / per;
    const int r = int(e - J * per);
    const int lane = r & 31, mt = (r >> 5) & 1, ks = (r >> 6) % kKS, s = (r >> 6) / kKS;
    const int a = 16 * s + 8 * mt + (lane >> 2), b = 4 * ks + (lane & 3);
    dst[e] = (a < nx && b < nx) ? scale * src[J * nn + size_t(a) * nx + b] : 0.0;
  }
}

__global__ void v6_copy_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) b[e] = a[e];
}

__global__ void v6_scale_kernel(int64_t n, double f, double* __restrict__ a) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) a[e] *= f;
}

bool off_plain() {  // KKT_V6_OFF=1: the plain-load off-chain kernel
  static const bool v = std::getenv("KKT_V6_OFF") != nullptr;
  return v;
}

template <int KN>
void launch_chain(Ctx* c, bool upper, const V6Params& P, int ngroups_wave) {
  V6_DIMS
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kSl * P.k * ngroups_wave);
  cfg.blockDim = dim3(kThr6);
  cfg.dynamicSmemBytes = chain_smem<KN>();
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA of the grid co-resident (row barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  V6Params p = P;
  void* args[] = {&p};
  const bool win = P.ll && P.bandPhi;
  if (win) cfg.dynamicSmemBytes = chainw_smem<KN>(P.wmax);
  const void* fn =
      win ? (upper ? reinterpret_cast<const void*>(&v6_chainw_kernel<KN, true>)
                   : reinterpret_cast<const void*>(&v6_chainw_kernel<KN, false>))
          : P.ll ? (upper ? reinterpret_cast<const void*>(&v6_chain_kernel<KN, true, true, false>)
                          : reinterpret_cast<const void*>(&v6_chain_kernel<KN, false, true, false>))
                 : (upper ? reinterpret_cast<const void*>(&v6_chain_kernel<KN, true, false, false>)
                          : reinterpret_cast<const void*>(&v6_chain_kernel<KN, false, false, false>));
  KKT_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  c->launches++;
}

// co-resident chain CTAs of the device; also sets the kernels' shared-memory limits
template <int KN>
int chain_capacity() {
  V6_DIMS
  static int cap = 0;
  if (!cap) {
    const int cs = int(chain_smem<KN>()), os = int(off_smem<KN>());
    KKT_CUDA(cudaFuncSetAttribute(v6_chain_kernel<KN, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs));
    KKT_CUDA(cudaFuncSetAttribute(v6_chain_kernel<KN, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs));
    KKT_CUDA(cudaFuncSetAttribute(v6_chain_kernel<KN, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs));
    KKT_CUDA(cudaFuncSetAttribute(v6_chain_kernel<KN, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs));
    const int ws = KN <= 512 ? (113 << 10) : (226 << 10);  // the windowed kernel's budget (see windows_pay)
    KKT_CUDA(cudaFuncSetAttribute(v6_chainw_kernel<KN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ws));
    KKT_CUDA(cudaFuncSetAttribute(v6_chainw_kernel<KN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ws));
    KKT_CUDA(cudaFuncSetAttribute(v6_off_kernel<KN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, os));
    KKT_CUDA(cudaFuncSetAttribute(v6_off_kernel<KN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, os));
    KKT_CUDA(cudaFuncSetAttribute(v6_inner_kernel<KN, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, os));
    KKT_CUDA(cudaFuncSetAttribute(v6_inner_kernel<KN, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, os));
    KKT_CUDA(cudaFuncSetAttribute(v6_inner_kernel<KN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, os));
    KKT_CUDA(cudaFuncSetAttribute(v6_inner_kernel<KN, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, os));
    const int os2 = int(off2_smem<KN, 2>());
    KKT_CUDA(cudaFuncSetAttribute(v6_off2_kernel<KN, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, os2));
    KKT_CUDA(cudaFuncSetAttribute(v6_off2_kernel<KN, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, os2));
    KKT_CUDA(cudaFuncSetAttribute(v6_off3_kernel<KN, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(off3_smem<KN, 2>())));
    KKT_CUDA(cudaFuncSetAttribute(v6_off3_kernel<KN, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(off3_smem<KN, 2>())));
    if constexpr (KN <= 512) {
      KKT_CUDA(cudaFuncSetAttribute(v6_off3_kernel<KN, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(off3_smem<KN, 4>())));
      KKT_CUDA(cudaFuncSetAttribute(v6_off3_kernel<KN, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(off3_smem<KN, 4>())));
    }
    if constexpr (KN <= 512) {
      const int os4 = int(off2_smem<KN, 4>());
      KKT_CUDA(cudaFuncSetAttribute(v6_off2_kernel<KN, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, os4));
      KKT_CUDA(cudaFuncSetAttribute(v6_off2_kernel<KN, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, os4));
    }
    int p0 = 0, p1 = 0;
    int q0 = 0, q1 = 0;
    int r0 = 0, r1 = 0;
    KKT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p0, v6_chain_kernel<KN, false, false, false>, kThr6, cs));
    KKT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, v6_chain_kernel<KN, true, false, false>, kThr6, cs));
    KKT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q0, v6_chain_kernel<KN, false, true, false>, kThr6, cs));
    KKT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q1, v6_chain_kernel<KN, true, true, false>, kThr6, cs));
    KKT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r0, v6_chainw_kernel<KN, false>, kThr6, ws));
    KKT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r1, v6_chainw_kernel<KN, true>, kThr6, ws));
    p0 = std::min(p0, std::min(q0, r0));
    p1 = std::min(p1, std::min(q1, r1));
    int dev = 0, nsm = kSmCount;
    KKT_CUDA(cudaGetDevice(&dev));
    KKT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    cap = std::max(1, std::min(p0, p1)) * nsm;
    if (std::getenv("KKT_V6_TIM"))
      std::fprintf(stderr, "v6 KN %d: %d chain CTAs per SM, %d co-resident\n", KN, std::min(p0, p1), cap);
  }
  return cap;
}

// chain groups (of 8 chains) per co-resident wave at grouping k
template <int KN>
int groups_per_wave(int k) {
  V6_DIMS
  return std::max(1, chain_capacity<KN>() / (kSl * k));
}

template <int KN>
void pack(Ctx* c, const double* src, int nJ, double scale, double* dst) {
  KKT_LAUNCH(c, v6_pack_kernel<KN>, kSmCount * 8, 256, 0, src, c->nx, nJ, scale, dst);
}

template <int KN>
void run_steps(Ctx* c, V6Params& P, int nsteps, int ngroups) {
  V6_DIMS
  // ngroups: (virtual) chain groups of the block vectors; the chain grid covers the REAL groups
  const int nchain_groups = P.twist ? P.nreal : ngroups;
  const int gpw = groups_per_wave<KN>(P.k);
  const int og = std::min(P.ny, kSmCount);
  const int og2 = std::min(P.ny * ((ngroups + 1) / 2), kSmCount), og4 = std::min(P.ny * ((ngroups + 3) / 4), kSmCount);  // off2: flat items
  const int npairs = (ngroups + 1) / 2;
  for (int t = 0; t < nsteps; ++t) {
    P.t = t;
    P.g0 = 0;
    KKT_LAUNCH(c, v6_form_b_kernel<KN>, (ngroups * P.ny + (P.twist ? P.nreal : 0)) * (KN / kFbChunk), kFbChunk, 0, P);
    for (int dir = 0; dir < 2; ++dir) {
      const bool up = dir == 1;
      if (up && P.twist)  // the two eliminations meet: x_M
        KKT_LAUNCH(c, v6_mid_kernel<KN>, kSl * P.nreal, kThr6, 0, P, 0);
      if (P.thomas) {
        // inverse-block form: no off-chain products (c = b / cy comes from v6_form_b_kernel, d = y)
      } else if (off_plain() || KN == 256) {  // 256-blocks: one small copy per slice, plain loads measured ahead
        if (up)
          KKT_LAUNCH(c, (v6_off_kernel<KN, true>), og, kThr6, off_smem<KN>(), P);
        else
          KKT_LAUNCH(c, (v6_off_kernel<KN, false>), og, kThr6, off_smem<KN>(), P);
      } else {
        static const bool ng2 = std::getenv("KKT_V6_OFF_NG2") != nullptr;  // testing: two groups per triangle pass
        static const bool off3 = std::getenv("KKT_V6_OFF3") == nullptr || std::atoi(std::getenv("KKT_V6_OFF3")) != 0;  // default on; 0: v6_off2_kernel
        bool four = false;
        if constexpr (KN <= 512) four = ngroups > 2 && !ng2;
        if (off3) {  // one 8-row tile per warp over the slice's whole k-range: no cross-warp reduction
          if constexpr (KN <= 512) {
            if (four) {
              if (up)
                KKT_LAUNCH(c, (v6_off3_kernel<KN, true, 4>), og4, kOffThr, (off3_smem<KN, 4>()), P);
              else
                KKT_LAUNCH(c, (v6_off3_kernel<KN, false, 4>), og4, kOffThr, (off3_smem<KN, 4>()), P);
            }
          }
          if (!four) {
            if (up)
              KKT_LAUNCH(c, (v6_off3_kernel<KN, true, 2>), og2, kOffThr, (off3_smem<KN, 2>()), P);
            else
              KKT_LAUNCH(c, (v6_off3_kernel<KN, false, 2>), og2, kOffThr, (off3_smem<KN, 2>()), P);
          }
        } else {
        if constexpr (KN <= 512) {
          if (four) {
            if (up)
              KKT_LAUNCH(c, (v6_off2_kernel<KN, true, 4>), og4, kOffThr, (off2_smem<KN, 4>()), P);
            else
              KKT_LAUNCH(c, (v6_off2_kernel<KN, false, 4>), og4, kOffThr, (off2_smem<KN, 4>()), P);
          }
        }
        if (!four) {
          if (up)
            KKT_LAUNCH(c, (v6_off2_kernel<KN, true, 2>), og2, kOffThr, (off2_smem<KN, 2>()), P);
          else
            KKT_LAUNCH(c, (v6_off2_kernel<KN, false, 2>), og2, kOffThr, (off2_smem<KN, 2>()), P);
        }
        }
      }
      if (up && P.thomas && P.k > 1) {  // grouped rows: the in-group passes run in place in W1, so d = y goes there
        const int64_t tot = int64_t(ngroups) * P.ny * KN * kG;
        KKT_LAUNCH(c, v6_copy_kernel, kSmCount * 8, 256, 0, tot, P.W0, P.W1);
      }
      if (up && P.twist)  // the inflow of the first outward row: d_{M-1} += H_{M-1} x_M
        KKT_LAUNCH(c, v6_mid_kernel<KN>, kSl * P.nreal, kThr6, 0, P, 1);
      for (int i = 1; i < P.k; ++i) {  // zero-inflow chains inside the groups, every group at once
        P.pass = i;
        if (up && P.rawH)
          KKT_LAUNCH(c, (v6_inner_kernel<KN, true, true>), P.ngr * npairs, kThr6, off_smem<KN>(), P);
        else if (up)
          KKT_LAUNCH(c, (v6_inner_kernel<KN, true, false>), P.ngr * npairs, kThr6, off_smem<KN>(), P);
        else if (P.thomas ? P.rawH != nullptr : P.rawG != nullptr)
          KKT_LAUNCH(c, (v6_inner_kernel<KN, false, true>), P.ngr * npairs, kThr6, off_smem<KN>(), P);
        else
          KKT_LAUNCH(c, (v6_inner_kernel<KN, false, false>), P.ngr * npairs, kThr6, off_smem<KN>(), P);
      }
      if (P.ll)  // every handoff slot of this sweep direction back to "empty", right before the chain: the
                 // slots are then L2-resident when the chain polls them (refilled a step early, from
                 // v6_form_b_kernel, they had gone cold: config 2 114 -> 127 ms)
        dev_fill(c, P.ll, 0xFF, sizeof(unsigned long long) * P.nll);
      else
        dev_fill(c, P.cnt, 0, sizeof(unsigned) * ngroups);  // counter handoff
      for (int g0 = 0; g0 < nchain_groups; g0 += gpw) {
        P.g0 = g0;
        launch_chain<KN>(c, up, P, std::min(gpw, nchain_groups - g0));
      }
      if (up && P.thomas) {  // x_0 = H_0 X_0 of both halves
        P.g0 = 0;
        KKT_LAUNCH(c, v6_mid_kernel<KN>, kSl * ngroups, kThr6, 0, P, 2);
      }
    }
    if (c->step_hook) c->step_hook(t);  // every output of step t is written (stream order)
  }
}

template <int KN>
int choose_k(int ngroups) {
  V6_DIMS
  return chain_capacity<KN>() / (kSl * std::max(1, ngroups));
}

}  // namespace

bool v6_supported(const Ctx* c) {
  static const bool off = std::getenv("KKT_SWEEP_V6_OFF") != nullptr;  // testing: sweep_fast.cu chains
  // 128 < nx <= 1023 (configs 2, 3 and 4).  P^-1 measured against v5's cluster chains:
  // config 2 181 vs 584 ms, config 3 310 vs 390 ms.  v5 stays as the KKT_SWEEP_V6_OFF=1 fallback.
  return !off && c->mode == KKT_MODE_FAST && c->ny >= 2 && c->nx <= 1024 && c->nx > 128;
}

// The block recursion D_J = T - cy^2 D_{J-1}^{-1} converges geometrically
// (factor_block.cu): from some row on, Li_J and Ui_J equal the last row's to
// rounding, so rows J >= jstar use row jstar's operators (as sweep v5 does),
// which stay in L2, and only jstar + 1 operator rows are packed.  jstar is the
// first row from which Li and Ui (and so G, H) stay within tol * max|M| of the
// last row's (KKT_V6_JTOL, default 1e-15; 0 disables); none: ny.
static int v6_find_jstar(Ctx* c, int nyv) {  // nyv: block rows the chains run over (ny, or the half chain's)
  const int nx = c->nx, ny = c->ny;
  static const char* jt = std::getenv("KKT_V6_JTOL");
  const double tol = jt ? std::atof(jt) : 1e-15;
  if (!(tol > 0.0) || ny < 3) return ny;
  DBuf<double> dev(2 * size_t(ny)), mag(2 * size_t(ny));
  KKT_LAUNCH(c, v6_conv_kernel, ny, 256, 0, c->Li.p, c->Ui.p, nx, ny, dev.p, mag.p);
  std::vector<double> hd(2 * ny), hm(2 * ny);
  KKT_CUDA(cudaMemcpyAsync(hd.data(), dev.p, sizeof(double) * 2 * ny, cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaMemcpyAsync(hm.data(), mag.p, sizeof(double) * 2 * ny, cudaMemcpyDeviceToHost, c->stream));
  KKT_CUDA(cudaStreamSynchronize(c->stream));
  int first = ny - 1;  // rows first .. ny-1 all within tol
  while (first > 0 && hd[2 * (first - 1)] <= tol * hm[2 * (ny - 1)] &&
         hd[2 * (first - 1) + 1] <= tol * hm[2 * (ny - 1) + 1])
    --first;
  const int js = first + 1;  // G_J needs Li_J and Ui_{J-1}
  return js <= nyv - 2 ? js : nyv;
}

// slot handoff instead of the release counter + bulk copy.  KKT_V6_LL=0/1 forces the choice.
static bool v6_ll_enabled() {
  static const char* ll_env = std::getenv("KKT_V6_LL");
  return ll_env ? std::atoi(ll_env) != 0 : true;
}

void build_v6(Ctx* c) {
  const int nx = c->nx, nyA = c->ny;
  // Two-sided (twisted) elimination for odd ny >= 3 (every BASELINE grid): two half-length chains
  // per spatial solve that meet in the middle block row; needs the slot handoff.  KKT_V6_TWIST=0: off.
  static const char* tw_env = std::getenv("KKT_V6_TWIST");
  const bool twist = (tw_env ? std::atoi(tw_env) != 0 : true) && v6_ll_enabled() && nyA >= 3 && (nyA & 1);
  const int ny = twist ? (nyA - 1) / 2 : nyA;  // block rows of a (half) chain: every "ny" below
  c->v6_twist = twist;
  c->v6_nyv = ny;
  c->v6_jstar = v6_find_jstar(c, ny);
  const int nops = std::min(ny, c->v6_jstar + 1);  // packed operator rows
  if (std::getenv("KKT_V6_TIM")) std::fprintf(stderr, "v6 jstar %d of ny %d\n", c->v6_jstar, ny);
  const int kn = nx <= 255 ? 256 : nx <= 511 ? 512 : 1024;
  const size_t mat = size_t(kn) * kn, nn = size_t(nx) * nx;
  c->v6_kn = kn;
  c->v6_nops = nops;
  c->v6_ops.alloc(4 * size_t(nops) * mat);
  double* Lp = c->v6_ops.p;
  double* Up = Lp + nops * mat;
  double* Gp = Up + nops * mat;
  double* Hp = Gp + nops * mat;
  auto pk = [&](const double* src, int nJ, double scale, double* dst) {
    if (kn == 256)
      pack<256>(c, src, nJ, scale, dst);
    else if (kn == 512)
      pack<512>(c, src, nJ, scale, dst);
    else
      pack<1024>(c, src, nJ, scale, dst);
  };
  pk(c->Li.p, nops, 1.0, Lp);
  pk(c->Ui.p, nops, 1.0, Up);
  KKT_CUDA(cudaMemsetAsync(Gp, 0, sizeof(double) * mat, c->stream));  // G_0: unused
  if (nops == ny && !twist)
    KKT_CUDA(cudaMemsetAsync(Hp + size_t(ny - 1) * mat, 0, sizeof(double) * mat, c->stream));  // H_{ny-1}
  // H_J rows computed (twisted: H_{M-1} exists and carries x_M into the first outward row)
  const int nh = twist ? nops : std::min(nops, ny - 1);
  const int Jb = std::max(1, std::min(ny - 1, 32));
  DBuf<double> T(size_t(Jb) * nn);
  for (int J0 = 1; J0 < nops; J0 += Jb) {  // G_J = cy Li_J Ui_{J-1}
    const int nb = std::min(Jb, nops - J0);
    GemmArgs g{c->Li.p + J0 * nn, c->Ui.p + (J0 - 1) * nn, T.p, nx, nx, nx,
               int64_t(nn), int64_t(nn), int64_t(nn), nx, nx, nx};
    gemm_f64(c, g, nb);
    pk(T.p, nb, c->cy, Gp + J0 * mat);
  }
  for (int J0 = 0; J0 < nh; J0 += Jb) {  // H_J = cy Ui_J Li_J
    const int nb = std::min(Jb, nh - J0);
    GemmArgs g{c->Ui.p + J0 * nn, c->Li.p + J0 * nn, T.p, nx, nx, nx,
               int64_t(nn), int64_t(nn), int64_t(nn), nx, nx, nx};
    gemm_f64(c, g, nb);
    pk(T.p, nb, c->cy, Hp + J0 * mat);
  }
  KKT_CUDA(cudaStreamSynchronize(c->stream));  // T is freed on return
  static const double bfrac = std::getenv("KKT_V6_BFRAC") ? std::atof(std::getenv("KKT_V6_BFRAC")) : 0.65;  // tuning
  auto make_band = [&](const double* packed, int rows, int2* out, int2* raw) {
    static const char* bt = std::getenv("KKT_V6_BTOL");
    const double tol = bt ? std::atof(bt) : 1e-17;
    if (kn == 256)
      KKT_LAUNCH(c, v6_band_kernel<256>, rows, 256, 0, packed, tol, out, raw);
    else if (kn == 512)
      KKT_LAUNCH(c, v6_band_kernel<512>, rows, 256, 0, packed, tol, out, raw);
    else
      KKT_LAUNCH(c, v6_band_kernel<1024>, rows, 256, 0, packed, tol, out, raw);
  };
  const int ksl = kn / 16;
  c->v6_band.alloc(size_t(2) * nops * ksl);  // k == 1: the windows of G and H
  c->v6_raw.alloc(size_t(4) * nops * ksl);   // raw ranges of Li, Ui, G, H
  make_band(Lp, nops, nullptr, c->v6_raw.p);
  make_band(Up, nops, nullptr, c->v6_raw.p + size_t(nops) * ksl);
  make_band(Gp, nops, c->v6_band.p, c->v6_raw.p + size_t(2) * nops * ksl);
  make_band(Hp, nops, c->v6_band.p + size_t(nops) * ksl, c->v6_raw.p + size_t(3) * nops * ksl);
  // the windowed product has a runtime trip count; it only pays where the band is clearly narrower
  // than the row (config 2: 55% of the k-steps; config 3: 84%, the config-4 slab: 90%, where the
  // windowed and range-cut kernels measured slower than the fixed ones)
  auto windows_pay = [&](const int2* dev, size_t n) {
    std::vector<int2> h(n);
    KKT_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(int2) * n, cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    double sum = 0.0;
    int wmax = 2;
    for (const int2& w : h) {
      sum += w.y;
      wmax = std::max(wmax, w.y);
    }
    c->v6_wmax = wmax;
    const double frac = sum / (double(n) * (kn / 32));
    // the windowed chain keeps only the window in shared memory (v6_chainw_kernel), twice for the
    // slots; it must leave room for as many CTAs per SM as the full-row kernel runs with
    const size_t wsm = kn == 256 ? chainw_smem<256>(wmax) : kn == 512 ? chainw_smem<512>(wmax) : chainw_smem<1024>(wmax);
    const size_t fsm = kn <= 512 ? size_t(113) << 10 : size_t(226) << 10;  // 2 CTAs per SM / 1 CTA per SM
    if (std::getenv("KKT_V6_TIM"))
      std::fprintf(stderr, "v6 band windows: %.0f%% of the k-steps, widest %d k-steps per warp (%zu KB shared)\n", 100.0 * frac, wmax,
                   wsm >> 10);
    // KKT_V6_CFRAC (tuning): the chain's own threshold (default: the common one)
    static const double cfrac = std::getenv("KKT_V6_CFRAC") ? std::atof(std::getenv("KKT_V6_CFRAC")) : bfrac;
    return frac < cfrac && wsm <= fsm;
  };
  c->v6_band_on = windows_pay(c->v6_band.p, size_t(2) * nops * ksl);
  {  // the raw ranges likewise: k-steps kept, relative to the triangle (Li, Ui) or the full row (G, H)
    std::vector<int2> h(size_t(4) * nops * ksl);
    KKT_CUDA(cudaMemcpyAsync(h.data(), c->v6_raw.p, sizeof(int2) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    const int kks = kn / 4;
    for (int set = 0; set < 4; ++set) {
      double kept = 0.0, full = 0.0;
      for (int r = 0; r < nops; ++r)
        for (int sl = 0; sl < ksl; ++sl) {
          const int2 b = h[(size_t(set) * nops + r) * ksl + sl];
          int lo = set == 1 ? 4 * sl : 0, hi = set == 0 ? 4 * sl + 4 : kks;  // set 0: Li (lower), 1: Ui (upper)
          full += hi - lo;
          kept += std::max(0, std::min(hi, b.y) - std::max(lo, b.x));
        }
      c->v6_raw_on[set] = kept < bfrac * full;
      if (std::getenv("KKT_V6_TIM"))
        std::fprintf(stderr, "v6 band of %s: %.0f%% of the k-steps\n", set == 0 ? "Li" : set == 1 ? "Ui" : set == 2 ? "G" : "H",
                     100.0 * kept / std::max(1.0, full));
    }
  }

  if (twist) {  // the middle block row: Dm^{-1} and E = cy Dm^{-1} Ui_{M-1}, packed like the operator rows
    DBuf<double> Dinv(nn), E(nn), E2(nn);
    build_twist_middle(c, ny, Dinv.p, E.p, E2.p);
    c->v6_mid.alloc(3 * mat);
    pk(Dinv.p, 1, 1.0, c->v6_mid.p);
    pk(E.p, 1, 1.0, c->v6_mid.p + mat);
    pk(E2.p, 1, 1.0, c->v6_mid.p + 2 * mat);
    // the inverse-block form (V6Params::thomas) is the default with the twisted elimination; KKT_V6_THOMAS=0: L/U factors
    static const bool th_env = std::getenv("KKT_V6_THOMAS") == nullptr || std::atoi(std::getenv("KKT_V6_THOMAS")) != 0;
    c->v6_thomas = th_env;
    KKT_CUDA(cudaStreamSynchronize(c->stream));  // the temporaries are freed here
    if (std::getenv("KKT_V6_TIM")) std::fprintf(stderr, "v6 twisted elimination: %d rows per half chain, middle row %d\n", ny, ny);
  }

  // ---- k-row grouping: as many rows per handoff as co-resident CTAs allow for the RASQ chains
  // (KKT_V6_K overrides; 1 = the plain row-by-row chain)
  const int rasq_groups = (std::max(1, c->ndl) + kG - 1) / kG;
  int k = kn == 256 ? choose_k<256>(rasq_groups) : kn == 512 ? choose_k<512>(rasq_groups) : choose_k<1024>(rasq_groups);
  k = std::min(k, 8);
  if (const char* e = std::getenv("KKT_V6_K")) k = std::atoi(e);
  k = std::max(1, std::min(k, ny));
  c->v6_k = k;
  if (k == 1) return;
  const int js = c->v6_jstar;               // rows >= js share row js's operators (ny: none)
  const int ngr = (ny + k - 1) / k;
  // L groups [0, nind) are built row by row, groups >= nind (all rows >= js) share one converged set;
  // U groups (from the top) [0, gconv) share the converged set, the rest are built row by row
  const int jsl = c->v6_thomas ? js + 1 : js;  // inverse-block form: L row J applies H_{J-1}, converged from row js + 1 on
  const int nind = jsl >= ny ? ngr : std::min(ngr, (jsl + k - 1) / k);
  const int gconv = js >= ny ? 0 : std::min(ngr, (ny - js) / k);
  c->v6_nind = nind;
  c->v6_gconv = gconv;
  c->v6_nphi = nind * k + k;
  c->v6_npsi = k + (ngr - gconv) * k;
  c->v6_phi.alloc(size_t(c->v6_nphi + c->v6_npsi) * mat);
  KKT_CUDA(cudaMemsetAsync(c->v6_phi.p, 0, sizeof(double) * c->v6_phi.n, c->stream));
  double* Phi = c->v6_phi.p;
  double* Psi = Phi + size_t(c->v6_nphi) * mat;
  auto opr = [&](int J) { return J < js ? J : js; };
  // unpacked scaled G_J (J >= 1) and H_J (J <= ny - 2) for the operator rows in use
  DBuf<double> Gu(size_t(nops) * nn), Hu(size_t(nops) * nn), Pu(size_t(k) * nn);
  KKT_CUDA(cudaMemsetAsync(Gu.p, 0, sizeof(double) * nn, c->stream));
  {
    GemmArgs g{c->Li.p + nn, c->Ui.p, Gu.p + nn, nx, nx, nx, int64_t(nn), int64_t(nn), int64_t(nn), nx, nx, nx};
    if (nops > 1) gemm_f64(c, g, nops - 1);
    GemmArgs h{c->Ui.p, c->Li.p, Hu.p, nx, nx, nx, int64_t(nn), int64_t(nn), int64_t(nn), nx, nx, nx};
    gemm_f64(c, h, nh);
    if (nh < nops) KKT_CUDA(cudaMemsetAsync(Hu.p + size_t(nh) * nn, 0, sizeof(double) * nn * (nops - nh), c->stream));
    const int64_t tot = int64_t(nops) * nn;
    KKT_LAUNCH(c, v6_scale_kernel, kSmCount * 8, 256, 0, tot, c->cy, Gu.p);
    KKT_LAUNCH(c, v6_scale_kernel, kSmCount * 8, 256, 0, tot, c->cy, Hu.p);
  }
  // one group's propagators: P_0 = M_{J(0)}, P_i = M_{J(i)} P_{i-1}; packed to dst[i]
  // Inverse-block form: row J's operator is H_{J-1} (L) / H_{J+1} (U) instead of G_J / H_J
  const bool th = c->v6_thomas;
  auto build_group = [&](const double* Mu, auto rowof, double* dst, int shift) {
    for (int i = 0; i < k; ++i) {
      const int J = rowof(i);
      if (J < 0 || J >= ny) break;
      const double* M = Mu + size_t(opr(std::max(0, J + shift))) * nn;
      if (i == 0) {
        KKT_CUDA(cudaMemcpyAsync(Pu.p, M, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c->stream));
      } else {
        GemmArgs g{M, Pu.p + size_t(i - 1) * nn, Pu.p + size_t(i) * nn, nx, nx, nx, 0, 0, 0, nx, nx, nx};
        gemm_f64(c, g, 1);
      }
      pk(Pu.p + size_t(i) * nn, 1, 1.0, dst + size_t(i) * mat);
    }
  };
  const double* GL = th ? Hu.p : Gu.p;
  const int sl = th ? -1 : 0, su = th ? 1 : 0;
  for (int gr = 1; gr < nind; ++gr)  // group 0 has no inflow
    build_group(GL, [&](int i) { return gr * k + i; }, Phi + size_t(gr) * k * mat, sl);
  if (nind < ngr) build_group(GL, [&](int i) { (void)i; return jsl; }, Phi + size_t(nind) * k * mat, sl);
  if (gconv > 0) build_group(Hu.p, [&](int i) { (void)i; return js; }, Psi, 0);
  for (int gr = std::max(1, gconv); gr < ngr; ++gr)
    build_group(Hu.p, [&](int i) { return ny - 1 - gr * k - i; }, Psi + size_t(k + (gr - gconv) * k) * mat, su);
  c->v6_band.alloc(size_t(c->v6_nphi + c->v6_npsi) * ksl);  // k > 1: the windows of the propagator sets
  make_band(Phi, c->v6_nphi, c->v6_band.p, nullptr);
  make_band(Psi, c->v6_npsi, c->v6_band.p + size_t(c->v6_nphi) * ksl, nullptr);
  c->v6_band_on = windows_pay(c->v6_band.p, size_t(c->v6_nphi + c->v6_npsi) * ksl);
  KKT_CUDA(cudaStreamSynchronize(c->stream));  // the temporaries are freed on return
  if (std::getenv("KKT_V6_TIM"))
    std::fprintf(stderr, "v6 grouping k %d: %d groups, L own %d, U converged %d\n", k, ngr, nind, gconv);
}

void v6_chains(Ctx* c, const FastStep* jobs_dev, int nchains, int nsteps, bool coarse_terms) {
  const bool twist = c->v6_twist;
  const int ny = c->v6_nyv;  // block rows of a (half) chain
  const int kn = c->v6_kn;
  const size_t mat = size_t(kn) * kn;
  const int nreal = (nchains + kG - 1) / kG;
  const int ngroups = twist ? 2 * nreal : nreal;  // (virtual) chain groups of the block vectors
  const size_t need = size_t(ngroups) * ny * kn * kG;
  const size_t midv = twist ? size_t(2) * nreal * kn * kG : 0;  // b_M and x_M
  if (c->v6_w.n < 2 * need + midv || c->v6_cnt.n < size_t(ngroups)) {
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    c->v6_w.alloc(2 * need + midv);
    c->v6_cnt.alloc(ngroups);
  }
  V6Params P;
  const int nops = c->v6_nops;
  P.Lp = c->v6_ops.p;
  P.Up = P.Lp + nops * mat;
  P.Gp = P.Up + nops * mat;
  P.Hp = P.Gp + nops * mat;
  P.jstar = c->v6_jstar;
  P.W0 = c->v6_w.p;
  P.W1 = c->v6_w.p + need;
  P.jobs = jobs_dev;
  P.nsteps = nsteps;
  P.nx = c->nx;
  P.ny = ny;
  P.nchains = nchains;
  P.ngroups = ngroups;
  P.twist = twist ? 1 : 0;
  P.wmax = c->v6_wmax;
  {
    static const int spin = std::getenv("KKT_V6_SPIN_NS") ? std::atoi(std::getenv("KKT_V6_SPIN_NS")) : 0;
    P.spin_ns = spin;
    static const int stag = std::getenv("KKT_V6_STAGGER") ? std::atoi(std::getenv("KKT_V6_STAGGER")) : 0;
    P.stagger = stag;
    static const bool nohold = std::getenv("KKT_V6_NOHOLD") != nullptr;
    P.nohold = nohold ? 1 : 0;
  }
  P.nyA = c->ny;
  P.nreal = nreal;
  P.Wm = c->v6_w.p + 2 * need;
  P.Dm = twist ? c->v6_mid.p : nullptr;
  P.Em = twist ? c->v6_mid.p + mat : nullptr;
  P.a1 = c->a1.p;
  P.a2 = c->a2.p;
  P.gam = c->gam.p;
  P.inv_ms = 1.0 / c->ms;
  P.coarse = coarse_terms ? 1 : 0;
  P.cnt = c->v6_cnt.p;
  P.k = c->v6_k;
  P.ngr = (ny + P.k - 1) / P.k;
  const bool ll_on = v6_ll_enabled();
  P.ll = nullptr;
  P.nll = 0;
  {
    static const bool np = std::getenv("KKT_V6_NOPOLL") != nullptr;
    P.nopoll = np ? 1 : 0;
  }
  if (ll_on) {
    const size_t npk = size_t(ngroups) * P.ngr * kn * kG;
    if (c->v6_ll.n < npk) {
      KKT_CUDA(cudaStreamSynchronize(c->stream));
      c->v6_ll.alloc(npk);
    }
    P.ll = c->v6_ll.p;
    P.nll = npk;
  }
  P.nind = c->v6_nind;
  P.gconv = c->v6_gconv;
  P.pass = 0;
  P.Phi = P.k == 1 ? P.Gp : c->v6_phi.p;
  P.Psi = P.k == 1 ? P.Hp : c->v6_phi.p + size_t(c->v6_nphi) * mat;
  static const bool band_off = std::getenv("KKT_V6_NOBAND") != nullptr;  // testing: full rows
  {
    const size_t rs = size_t(nops) * (kn / 16);
    P.rawL = (band_off || !c->v6_raw_on[0]) ? nullptr : c->v6_raw.p;
    P.rawU = (band_off || !c->v6_raw_on[1]) ? nullptr : c->v6_raw.p + rs;
    P.rawG = (band_off || !c->v6_raw_on[2]) ? nullptr : c->v6_raw.p + 2 * rs;
    P.rawH = (band_off || !c->v6_raw_on[3]) ? nullptr : c->v6_raw.p + 3 * rs;
  }
  const bool win = !band_off && c->v6_band_on;
  P.bandPhi = win ? c->v6_band.p : nullptr;
  P.bandPsi = win ? c->v6_band.p + size_t(P.k == 1 ? nops : c->v6_nphi) * (kn / 16) : nullptr;
  {  // the inverse-block form (see V6Params::thomas): H is the only operator set, no off-chain products
    static const bool th_env = std::getenv("KKT_V6_THOMAS") == nullptr || std::atoi(std::getenv("KKT_V6_THOMAS")) != 0;  // default on; 0: the L/U form
    (void)th_env;
    P.thomas = (c->v6_thomas && twist && ll_on) ? 1 : 0;  // decided at setup (build_v6): the grouped propagators follow it
    P.inv_cy = 1.0 / c->cy;
    if (P.thomas) {
      if (P.k == 1) {
        P.Phi = P.Psi = P.Hp;
        P.bandPhi = P.bandPsi;
      }
      P.Em = c->v6_mid.p + 2 * mat;
    }
  }
  static const bool dbg = std::getenv("KKT_V6_TIM") != nullptr;
  DBuf<long long> tim;
  P.tim = nullptr;
  if (dbg) {
    tim.alloc(12 + 1024);
    KKT_CUDA(cudaMemsetAsync(tim.p, 0xFF, sizeof(long long) * (12 + 1024), c->stream));
    KKT_CUDA(cudaMemsetAsync(tim.p, 0, sizeof(long long) * 12, c->stream));
    P.tim = tim.p;
  }
  if (dbg) std::fprintf(stderr, "v6 elimination form: %s\n", P.thomas ? "inverse blocks (no off-chain products)" : "L/U factors");
  c->tbegin(3);
  if (kn == 256)
    run_steps<256>(c, P, nsteps, ngroups);
  else if (kn == 512)
    run_steps<512>(c, P, nsteps, ngroups);
  else
    run_steps<1024>(c, P, nsteps, ngroups);
  c->tend(3);
  if (dbg) {
    static long long h[12 + 1024];
    KKT_CUDA(cudaMemcpyAsync(h, tim.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KKT_CUDA(cudaStreamSynchronize(c->stream));
    {  // chain CTAs per SM, and how many co-resident pairs come from different halves of the groups
      int ncta = 0;
      while (ncta < 1024 && h[12 + ncta] >= 0) ++ncta;
      if (ncta > 0) {
        const int per_g = ncta / std::max(1, nreal);
        int same = 0, diff = 0, alone = 0;
        for (int a = 0; a < ncta; ++a) {
          int mate = -1;
          for (int b = 0; b < ncta; ++b)
            if (b != a && h[12 + b] == h[12 + a]) mate = b;
          if (mate < 0) ++alone;
          else if ((2 * (a / per_g) >= nreal) != (2 * (mate / per_g) >= nreal)) ++diff;
          else ++same;
        }
        std::fprintf(stderr, "v6 chain placement: %d CTAs, alone on their SM %d, paired across the halves %d, paired inside a half %d; CTA 0..3 on SM %lld %lld %lld %lld, CTA 148 on SM %lld\n",
                     ncta, alone, diff, same, h[12], h[13], h[14], h[15], ncta > 148 ? h[12 + 148] : -1LL);
      }
    }
    const double rows = double(ny - 1) * nsteps;
    for (int u = 0; u < 2; ++u)
      std::fprintf(stderr, "v6 %s cycles/row (middle slice of group 0): poll %.0f waitA %.0f waitB %.0f mma %.0f emit %.0f signal %.0f\n",
                   u ? "U" : "L", h[6 * u] / rows, h[6 * u + 1] / rows, h[6 * u + 2] / rows, h[6 * u + 3] / rows,
                   h[6 * u + 4] / rows, h[6 * u + 5] / rows);
  }
}

}  // namespace kkt
