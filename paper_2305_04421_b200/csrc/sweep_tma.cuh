// sweep_tma.cuh — shared device helpers of the TMA-staged blocked sweeps
// (sweep_tma.cu: one CTA per chain; sweep_group.cu: group-parallel).
#pragma once

#include "sweep.cuh"

namespace kkt {
namespace tma {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxNx = 128;
constexpr int kK = kMaxNx / 32;        // column registers per lane
constexpr int kR = kMaxNx / kWarps;    // rows per warp
constexpr int kLogR = kR == 16 ? 4 : kR == 8 ? 3 : kR == 4 ? 2 : kR == 2 ? 1 : 0;
static_assert((1 << kLogR) == kR, "rows per warp must be a power of two");
// row a = warp + kWarps*r lies in column chunk (kWarps*r)/32 for every warp
static_assert(kWarps <= 32 && 32 % kWarps == 0, "chunk of a row must be warp-independent");
__host__ __device__ constexpr int chunk_of(int r) { return (kWarps * r) / 32; }
constexpr int kSlots = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// TMA bulk copy global -> shared, completion counted on `bar` (one
// expect_tx for the total; splitting into 16 KB pieces measured 5% slower).
__device__ __forceinline__ void tma_load(double* dst, const double* src, uint32_t bytes,
                                         uint64_t* bar) {
  constexpr uint32_t kPiece = 1u << 20;  // one request per copy (pieces measured slower)
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  for (uint32_t off = 0; off < bytes; off += kPiece) {
    const uint32_t len = bytes - off < kPiece ? bytes - off : kPiece;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(reinterpret_cast<char*>(dst) + off)),
        "l"(reinterpret_cast<const char*>(src) + off), "r"(len), "r"(smem_u32(bar))
        : "memory");
  }
}

__device__ __forceinline__ int zig(long q, int ny) {
  if (ny == 1) return 0;
  const long P = 2L * (ny - 1);
  const int r = int(q % P);
  return r < ny ? r : int(P - r);
}

// Row a = warp + kWarps*r of the packed triangle starts at a(a+1)/2; its
// column chunk k (b = 32k + lane) is entirely below the diagonal for
// k < chunk_of(r) and straddles it for k == chunk_of(r), so the
// chunk loops have compile-time bounds and only the diagonal chunk is
// predicated.  `roff[r]` = (a(a+1)/2 + lane), precomputed per thread.
__device__ __forceinline__ void row_offsets(int (&roff)[kR]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int a = warp + kWarps * r;
    roff[r] = (a * (a + 1)) / 2 + lane;
  }
}

// Reduce the kR per-row partial sums of a warp (rows a = warp + kWarps*r)
// across its 32 lanes with a transpose-reduction (one halving shuffle step per
// row-index bit, then plain butterflies) and store row sums to out[a].
__device__ __forceinline__ void rows_reduce_store(double (&s)[kR], double* out, int nx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int step = 0; step < kLogR; ++step) {
    const int o = 16 >> step, n = kR >> step;
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const double keep = hi ? s[i + n / 2] : s[i];
      const double send = hi ? s[i] : s[i + n / 2];
      s[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 >> kLogR; o >= 1; o >>= 1) s[0] += __shfl_xor_sync(0xffffffffu, s[0], o);
  int r = 0;
#pragma unroll
  for (int step = 0; step < kLogR; ++step) r |= ((lane >> (4 - step)) & 1) << (kLogR - 1 - step);
  const int a = warp + kWarps * r;
  if ((lane & ((32 >> kLogR) - 1)) == 0 && a < nx) out[a] = s[0];
}

// out[a] = sum_b M[a*ld + b] v[b] for a dense nx x nx matrix (global or shared)
__device__ __forceinline__ void dense_mv(const double* __restrict__ M, int ld,
                                         const double (&vr)[kK], double* out, int nx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int a = warp + kWarps * r;
    double acc = 0.0;
    if (a < nx) {
      const double* row = M + int64_t(a) * ld;
#pragma unroll
      for (int k = 0; k < kK; ++k) {
        const int b = lane + 32 * k;
        if (b < nx) acc = fma(row[b], vr[k], acc);
      }
    }
    s[r] = acc;
  }
  rows_reduce_store(s, out, nx);
}

// out[a] = sum_{b<=a} L[a][b] v[b], v in lane registers (vr[k] = v[lane+32k]).
// All 16 rows of a warp are in flight; the partial sums are reduced across
// the warp with a transpose-reduction (16 shuffles instead of 16 x 5).
__device__ __forceinline__ void lower_mv(const double* __restrict__ L, const int (&roff)[kR],
                                         const double (&vr)[kK], double* out, int nx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int a = warp + kWarps * r;
    double acc = 0.0;
    if (a < nx) {  // warp-uniform
      const double* row = L + roff[r];
#pragma unroll
      for (int k = 0; k < chunk_of(r); ++k) acc = fma(row[32 * k], vr[k], acc);
      if (lane + 32 * chunk_of(r) <= a) acc = fma(row[32 * chunk_of(r)], vr[chunk_of(r)], acc);
    }
    s[r] = acc;
  }
  rows_reduce_store(s, out, nx);
}

// out[b] = sum_{a>=b} L[a][b] w_a with w_a = D^{-1}_a (base[a] + cy * add[a])
// (add == nullptr: w_a = D^{-1}_a base[a]).  Per-lane column accumulators,
// rows split over warps, partials reduced through `part`.  Ends with the
// outputs written (caller syncs before reading them).
__device__ __forceinline__ void lowerT_mv(const double* __restrict__ L, const int (&roff)[kR],
                                          const double* dinv, const double* base,
                                          const double* add, double cy, double* part,
                                          double* out, int nx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[kK];
#pragma unroll
  for (int k = 0; k < kK; ++k) acc[k] = 0.0;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int a = warp + kWarps * r;
    if (a < nx) {
      const double* row = L + roff[r];
      const double wa = dinv[a] * (add ? fma(cy, add[a], base[a]) : base[a]);
#pragma unroll
      for (int k = 0; k < chunk_of(r); ++k) acc[k] = fma(row[32 * k], wa, acc[k]);
      if (lane + 32 * chunk_of(r) <= a) acc[chunk_of(r)] = fma(row[32 * chunk_of(r)], wa, acc[chunk_of(r)]);
    }
  }
#pragma unroll
  for (int k = 0; k < kK; ++k) part[warp * kMaxNx + lane + 32 * k] = acc[k];
  __syncthreads();
  for (int b = threadIdx.x; b < nx; b += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < kWarps; ++w2) s += part[w2 * kMaxNx + b];
    out[b] = s;
  }
}

// vr[k] = base[b] (+ cy * add[b]), b = lane + 32k
__device__ __forceinline__ void load_vr(const double* base, const double* add, double cy,
                                        double (&vr)[kK], int nx) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    const int b = lane + 32 * k;
    vr[k] = b < nx ? (add ? fma(cy, add[b], base[b]) : base[b]) : 0.0;
  }
}


}  // namespace tma
}  // namespace kkt
