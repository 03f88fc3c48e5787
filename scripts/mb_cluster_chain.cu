// mb_cluster_chain.cu — microbenchmark for the sweep-v4 design question:
// per-step latency of the block recurrence y_J = c_J + G_J y_{J-1}
// (G_J dense 128x128, 16 chains) when the rows of each step are split over
// an 8-CTA cluster (16 rows per CTA, fp64 mma.sync m8n8k4), G_J row slices
// are TMA-streamed from L2, and the step result is exchanged through DSMEM
// bulk copies (cp.async.bulk shared::cta -> shared::cluster, mbarrier tx).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb scripts/mb_cluster_chain.cu
//   /tmp/mb   -> prints us/step for a few configurations and the max error
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));          \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

constexpr int kN = 128;          // padded block size
constexpr int kC = 16;           // chains
constexpr int kCl = 8;           // CTAs per cluster
constexpr int kRows = kN / kCl;  // 16 rows per CTA
constexpr int kSlice = kRows * kN;  // doubles per matrix slice (16 KB)
constexpr int kXs = kN * kC;        // doubles per exchange buffer (16 KB)
constexpr int kRing = 3;
constexpr int kThr = 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
  }
}
__device__ __forceinline__ void tma_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void s2peer(uint32_t dst_cluster, const void* src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   dst_cluster),
               "r"(su32(src)), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// exchange-buffer layout [ks 32][ct 2][kl 4][nl 8]: rows k = 4ks+kl, chain n = 8ct+nl.
// B fragment (b = B[k = lane%4][n = lane/4]) -> index ks*64 + ct*32 + (lane%4)*8 + lane/4.
// D fragment pairs (chains 8ct + 2(lane%4) + {0,1}) are contiguous.
__device__ __forceinline__ int xidx(int k, int n) { return (k >> 2) * 64 + (n >> 3) * 32 + (k & 3) * 8 + (n & 7); }

struct Params {
  const double* G;   // [J][r][ks 32][rt 2][lane 32] fragment-ordered slices
  const double* c;   // [J][k 128][n 16]
  double* y;         // [J][k 128][n 16]
  int g, ny;
  int reps;
  long long* T;      // per-CTA cycle breakdown (thread 0)
  int skip;          // 1: no DMMA, 2: no exchange wait/send
};

template <int kMode>  // 0: DSMEM bulk exchange, 1: cluster barrier + ld.shared::cluster pulls, 2: st.async pushes
__global__ void __launch_bounds__(kThr, 1) chain_kernel(Params P) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                               // kRing slices
  double* X = ring + kRing * kSlice;               // 2 exchange buffers
  double* part = X + 2 * kXs;                      // 4 tiles x 32 lanes x 2
  __shared__ __align__(8) uint64_t tbar[kRing];
  __shared__ __align__(8) uint64_t xbar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = int(ctarank());
  const int grp = blockIdx.x / kCl;
  const int J0 = grp * P.g;
  const int len = min(P.g, P.ny - J0);
  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&tbar[i], 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cluster_sync();
  const int t = warp & 3, rt = t >> 1, ct = t & 1, kh = warp >> 2;
  uint32_t tph[kRing] = {0, 0, 0};
  uint32_t xph[2] = {0, 0};
  int issued = 0;  // TMA slices issued (global count over reps)
  const int total = P.reps * len;
  auto issue = [&](int s) {  // s = global step counter
    if (tid == 0 && s < total) {
      const int q = s % len;
      mbar_expect(&tbar[s % kRing], kSlice * 8);
      tma_g2s(ring + (s % kRing) * kSlice, P.G + (size_t(J0 + q) * kCl + r) * kSlice, kSlice * 8, &tbar[s % kRing]);
    }
  };
  for (; issued < kRing - 1; ++issued) issue(issued);
  if (kMode != 1 && tid == 0) {
    mbar_expect(&xbar[0], (kCl - 1) * kRows * kC * 8);
    mbar_expect(&xbar[1], (kCl - 1) * kRows * kC * 8);
  }
  int sglob = 0;
  for (int rep = 0; rep < P.reps; ++rep) {
    for (int q = 0; q < len; ++q, ++sglob) {
      const int J = J0 + q;
      issue(issued++);
      const int slot = sglob % kRing;
      double cv0 = 0.0, cv1 = 0.0;
      {
        const int k = r * kRows + rt * 8 + (lane >> 2);
        const int n = ct * 8 + 2 * (lane & 3);
        if (kh == 0) {
          const double2 cc = *reinterpret_cast<const double2*>(P.c + size_t(J) * kN * kC + k * kC + n);
          cv0 = cc.x;
          cv1 = cc.y;
        }
      }
      long long c0 = clock64();
      mbar_wait(&tbar[slot], tph[slot]);
      long long c1 = clock64(), c2 = c1;
      tph[slot] ^= 1;
      const double* A = ring + slot * kSlice;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      if (q > 0) {
        const int xb = (q - 1) & 1;
        if (kMode != 1 && P.skip != 2) {
          mbar_wait(&xbar[xb], xph[xb]);
          xph[xb] ^= 1;
        }
        c2 = clock64();
        const double* Xb = X + xb * kXs;
        double f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int i = 0; i < (P.skip == 1 ? 0 : 16); i += 4) {
          const int ks = kh * 16 + i;
          double a[4], b[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            a[u] = A[((ks + u) * 2 + rt) * 32 + lane];
            b[u] = Xb[(ks + u) * 64 + ct * 32 + (lane & 3) * 8 + (lane >> 2)];
          }
          dmma(d0, d1, a[0], b[0]);
          dmma(e0, e1, a[1], b[1]);
          dmma(f0, f1, a[2], b[2]);
          dmma(g0, g1, a[3], b[3]);
        }
        d0 += e0 + (f0 + g0);
        d1 += e1 + (f1 + g1);
        if (kh == 1) {
          part[(t * 32 + lane) * 2] = d0;
          part[(t * 32 + lane) * 2 + 1] = d1;
        }
      }
      __syncthreads();  // partials visible; all reads of X[(q-1)&1] and ring slot done
      long long c3 = clock64();
      if (tid == 0 && kMode != 1 && q > 0 && P.skip != 2) {
        // re-arm the buffer just consumed for its next use (peers write it only
        // after they have our next slice, which we send below)
        mbar_expect(&xbar[(q - 1) & 1], (kCl - 1) * kRows * kC * 8);
      }
      if (kh == 0) {
        if (q > 0) {
          d0 += part[(t * 32 + lane) * 2];
          d1 += part[(t * 32 + lane) * 2 + 1];
        }
        const int k = r * kRows + rt * 8 + (lane >> 2);
        const int n = ct * 8 + 2 * (lane & 3);
        const double y0 = d0 + cv0, y1 = d1 + cv1;
        double* yj = P.y + size_t(J) * kN * kC + k * kC + n;
        *reinterpret_cast<double2*>(yj) = make_double2(y0, y1);
        if (kMode == 2 && q + 1 < len && P.skip != 2) {
          const uint32_t loc = su32(X + (q & 1) * kXs + xidx(k, n));
          const uint32_t bl = su32(&xbar[q & 1]);
#pragma unroll
          for (int p = 1; p < kCl; ++p) {
            const uint32_t peer = (uint32_t(r) + p) % kCl;
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                             mapa(loc, peer)),
                         "d"(y0), "d"(y1), "r"(mapa(bl, peer))
                         : "memory");
          }
        }
        double2* xs = reinterpret_cast<double2*>(X + (q & 1) * kXs + xidx(k, n));
        *xs = make_double2(y0, y1);
      }
      if (q + 1 < len && P.skip != 2) {
        if (kMode == 2) {
        } else if (kMode == 0) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncthreads();
          if (tid == 0) {
            const double* src = X + (q & 1) * kXs + r * (kRows / 4) * 64;
            for (int p = 1; p < kCl; ++p) {
              const uint32_t peer = (uint32_t(r) + p) % kCl;
              s2peer(mapa(su32(src), peer), src, kRows * kC * 8, mapa(su32(&xbar[q & 1]), peer));
            }
          }
        } else {
          cluster_sync();  // every slice of y_J is in its owner's X[q&1]
          // pull the peers' slices into the local buffer
          double* dst = X + (q & 1) * kXs;
          for (int i = tid; i < kXs / 2; i += kThr) {
            const int e = 2 * i;
            const int owner = (e / 64) / (kRows / 4);
            if (owner == r) continue;
            const uint32_t ra = mapa(su32(dst + e), owner);
            double v0, v1;
            asm volatile("ld.shared::cluster.v2.f64 {%0,%1}, [%2];\n" : "=d"(v0), "=d"(v1) : "r"(ra));
            dst[e] = v0;
            dst[e + 1] = v1;
          }
          __syncthreads();
          cluster_sync();  // nobody overwrites a slice a peer is still pulling
        }
      }
      if (tid == 0) {
        long long c4 = clock64();
        long long* T = P.T + blockIdx.x * 4;
        T[0] += c1 - c0;
        T[1] += c2 - c1;
        T[2] += c3 - c2;
        T[3] += c4 - c3;
      }
    }
    cluster_sync();  // next rep's first exchange must not overwrite buffers still read here
  }
  cluster_sync();
}

int main() {
  const int ny = 128, g = 8, NG = ny / g;
  // host data: G_J with spectral norm < 1 (random / (2 sqrt N)), c random
  std::vector<double> G(size_t(ny) * kN * kN), c(size_t(ny) * kN * kC);
  uint64_t s = 12345;
  auto rnd = [&]() {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return double((s >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
  };
  for (auto& v : G) v = rnd() / std::sqrt(double(kN));
  for (auto& v : c) v = rnd();
  // fragment-ordered slices
  std::vector<double> Gf(G.size());
  for (int J = 0; J < ny; ++J)
    for (int r = 0; r < kCl; ++r)
      for (int ks = 0; ks < 32; ++ks)
        for (int rt = 0; rt < 2; ++rt)
          for (int l = 0; l < 32; ++l) {
            const int row = r * kRows + rt * 8 + l / 4, col = ks * 4 + l % 4;
            Gf[((size_t(J) * kCl + r) * 32 * 2 + ks * 2 + rt) * 32 + l] = G[(size_t(J) * kN + row) * kN + col];
          }
  // reference
  std::vector<double> yref(c.size());
  for (int grp = 0; grp < NG; ++grp)
    for (int q = 0; q < g; ++q) {
      const int J = grp * g + q;
      for (int k = 0; k < kN; ++k)
        for (int n = 0; n < kC; ++n) {
          double acc = c[(size_t(J) * kN + k) * kC + n];
          if (q > 0)
            for (int b = 0; b < kN; ++b) acc += G[(size_t(J) * kN + k) * kN + b] * yref[(size_t(J - 1) * kN + b) * kC + n];
          yref[(size_t(J) * kN + k) * kC + n] = acc;
        }
    }
  double *dG, *dc, *dy;
  CK(cudaMalloc(&dG, Gf.size() * 8));
  CK(cudaMalloc(&dc, c.size() * 8));
  CK(cudaMalloc(&dy, c.size() * 8));
  CK(cudaMemcpy(dG, Gf.data(), Gf.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dc, c.data(), c.size() * 8, cudaMemcpyHostToDevice));
  const size_t smem = sizeof(double) * (kRing * kSlice + 2 * kXs + 4 * 32 * 2);
  auto run = [&](auto kern, const char* name, int reps, int launches, int skip) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(NG * kCl);
    cfg.blockDim = dim3(kThr);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    long long* dT;
    CK(cudaMalloc(&dT, NG * kCl * 4 * 8));
    CK(cudaMemset(dT, 0, NG * kCl * 4 * 8));
    Params P{dG, dc, dy, g, ny, reps, dT, skip};
    CK(cudaMemset(dy, 0, c.size() * 8));
    CK(cudaLaunchKernelEx(&cfg, kern, P));
    CK(cudaDeviceSynchronize());
    std::vector<double> y(c.size());
    CK(cudaMemcpy(y.data(), dy, y.size() * 8, cudaMemcpyDeviceToHost));
    double err = 0, nrm = 0;
    for (size_t i = 0; i < y.size(); ++i) {
      err = std::fmax(err, std::fabs(y[i] - yref[i]));
      nrm = std::fmax(nrm, std::fabs(yref[i]));
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < launches; ++i) CK(cudaLaunchKernelEx(&cfg, kern, P));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us_launch = 1000.0 * ms / launches;
    std::vector<long long> T(NG * kCl * 4);
    CK(cudaMemcpy(T.data(), dT, T.size() * 8, cudaMemcpyDeviceToHost));
    double tb[4] = {0, 0, 0, 0};
    for (int b = 0; b < NG * kCl; ++b)
      for (int i = 0; i < 4; ++i) tb[i] += double(T[b * 4 + i]) / (NG * kCl) / ((launches + 1.0) * reps * g);
    printf("%-22s skip=%d reps=%3d %8.2f us/launch %6.3f us/step err %.1e | cyc/step: tma %5.0f xwait %5.0f mma+sync %5.0f store+send %5.0f\n",
           name, skip, reps, us_launch, us_launch / (reps * g), err / nrm, tb[0], tb[1], tb[2], tb[3]);
    cudaFree(dT);
  };
  for (int reps : {1, 64}) {
    for (int skip : {0, 1, 2}) run(chain_kernel<0>, "dsmem-bulk-exchange", reps, 200, skip);
    for (int skip : {0, 1}) run(chain_kernel<2>, "st.async-push", reps, 200, skip);
  }
  return 0;
}
