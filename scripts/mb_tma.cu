// Microbenchmark: cp.async.bulk (global -> shared) streaming throughput per SM,
// the operator stream of sweep_v5.cu.  One CTA per SM (grid = nblk), a producer
// thread fills a ring of `slots` chunks of `chunk` bytes from a large buffer,
// 4 consumer warps wait on each chunk and release it (optionally reading it).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tma scripts/mb_tma.cu
//   /tmp/mb_tma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ bool tw(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
               : "=r"(ok) : "r"(su(b)), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ void wt(uint64_t* b, uint32_t par) { while (!tw(b, par)) {} }

__global__ void __launch_bounds__(160, 1) stream(const char* src, size_t span, int chunk, int slots, int iters,
                                                 int readit, int perwarp, unsigned long long* cyc, double* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[16], freeb[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < slots; ++i) { init(&full[i], perwarp == 2 ? 32 : 1); init(&freeb[i], perwarp == 1 ? 4 : 128); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const size_t per = (span / gridDim.x) & ~size_t(65535);
  const char* base = src + per * blockIdx.x;
  const int nch = int(per / chunk);
  long long t0 = clock64();
  if (perwarp == 2 && tid >= 128) {  // LDGSTS by one producer warp
    const int ln = tid - 128;
    for (int it = 0; it < iters; ++it) {
      const int s = it % slots;
      if (it >= slots) wt(&freeb[s], ((it / slots) - 1) & 1);
      const char* g = base + size_t(it % nch) * chunk;
      const uint32_t d = su(sm + size_t(s) * chunk);
      for (int o = ln * 16; o < chunk; o += 32 * 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + o), "l"(g + o) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su(&full[s])) : "memory");
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else if (tid == 128) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % slots;
      if (it >= slots) wt(&freeb[s], ((it / slots) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(&full[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       su(sm + size_t(s) * chunk)), "l"(base + size_t(it % nch) * chunk), "r"(chunk), "r"(su(&full[s]))
                   : "memory");
    }
  } else if (tid < 128) {
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
      const int s = it % slots;
      wt(&full[s], (it / slots) & 1);
      if (readit) {
        const double* d = reinterpret_cast<const double*>(sm + size_t(s) * chunk);
        for (int e = tid; e < chunk / 8; e += 128) acc += d[e];
      }
      if (perwarp) {
        __syncwarp();
        if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su(&freeb[s])) : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su(&freeb[s])) : "memory");
      }
    }
    if (acc == 1.2345) sink[0] = acc;
  }
  __syncthreads();
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t span = size_t(2) << 30;  // 2 GB: HBM-resident
  char* src;
  cudaMalloc(&src, span);
  cudaMemset(src, 1, span);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  double* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int chunks[] = {4096, 16384, 32768};
  const int grids[] = {1, 16, 32, 128, 148};
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int perwarp = 0; perwarp < 3; perwarp += 2)
  for (int readit = 0; readit < 1; ++readit)
    for (int chunk : {16384, 32768})
      for (int gi = 0; gi < 5; gi += 2)
        for (int sl : {2, 3, 4, 6, 12}) {
          const int grid = grids[gi];
          if (size_t(sl) * chunk > 200 * 1024) continue;
          const int iters = int((size_t(64) << 20) / chunk);  // 64 MB per CTA
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          stream<<<grid, 160, sl * chunk>>>(src, span, chunk, sl, 64, readit, perwarp, cyc, sink);  // warm
          cudaEventRecord(a);
          stream<<<grid, 160, sl * chunk>>>(src, span, chunk, sl, iters, readit, perwarp, cyc, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          unsigned long long h[148];
          cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
          const double bytes = double(iters) * chunk;
          std::printf("perwarp=%d read=%d chunk=%6d grid=%3d slots=%2d: %7.1f B/clk/SM  %8.1f GB/s total  (%s)\n", perwarp, readit, chunk,
                      grid, sl, bytes / double(h[0]), bytes * grid / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
