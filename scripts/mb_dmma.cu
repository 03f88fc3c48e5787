// mb_dmma.cu — fp64 mma.sync.m8n8k4 latency and throughput on one SM (B200).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mbd scripts/mb_dmma.cu && /tmp/mbd
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// each warp: `chains` independent accumulator chains, `n` DMMAs per chain
template <int kChains>
__global__ void k(int n, double* out, long long* cyc) {
  double acc[kChains][2];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kC>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * 1024);
  cudaMalloc(&cyc, sizeof(long long));
  const int n = 4096;
  k<kC><<<1, 32 * warps>>>(n, out, cyc);
  k<kC><<<1, 32 * warps>>>(n, out, cyc);
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per = double(c) / n;  // cycles per round of kC DMMAs per warp
  printf("warps %2d chains/warp %d: %.1f cycles per dependent round, %.2f cycles per DMMA per SM, %.0f FMA/clk/SM\n",
         warps, kC, per, per / (kC * warps), 256.0 * kC * warps / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
    run<8>(w);
  }
  return 0;
}
