// Microbenchmark: fp64 m8n8k4 DMMA throughput with both operands read from
// shared memory, the inner loop of the sweep kernels (sweep_v4.cu warp_mma,
// sweep_v5.cu chunk_mma).  One CTA per SM, W warps.
//   mode 0: one 8x8 tile per warp, A and B loaded from smem for every DMMA
//           (512 B of shared loads per DMMA)
//   mode 1: 2x2 tiles per warp (16 rows x 16 chains): per k-step 2 A + 2 B
//           fragments feed 4 DMMAs (256 B per DMMA)
//   mode 2: operands from registers (the pipe alone)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_dmma_smem scripts/mb_dmma_smem.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int kMode>
__global__ void kern(int iters, long long* cyc, double* out) {
  __shared__ double A[32 * 4 * 32];  // [ks 32][rt 4][lane 32]
  __shared__ double B[32 * 64];      // [ks 32][ct 2][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 32 * 4 * 32; i += blockDim.x) A[i] = 1.0 + i * 1e-7;
  for (int i = tid; i < 32 * 64; i += blockDim.x) B[i] = 1.0 - i * 1e-7;
  __syncthreads();
  double acc[4][2] = {};
  const int rt = warp & 3, ct = (warp >> 2) & 1;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (kMode == 0) {
      const double* Ap = A + rt * 32 + lane;
      const double* Bp = B + ct * 32 + lane;
#pragma unroll
      for (int ks = 0; ks < 32; ks += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = Ap[(ks + u) * 128];
          bv[u] = Bp[(ks + u) * 64];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(acc[u][0], acc[u][1], av[u], bv[u]);
      }
    } else if (kMode == 1) {  // 2 row tiles x 2 chain tiles, half the k-steps (same DMMA count)
      const double* Ap = A + (rt & 2) * 32 + lane;
      const double* Bp = B + lane;
#pragma unroll
      for (int ks = 0; ks < 32; ks += 4) {
        const int k = ks + 2 * (warp & 1);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double a0 = Ap[(k + u) * 128], a1 = Ap[(k + u) * 128 + 32];
          const double b0 = Bp[(k + u) * 64], b1 = Bp[(k + u) * 64 + 32];
          dmma(acc[0][0], acc[0][1], a0, b0);
          dmma(acc[1][0], acc[1][1], a0, b1);
          dmma(acc[2][0], acc[2][1], a1, b0);
          dmma(acc[3][0], acc[3][1], a1, b1);
        }
      }
    } else {
      const double a = A[lane], b = B[lane];
#pragma unroll
      for (int ks = 0; ks < 32; ks += 4)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(acc[u][0], acc[u][1], a, b);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < 4; ++u) s += acc[u][0] + acc[u][1];
  if (s == 1.2345) out[0] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  long long* cyc;
  double* out;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&out, 8);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {2, 4, 8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) kern<0><<<148, warps * 32>>>(iters, cyc, out);
        if (mode == 1) kern<1><<<148, warps * 32>>>(iters, cyc, out);
        if (mode == 2) kern<2><<<148, warps * 32>>>(iters, cyc, out);
      }
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double dmmas = double(iters) * 32 * warps;  // per SM
      std::printf("mode %d (%s) warps %2d: %.2f cycles per DMMA per SM (%.1f per warp-DMMA)  %s\n", mode,
                  mode == 0 ? "smem A+B per DMMA" : mode == 1 ? "2x2 tiles, smem" : "registers", warps,
                  double(h) / dmmas, double(h) / (double(iters) * 32), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
