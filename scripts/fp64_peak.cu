// fp64 tensor-core (mma.sync m8n8k4 f64) and fp64 FMA peak microbenchmark:
// register-resident operands, many independent accumulators per warp, every
// SM busy.  Prints JSON {"dmma_tflops": .., "dfma_tflops": ..}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_loop(int iters, double* out) {
  double acc[8][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int t = 0; t < iters; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(int iters, double* out) {
  double acc[8];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int t = 0; t < iters; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 4, iters = 20000;
  float best_mma = 1e30f, best_fma = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best_mma) best_mma = ms;
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best_fma) best_fma = ms;
  }
  const double warps = double(blocks) * threads / 32;
  const double mma_flops = warps * iters * 8 * (8.0 * 8 * 4 * 2);
  const double fma_flops = double(blocks) * threads * iters * 8 * 2.0;
  printf("{\"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"sms\": %d, \"how\": \"%d blocks x %d threads, %d iters x 8 independent m8n8k4 f64 MMAs (or FMAs) per warp (thread), best of 4\"}\n",
         mma_flops / (best_mma * 1e-3) / 1e12, fma_flops / (best_fma * 1e-3) / 1e12, sms, blocks, threads, iters);
  return 0;
}
