// fp64 peak microbenchmark: sustained DFMA throughput on one B200.
// Each thread runs 8 independent DFMA chains; grid = 148 SMs x 8 CTAs x 256 threads.
// Prints achieved DFMA/s (1 DFMA = 2 flop) for a burst (~0.2 s) and a sustained (~4 s) run.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, long iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256;
  double* out; cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  // burst (~9 ms), ~0.18 s, and a sustained run of 25 back-to-back ~0.18 s launches (~4.5 s,
  // clocks sampled by the caller with nvidia-smi)
  for (long iters : {4000L, 80000L, -80000L}) {
    const int reps = iters < 0 ? 25 : 1;
    if (iters < 0) iters = -iters;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dfma = (double)blocks * threads * iters * 16 * 8 * reps;
    printf("{\"iters\": %ld, \"launches\": %d, \"ms\": %.3f, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_1965\": %.2f}\n",
           iters, reps, ms, dfma / (ms * 1e-3), 2 * dfma / (ms * 1e-3) / 1e12, dfma / (ms * 1e-3) / sms / 1.965e9);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
