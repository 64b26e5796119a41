// FFMA throughput microbenchmark: the fp32 SIMT roofline denominator.
// Each thread runs 16 independent FMA chains (register operands, 3-register form),
// enough ILP to cover the 4-cycle latency; grid = 148 x 8 CTAs x 256 threads.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void __launch_bounds__(256) ffma(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], b, a);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 123.456f) out[0] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  int iters = 20000; int grid = 148 * 8, block = 256;
  ffma<<<grid, block>>>(o, 100, 0.999f, 1e-4f); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ffma<<<grid, block>>>(o, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 32 * iters * (double)grid * block;
    printf("FFMA fp32: %.1f TFLOP/s (%.3f ms)\n", flops / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}
