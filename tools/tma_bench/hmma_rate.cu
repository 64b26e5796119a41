// Legacy tensor-core rate on sm_100a: warps issue back-to-back mma.sync.m16n8k16 bf16 -> fp32 on
// ACC independent accumulators; reports HMMA per SM per cycle and dense TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
template <int ACC>
__global__ void hmma_kernel(float* out, int iters) {
    float d[ACC][4] = {};
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < ACC; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < ACC; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ACC>
void run(int warps_per_sm) {
    int sms = 148, iters = 4096;
    float* out; cudaMalloc(&out, sms * warps_per_sm * 32 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    hmma_kernel<ACC><<<sms, warps_per_sm * 32>>>(out, 16);
    cudaEventRecord(e0);
    hmma_kernel<ACC><<<sms, warps_per_sm * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)sms * warps_per_sm * iters * ACC;   // HMMA instructions
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("ACC %d warps/SM %2d: %.3f ms  %.3f HMMA/SM/clk (at %d MHz nominal)  %.1f TFLOP/s  err=%s\n", ACC, warps_per_sm,
           ms, n / sms / cyc, clk / 1000, n * 4096 * 2 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}
int main() {
    for (int w : {4, 8, 16, 32}) { run<1>(w); run<4>(w); run<8>(w); }
    return 0;
}
