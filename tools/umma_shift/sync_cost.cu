// Microbenchmark: cycles per tcgen05.commit (no MMAs in flight), per tcgen05.fence::before/after_thread_sync,
// per satisfied mbarrier try_wait, per named barrier among 4 warps, per tcgen05.ld 32x32b.x32 + wait,
// one CTA per SM (grid 148), 256 threads, TMEM allocated.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc sync_cost.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace xtc;
constexpr int N = 256;
__global__ void __launch_bounds__(256, 1) k(unsigned long long* out) {
    __shared__ uint64_t bar[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::fence_mbarrier_init(); }
    if (warp == 0) { ptx::tmem_alloc<1>(&slot, 128); ptx::tmem_relinquish<1>(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    unsigned long long t[8] = {0};
    if (warp == 1) {
        long long a = clock64();
        if (ptx::elect_one()) for (int i = 0; i < N; ++i) ptx::umma_commit<1>(&bar[i & 1]);
        __syncwarp();
        long long b = clock64(); t[0] = b - a;
        a = clock64();
        for (int i = 0; i < N; ++i) ptx::tc_fence_before();
        b = clock64(); t[1] = b - a;
        a = clock64();
        for (int i = 0; i < N; ++i) ptx::tc_fence_after();
        b = clock64(); t[2] = b - a;
        a = clock64();
        for (int i = 0; i < N; ++i) ptx::mbar_try_wait(ptx::smem_u32(&bar[0]), 1);   // completed phase: immediate
        b = clock64(); t[3] = b - a;
    }
    if (warp >= 4) {
        long long a = clock64();
        for (int i = 0; i < N; ++i) ptx::named_bar_sync(3, 128);
        long long b = clock64(); t[4] = b - a;
        uint32_t v[32]; float acc = 0;
        a = clock64();
        for (int i = 0; i < N; ++i) {
            ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((i & 1) * 32), v);
            ptx::tmem_ld_wait();
            acc += __uint_as_float(v[i & 31]);
        }
        b = clock64(); t[5] = b - a;
        a = clock64();
        for (int i = 0; i < N; ++i) {
            float x = __uint_as_float(v[i & 31]);
#pragma unroll
            for (int j = 0; j < 32; ++j) x += __shfl_down_sync(0xffffffffu, __uint_as_float(v[j]), 1);
            acc += x;
        }
        b = clock64(); t[6] = b - a;
        if (acc == 12345.f) t[7] = 1;
    }
    if (lane == 0 && (warp == 1 || warp == 4))
        for (int i = 0; i < 8; ++i) if (t[i]) out[blockIdx.x * 16 + (warp == 1 ? 0 : 8) + i] = t[i];
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<1>(tmem, 128); }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 16 * 8); cudaMemset(d, 0, 148 * 16 * 8);
    k<<<148, 256>>>(d); k<<<148, 256>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[16] = {"tcgen05.commit (elected lane)", "tcgen05.fence::before_thread_sync", "tcgen05.fence::after_thread_sync",
                             "mbarrier.try_wait (completed)", "", "", "", "", "", "", "", "", "bar.sync 128 threads (4 warps)",
                             "tcgen05.ld 32x32b.x32 + wait::ld", "32 shfl.down + 32 fadd", ""};
    for (int i : {0, 1, 2, 3, 12, 13, 14}) printf("%-40s %8.1f cycles\n", names[i], (double)h[i] / N);
    printf("%s\n", cudaGetErrorString(e));
}
