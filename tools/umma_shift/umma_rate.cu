// Microbenchmark: tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) issue rate with the
// A descriptor 1024-byte aligned vs advanced by s 128-byte rows, for N = 64/128/256, A and
// B both in SMEM (SS mode).  One CTA per SM (grid 148), 2048 back-to-back MMAs into one
// accumulator, cycles from clock64 around issue..commit-wait.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc umma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace xtc;

constexpr int NMMA = 2048;

__global__ void __launch_bounds__(128, 1) k_rate(int n, int shift, int a_stride_rows, unsigned long long* cyc) {
    extern __shared__ uint8_t raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u;
    uint8_t* sm = raw + pad;
    uint8_t* sA = sm;                        // 256 rows x 128 B (zeros are fine for timing)
    uint8_t* sB = sm + 256 * 128;            // 16 K-rows x 256 N, MN-major: 4 blocks of 16 x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 4 * 16 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (256 * 128 + 4 * 16 * 128) / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (tid == 0) { ptx::mbar_init(bar, 1); ptx::fence_mbarrier_init(); }
    if (warp == 0) { ptx::tmem_alloc<1>(slot, 256); ptx::tmem_relinquish<1>(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    if (warp == 1) {
        const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(sA) + shift * 128, 16, 1024);
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sB), 16 * 128, 1024, 2);
        __syncwarp();
        const unsigned long long t0 = clock64();
        if (ptx::elect_one()) {
            for (int i = 0; i < NMMA; ++i) {
                // cycle the A start over a few row offsets (a_stride_rows apart) like the conv taps do
                const uint64_t ad = ad0 + (uint64_t)(((i & 7) * a_stride_rows) * 8);
                ptx::umma<false, 1>(tmem, ad, bd, idesc, i > 0 ? 1u : 0u);
            }
            ptx::umma_commit<1>(bar);
        }
        __syncwarp();
        ptx::mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        if ((tid & 31) == 0) cyc[blockIdx.x] = t1 - t0;
    } else {
        ptx::mbar_wait(bar, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<1>(tmem, 256); }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * sizeof(unsigned long long));
    const int smem = 256 * 128 + 4 * 16 * 128 + 64 + 1024;
    cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long h[148];
    printf("N    shift  a_step_rows  cycles/MMA (median CTA)  floor=128*N/256\n");
    for (int n : {64, 128, 256})
        for (int shift : {0, 1, 3, 8})
            for (int step : {0, 1, 8, 16}) {
                if (shift + 7 * step + 128 > 256 && step) continue;
                k_rate<<<148, 128, smem>>>(n, shift, step, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                unsigned long long v[148];
                for (int i = 0; i < 148; ++i) v[i] = h[i];
                for (int i = 0; i < 148; ++i)
                    for (int j = i + 1; j < 148; ++j)
                        if (v[j] < v[i]) { unsigned long long t = v[i]; v[i] = v[j]; v[j] = t; }
                printf("%-4d %-6d %-12d %-24.1f %d\n", n, shift, step, (double)v[74] / NMMA, 128 * n / 256);
            }
    return 0;
}
