// Microbenchmark: the conv_halo L56 UMMA stream in isolation -- M=128, N=64, K=16 bf16 UMMAs, 9 taps x 4
// k-steps per "tile", A = a 4-row x 64-slot patch viewed at row shift r*64 + s, B = a resident 9 x 8 KB
// filter (MN-major, SW128) -- with zero or random operand data, one CTA per SM, cycles per UMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc umma_conv_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace xtc;
__device__ int g_tiles = 64;   // tiles per CTA (runtime: the kernel-like 7 or a long 64)
#define TILES g_tiles
__global__ void __launch_bounds__(256, 1) k_conv(int n, int random, int taps_mode, int commits, unsigned long long* cyc, int fence = 0, int v = 0) {
    extern __shared__ uint8_t raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u;
    uint8_t* sm = raw + pad;
    uint8_t* sA = (v & 1) ? sm + 9 * 64 * 128 : sm;    // 320 rows x 128 B (v&1: 3 rotating 32 KB buffers after B)
    uint8_t* sB = (v & 1) ? sm : sm + 320 * 128;        // 9 taps x 64 k x 128 B (N = 64 bf16)
    uint64_t* bar = reinterpret_cast<uint64_t*>((v & 1) ? sm + 9 * 64 * 128 + 3 * 32768 + 8192 : sB + 9 * 64 * 128);
    uint64_t* tb = bar + 1;                    // per-tile commit barriers (2, by tile parity)
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int words = ((v & 1) ? 9 * 64 * 128 + 3 * 32768 + 8192 : 320 * 128 + 9 * 64 * 128) / 4;
    for (int i = tid; i < words; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        // bf16 pairs with exponent near 1.0 and random mantissa/sign
        const uint32_t lo = 0x3f00u | (h & 0x80ffu), hi = 0x3f00u | ((h >> 16) & 0x80ffu);
        // v&2: uniform[-1,1) like the seeded generator (small magnitudes included)
        const uint32_t lo2 = (uint32_t)__float_as_uint(((float)(h & 0xffff) / 32768.f) - 1.f) >> 16;
        const uint32_t hi2 = (uint32_t)__float_as_uint(((float)(h >> 16) / 32768.f) - 1.f) >> 16;
        reinterpret_cast<uint32_t*>(sm)[i] = random ? ((v & 2) ? (lo2 | (hi2 << 16)) : (lo | (hi << 16))) : 0u;
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) { ptx::mbar_init(bar, 1); ptx::mbar_init(&tb[0], 1); ptx::mbar_init(&tb[1], 1); ptx::fence_mbarrier_init(); }
    if (warp == 0) { ptx::tmem_alloc<1>(slot, (v & 4) ? 128 : 256); ptx::tmem_relinquish<1>(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    if (warp == 1) {
        const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(sA), 16, 1024);
        const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(sB), 64 * 128, 1024, 2);
        __syncwarp();
        const unsigned long long t0 = clock64();
        if (ptx::elect_one()) {
            for (int t = 0; t < TILES; ++t) {
                if (fence == 1) ptx::tc_fence_after();       // like the conv kernel's per-tile tcgen05.fence::after_thread_sync
                if (fence == 2) ptx::tc_fence_before();
                const uint32_t d = tmem + (uint32_t)((t & 1) * 64);
                const int ntap = n == 192 ? 3 : 9;     // N = 192: the s-fold (3 taps of a filter row per UMMA)
                for (int tap0 = 0; tap0 < ntap; ++tap0) {
                    const int tap = n == 192 ? tap0 * 3 : tap0;
                    const int shift = taps_mode ? (tap / 3) * 64 + (n == 192 ? 0 : tap % 3) : 0;
                    const uint64_t ad = ad0 + (uint64_t)(shift * 8) + (uint64_t)((v & 1) ? (t % 3) * 2048 : 0);
                    const uint64_t bd = bd0 + (uint64_t)(tap * 64 * 128 / 16);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        // v&8: two independent accumulator chains (taps alternate between d and d + 128 columns)
                        ptx::umma<false, 1>((v & 8) ? d + (uint32_t)((tap0 & 1) * 128) : d, ad + (uint64_t)(kk * 2),
                                            bd + (uint64_t)(kk * 16 * 8), idesc,
                                            ((v & 8) ? ((tap0 >> 1) | kk) : (tap0 | kk)) ? 1u : 0u);
                }
                if (commits) ptx::umma_commit<1>(&tb[t & 1]);   // like the conv kernel: pempty / tfull per tile
                if (commits > 1) ptx::umma_commit<1>(&tb[t & 1]);
            }
            ptx::umma_commit<1>(bar);
        }
        __syncwarp();
        ptx::mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        if ((tid & 31) == 0) cyc[blockIdx.x] = t1 - t0;
    } else if (commits && warp >= 4) {
        // epilogue-like warps: poll the per-tile commit barriers (like the tfull waits) until the end
        const uint32_t a0 = ptx::smem_u32(&tb[0]), a1 = ptx::smem_u32(&tb[1]), ab = ptx::smem_u32(bar);
        while (!ptx::mbar_try_wait(ab, 0)) { ptx::mbar_try_wait(a0, 0); ptx::mbar_try_wait(a1, 0); }
    } else {
        ptx::mbar_wait(bar, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<1>(tmem, (v & 4) ? 128 : 256); }
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * sizeof(unsigned long long));
    const int smem = 213900;
    cudaFuncSetAttribute(k_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long h[148];
    printf("N   data    taps        cycles/UMMA (median CTA over 148)   floor = 128*N/256\n");
    for (int nt : {64, 7})
    for (int n : {64})
        for (int rnd : {1})
            for (int cm : {1})
            for (int tm : {1})
            for (int fe : {1})
            for (int vv : {0, 8}) {
                cudaMemcpyToSymbol(g_tiles, &nt, sizeof nt);
                printf("tiles %d: ", nt);
                k_conv<<<148, 256, smem>>>(n, rnd, tm, cm, d, fe, vv);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                for (int i = 0; i < 148; ++i)
                    for (int j = i + 1; j < 148; ++j)
                        if (h[j] < h[i]) { unsigned long long t = h[i]; h[i] = h[j]; h[j] = t; }
                printf("%-3d %-7s %-11s commits/tile %d fence %d variant %d %-20.1f %d\n", n, rnd ? "random" : "zeros", tm ? "conv shifts" : "no shift", cm, fe, vv,
                       (double)h[74] / (nt * (n == 192 ? 12 : 36)), 128 * n / 256);
            }
    return 0;
}
