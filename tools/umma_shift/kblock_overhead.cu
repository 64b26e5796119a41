// Microbenchmark: per-k-block hand-off cost of a tcgen05 ring.  One MMA thread issues KB k-blocks of
// U UMMAs (M=128, N, K=16 bf16, operands resident in SMEM, 1 CTA per SM).  Modes per k-block:
//   0  UMMAs only
//   1  + an mbarrier wait that passes at once (a completed phase) + tcgen05.fence::after_thread_sync +
//        tcgen05.commit to the stage's empty barrier
//   2  like 1 with a producer warp that re-arms each full barrier only after the consumer's commit on the
//        empty barrier has fired (a real S-stage ring with zero-latency "loads": plain arrives)
// Cycles per UMMA (median CTA).  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc kblock_overhead.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include "ptx.cuh"
using namespace xtc;
constexpr int KB = 144, S = 4;
__global__ void __launch_bounds__(256, 1) k(int n, int u, int mode, unsigned long long* cyc, int v) {
    extern __shared__ uint8_t raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u;
    uint8_t* sm = raw + pad;
    uint8_t* sA = sm;                          // 128 rows x 128 B x 8 (k atoms)
    uint8_t* sB = sm + 128 * 1024;             // N x 16 x ... (MN-major, SW128)
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + 200 * 1024);
    uint64_t* empty = full + S;
    uint64_t* done = empty + S;
    uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        const uint32_t lo = 0x3f00u | (h & 0x80ffu), hi = 0x3f00u | ((h >> 16) & 0x80ffu);
        reinterpret_cast<uint32_t*>(sm)[i] = (v & 1) ? (lo | (hi << 16)) : (0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu));
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        ptx::mbar_init(done, 1);
        ptx::fence_mbarrier_init();
        if (mode == 1) ptx::mbar_arrive(&full[0]);    // phase 0 of full[0] complete: every wait passes at once
    }
    if (warp == 0) { ptx::tmem_alloc<1>(slot, 256); ptx::tmem_relinquish<1>(); }
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
            int s = 0; uint32_t ph = 0;
            for (int kb = 0; kb < KB; ++kb) {
                if (mode == 1) { ptx::mbar_wait(&full[0], 0); ptx::tc_fence_after(); }
                if (mode == 2) { ptx::mbar_wait(&full[s], ph); ptx::tc_fence_after(); }
                if (u == 4) {                          // the kernels' form: k-steps unrolled, constant offsets
                    const uint64_t bk = bd0 + (uint64_t)((v & 2) ? (kb % 8) * 512 : 0);
                    const uint32_t dk = tmem + (uint32_t)((v & 4) ? ((kb / 9) & 1) * 128 : 0);
                    const uint32_t acc0 = ((v & 4) && kb % 9 == 0) ? 0u : 1u;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        ptx::umma<false, 1>(dk, ad0 + (uint64_t)(j * 2), bk + (uint64_t)(j * 128), idesc,
                                            (kb | j) ? (j ? 1u : acc0) : 0u);
                } else {                               // runtime k-step index (descriptor math per UMMA)
                    for (int j = 0; j < u; ++j)
                        ptx::umma<false, 1>(tmem, ad0 + (uint64_t)((j & 3) * 2), bd0 + (uint64_t)((j & 3) * 128), idesc,
                                            (kb | j) ? 1u : 0u);
                }
                if (mode == 1 || mode == 2) ptx::umma_commit<1>(&empty[s]);
                if (mode == 3 && kb % 9 == 8) ptx::umma_commit<1>(&empty[(kb / 9) & 1]);   // a commit per 36 UMMAs, no waits
                if (mode == 4) ptx::umma_commit<1>(&empty[s]);                            // a commit per k-block, no waits
                if (++s == S) { s = 0; ph ^= 1u; }
            }
            ptx::umma_commit<1>(done);
        }
        __syncwarp();
        ptx::mbar_wait(done, 0);
        const unsigned long long t1 = clock64();
        if ((tid & 31) == 0) cyc[blockIdx.x] = t1 - t0;
    } else if (warp == 2 && mode == 2) {
        if (ptx::elect_one()) {
            int s = 0; uint32_t ph = 0;
            for (int kb = 0; kb < KB; ++kb) {
                if (kb >= S) ptx::mbar_wait(&empty[s], ph ^ 1u);
                ptx::mbar_arrive(&full[s]);
                if (++s == S) { s = 0; ph ^= 1u; }
            }
        }
        __syncwarp();
        ptx::mbar_wait(done, 0);
    } else {
        ptx::mbar_wait(done, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<1>(tmem, 256); }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 8);
    const int smem = 200 * 1024 + 1024 + 256;   // B region 72 KB = 9 x 8 KB blocks (v&2)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long h[148];
    printf("N   U/kb  mode  cycles/UMMA  (floor 128*N/256)\n");
    for (int n : {64, 128})
        for (int u : {4})
            for (int mode : {0, 3, 4})
            for (int v : {0, 1, 2, 6}) {
                k<<<148, 256, smem>>>(n, u, mode, d, v);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                std::sort(h, h + 148);
                printf("%-3d %-5d %-5d v%d %-12.1f %d\n", n, u, mode, v, (double)h[74] / (KB * u), 128 * n / 256);
            }
    return 0;
}
