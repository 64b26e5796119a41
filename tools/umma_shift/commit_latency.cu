// Microbenchmark: round-trip latency of the tcgen05.commit -> mbarrier -> waiting warp
// handoff, the per-tile handshake of the warp-specialised kernels.
//   issuer warp 1: for i: [wait back-barrier] [optional UMMA] tcgen05.commit -> bar
//   waiter warp 4: for i: wait bar (try_wait spin | test_wait spin) ; arrive back-barrier
// Also the same round trip with a plain mbarrier.arrive instead of tcgen05.commit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc commit_latency.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace xtc;

__device__ __forceinline__ bool test_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    return ok != 0;
}

template <int TEST>
__device__ __forceinline__ void spin(uint64_t* bar, uint32_t parity) {
    const uint32_t a = ptx::smem_u32(bar);
    if constexpr (TEST == 1) { while (!test_wait(a, parity)) {} }
    else if constexpr (TEST == 2) { ptx::mbar_wait(bar, parity); }      // the kernels' wait (watchdog reads %globaltimer)
    else if constexpr (TEST == 3) {                                     // same, clock64-based watchdog
        if (ptx::mbar_try_wait(a, parity)) return;
        const long long t0 = clock64();
        uint32_t n = 0;
        while (!ptx::mbar_try_wait(a, parity))
            if ((++n & 1023u) == 0 && clock64() - t0 > (1ll << 40)) __trap();
    }
    else { while (!ptx::mbar_try_wait(a, parity)) {} }
}

// mode: 0 commit (no MMA), 1 commit after one UMMA, 2 plain mbarrier.arrive
template <int TEST>
__global__ void __launch_bounds__(256, 1) k(int mode, int iters, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u;
    uint8_t* sm = raw + pad;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768);
    uint64_t* back = bar + 1;
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 32768 / 16; i += 256) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::mbar_init(back, 1); ptx::fence_mbarrier_init(); }
    if (warp == 2) { ptx::tmem_alloc<1>(slot, 64); ptx::tmem_relinquish<1>(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    unsigned long long t0 = clock64();
    if (warp == 1) {
        for (int i = 0; i < iters; ++i) {
            if (i > 0) spin<TEST>(back, (uint32_t)((i - 1) & 1));
            if (ptx::elect_one()) {
                if (mode == 1)
                    ptx::umma<false, 1>(tmem, ptx::smem_desc_sw128(ptx::smem_u32(sm), 16, 1024),
                                        ptx::smem_desc_sw128(ptx::smem_u32(sm) + 16384, 1024, 1024, 2), idesc, 0u);
                if (mode == 2) ptx::mbar_arrive(bar);
                else ptx::umma_commit<1>(bar);
            }
            __syncwarp();
        }
    } else if (warp == 4) {
        for (int i = 0; i < iters; ++i) {
            spin<TEST>(bar, (uint32_t)(i & 1));
            if (lane == 0) ptx::mbar_arrive(back);
            __syncwarp();
        }
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc<1>(tmem, 64); }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 32768 + 64 + 1024;
    const char* mname[3] = {"tcgen05.commit (no MMA)", "UMMA + tcgen05.commit", "mbarrier.arrive"};
    const char* wname[4] = {"try_wait", "test_wait", "mbar_wait", "clk-wdog"};
    for (int test = 0; test < 4; ++test)
        for (int mode = 0; mode < 3; ++mode) {
            auto kern = test == 0 ? k<0> : test == 1 ? k<1> : test == 2 ? k<2> : k<3>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int iters = 200;
            kern<<<148, 256, smem>>>(mode, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            printf("%-26s waiter %-9s: %8.1f cycles per round trip (%s)\n", mname[mode], wname[test],
                   avg / iters, cudaGetErrorString(e));
        }
    return 0;
}
