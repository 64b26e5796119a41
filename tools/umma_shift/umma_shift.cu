// Microtest: can a K-major SW128 UMMA A operand start at a row that is not a multiple of
// 8 (i.e. not 1024-byte aligned)?  The haloed-patch conv producer needs the 9 filter taps
// of a stride-1 conv as row-shifted views of one SMEM patch.  For s = 0..15 rows of shift,
// run one tcgen05.mma (M=128, N=64, K=16, bf16) with the descriptor's start advanced by
// s*128 B, once with base_offset = 0 and once with base_offset = s & 7 (descriptor bits
// 49-51), and compare with the host product.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc umma_shift.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"

using namespace xtc;

constexpr int ROWS = 144;     // A rows in SMEM (128 + max shift 16)
constexpr int NTEST = 48;     // 16 shifts x {(base_offset 0, k 0..15), (s&7, k 0..15), (s&7, k 32..47)}

__device__ __host__ inline float aval(int i, int k) { return (float)(((i * 7 + k * 3) % 9) - 4); }
__device__ __host__ inline float bval(int k, int n) { return (float)(((n * 5 + k) % 7) - 3); }

__device__ inline uint16_t bf16(float f) { return (uint16_t)(ptx::pack_bf16x2(f, 0.f) & 0xFFFFu); }

__global__ void __launch_bounds__(128, 1) k_shift(float* out) {
    extern __shared__ uint8_t raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u;
    uint8_t* sm = raw + pad;
    uint8_t* sA = sm;                      // ROWS x 128 B, SW128 by absolute row (row & 7)
    uint8_t* sB = sm + ROWS * 128;         // 64 K-rows x 64 N (128 B), MN-major SW128
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 64 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < ROWS * 64; e += 128) {
        const int i = e / 64, k = e % 64;
        const int chunk = (k / 8) ^ (i & 7);
        reinterpret_cast<uint16_t*>(sA + i * 128 + chunk * 16)[k % 8] = bf16(aval(i, k));
    }
    for (int e = tid; e < 64 * 64; e += 128) {
        const int k = e / 64, n = e % 64;
        const int chunk = (n / 8) ^ (k & 7);
        reinterpret_cast<uint16_t*>(sB + k * 128 + chunk * 16)[n % 8] = bf16(bval(k, n));
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) { ptx::mbar_init(bar, 1); ptx::fence_mbarrier_init(); }
    if (warp == 0) { ptx::tmem_alloc<1>(slot, 64); ptx::tmem_relinquish<1>(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((64u >> 3) << 17) |
                           ((128u >> 4) << 24);
    for (int t = 0; t < NTEST; ++t) {
        const int s = t / 3, var = t % 3;
        const uint64_t base_off = var ? (uint64_t)(s & 7) : 0ull;
        const uint32_t kk = var == 2 ? 2u : 0u;           // k-step inside the 128-B row: +32 B each
        if (tid == 0) {
            uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(sA) + s * 128 + kk * 32, 16, 1024) | (base_off << 49);
            uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sB) + kk * 16 * 128, 2048, 1024, 2);
            ptx::umma<false, 1>(tmem, ad, bd, idesc, 0u);
            ptx::umma_commit<1>(bar);
        }
        ptx::mbar_wait(bar, (uint32_t)(t & 1));
        ptx::tc_fence_after();
        for (int c = 0; c < 64; c += 32) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
            ptx::tmem_ld_wait();
            for (int j = 0; j < 32; ++j) out[((size_t)t * 128 + 32 * warp + lane) * 64 + c + j] = __uint_as_float(v[j]);
        }
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
    }
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<1>(tmem, 64);
}

int main() {
    float* d;
    cudaMalloc(&d, (size_t)NTEST * 128 * 64 * 4);
    const int smem = ROWS * 128 + 64 * 128 + 64 + 1024;
    cudaFuncSetAttribute(k_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_shift<<<1, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> h((size_t)NTEST * 128 * 64);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    int bad_total = 0;
    for (int t = 0; t < NTEST; ++t) {
        const int s = t / 3, var = t % 3, k0 = var == 2 ? 32 : 0;
        int bad = 0;
        for (int i = 0; i < 128; ++i)
            for (int n = 0; n < 64; ++n) {
                float ref = 0;
                for (int k = k0; k < k0 + 16; ++k) ref += aval(i + s, k) * bval(k, n);
                if (h[((size_t)t * 128 + i) * 64 + n] != ref) ++bad;
            }
        printf("shift %2d base_offset %d k0 %2d: %s (%d/8192 wrong)\n", s, var ? (s & 7) : 0, k0, bad ? "WRONG" : "ok", bad);
        if (var) bad_total += bad;
    }
    printf("base_offset=(s&7) for all shifts: %s\n", bad_total ? "FAILS" : "PASSES");
    return 0;
}
