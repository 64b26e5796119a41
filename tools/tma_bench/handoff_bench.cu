// Cross-CTA partial hand-off microbenchmark (the split-K / stream-K fix-up step): 148 CTAs x 4
// warps; CTA g writes a 128-row x 64-column fp32 partial (32 KB) to its slot, publishes a flag
// (warp: __syncwarp, lane 0 fence.acq_rel.gpu + st.relaxed flag), then reads CTA g+1's slot
// after seeing its flag.  Write / publish / read phases are timed per warp with %clock64 and
// reported as the median over warps, for three access patterns of the SAME data:
//   0 row-per-thread : lane = row, 8 x 16-byte stores/loads per 32 columns (the TMEM-lane layout)
//   1 coalesced      : a warp covers whole 128-byte row segments (lane -> (row, 16-byte chunk))
//   2 bulk copy      : rows staged in SMEM, one 4 KB cp.async.bulk per 32 rows x 32 columns
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc handoff_bench.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#include "ptx.cuh"

using namespace xtc;

__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(ptx::smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ptx::smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

template <int PAT>
__global__ void __launch_bounds__(128, 1) k_handoff(float* slots, uint32_t* flags, uint32_t epoch, long long* out) {
    __shared__ __align__(1024) uint8_t stage[4][2][4096];
    __shared__ uint64_t bar[4];
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x, G = gridDim.x;
    float* mine = slots + (size_t)g * 128 * 64;
    const float* peer = slots + (size_t)((g + 1) % G) * 128 * 64;
    if (lane == 0) { ptx::mbar_init(&bar[q], 1); ptx::fence_mbarrier_init(); }
    __syncwarp();
    float v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = (float)(g * 7 + j + lane);
    const long long t0 = clock64();
    // ---- write the warp's 32 rows x 64 columns ----
    for (int c = 0; c < 64; c += 32) {
        if (PAT == 0) {
            uint4* dst = reinterpret_cast<uint4*>(mine + (size_t)(32 * q + lane) * 64 + c);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_uint4(__float_as_uint(v[c + 4 * j]), __float_as_uint(v[c + 4 * j + 1]),
                                    __float_as_uint(v[c + 4 * j + 2]), __float_as_uint(v[c + 4 * j + 3]));
        } else {
            uint8_t* st = stage[q][c >> 5];
#pragma unroll
            for (int j = 0; j < 8; ++j)   // row = lane, 16-byte chunk j at (j ^ (lane & 7))
                *reinterpret_cast<uint4*>(st + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(__float_as_uint(v[c + 4 * j]), __float_as_uint(v[c + 4 * j + 1]),
                               __float_as_uint(v[c + 4 * j + 2]), __float_as_uint(v[c + 4 * j + 3]));
            __syncwarp();
            float* chunk = mine + ((size_t)(c >> 5) * 4 + q) * 1024;   // [chunk][warp] blocks of 32 x 32 fp32
            if (PAT == 1) {
                for (int i = lane >> 3; i < 32; i += 4) {
                    const int j = lane & 7;
                    reinterpret_cast<uint4*>(chunk + i * 32)[j] =
                        *reinterpret_cast<const uint4*>(st + i * 128 + ((j ^ (i & 7)) << 4));
                }
            } else if (lane == 0) {
                ptx::fence_proxy_async_smem();
                bulk_store(chunk, st, 4096);
                ptx::bulk_commit();
            }
        }
    }
    const long long t1 = clock64();
    __syncwarp();
    if (lane == 0) {
        if (PAT == 2) { ptx::bulk_wait<0>(); asm volatile("fence.proxy.async.global;" ::: "memory"); }
        ptx::fence_acq_rel_gpu();
        st_relaxed(flags + g * 4 + q, epoch);
    }
    __syncwarp();
    const long long t2 = clock64();
    if (lane == 0)
        while (ld_acquire(flags + ((g + 1) % G) * 4 + q) != epoch) {}
    __syncwarp();
    const long long t3 = clock64();
    // ---- read the peer's rows into registers (sum as the owner would) ----
    float acc = 0.f;
    for (int c = 0; c < 64; c += 32) {
        if (PAT == 0) {
            const float4* src = reinterpret_cast<const float4*>(peer + (size_t)(32 * q + lane) * 64 + c);
#pragma unroll
            for (int j = 0; j < 8; ++j) { const float4 w = __ldcg(src + j); acc += w.x + w.y + w.z + w.w; }
        } else {
            uint8_t* st = stage[q][c >> 5];
            const float* chunk = peer + ((size_t)(c >> 5) * 4 + q) * 1024;
            if (PAT == 1) {
                for (int i = lane >> 3; i < 32; i += 4) {
                    const int j = lane & 7;
                    *reinterpret_cast<float4*>(st + i * 128 + ((j ^ (i & 7)) << 4)) =
                        __ldcg(reinterpret_cast<const float4*>(chunk + i * 32) + j);
                }
                __syncwarp();
            } else {
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(&bar[q], 4096);
                    bulk_load(st, chunk, 4096, &bar[q]);
                }
                ptx::mbar_wait(&bar[q], (uint32_t)(c >> 5));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 w = *reinterpret_cast<const float4*>(st + lane * 128 + ((j ^ (lane & 7)) << 4));
                acc += w.x + w.y + w.z + w.w;
            }
            __syncwarp();
        }
    }
    const long long t4 = clock64();
    if (lane == 0) {
        long long* o = out + ((size_t)g * 4 + q) * 4;
        o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t2; o[3] = t4 - t3;
    }
    if (acc == 12345.f) out[0] = 0;   // keep the loads
}

int main() {
    const int G = 148;
    float* slots;
    uint32_t* flags;
    long long* out;
    cudaMalloc(&slots, (size_t)G * 128 * 64 * 4);
    cudaMalloc(&flags, G * 4 * 4);
    cudaMemset(flags, 0, G * 4 * 4);
    cudaMalloc(&out, (size_t)G * 4 * 4 * 8);
    void* flush;
    const size_t fb = 512ull << 20;
    cudaMalloc(&flush, fb);
    std::vector<long long> h((size_t)G * 4 * 4);
    const char* names[3] = {"row-per-thread", "coalesced", "bulk-copy"};
    uint32_t epoch = 0;
    for (int pat = 0; pat < 3; ++pat) {
        std::vector<double> ph[4];
        for (int rep = 0; rep < 20; ++rep) {
            cudaMemset(flush, rep, fb);                      // cold L2, like the flushed protocol
            ++epoch;
            if (pat == 0) k_handoff<0><<<G, 128>>>(slots, flags, epoch, out);
            if (pat == 1) k_handoff<1><<<G, 128>>>(slots, flags, epoch, out);
            if (pat == 2) k_handoff<2><<<G, 128>>>(slots, flags, epoch, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            if (rep < 2) continue;
            cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
            for (int i = 0; i < G * 4; ++i)
                for (int k = 0; k < 4; ++k) ph[k].push_back((double)h[i * 4 + k]);
        }
        printf("%-15s", names[pat]);
        const char* pn[4] = {"write", "publish", "wait", "read"};
        for (int k = 0; k < 4; ++k) {
            std::sort(ph[k].begin(), ph[k].end());
            printf("  %s med %6.0f p90 %6.0f cyc", pn[k], ph[k][ph[k].size() / 2], ph[k][ph[k].size() * 9 / 10]);
        }
        printf("\n");
    }
    return 0;
}
