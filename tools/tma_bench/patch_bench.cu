// Microbenchmark: TMA cost of the haloed conv patch (conv_halo.cu's A operand) on an
// L56-shaped NHWC tensor (32 x 56 x 56 x 64 bf16), 148 CTAs, one producer lane, a consumer
// lane re-arming the buffers (no MMA).  Variants:
//   box {64 ch, slots, rows, 1} at w0 = -1 or 0 (OOB zero fill on the left / right),
//   one box per patch vs one {64, slots, 1, 1} box per patch row,
//   S patches in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 patch_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ bool tw(uint32_t a, uint32_t par) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(a), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) { while (!tw(su32(b), par)) {} }

__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap tm, int rows, int slots, int w0,
                                            int per_row, int S, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
    const int patch = 128 * slots * rows;
    uint64_t* full = (uint64_t*)(base + S * patch);
    uint64_t* empty = full + 16;
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint64_t t0 = gt();
    if (w == 0 && l == 0) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % S, u = i / S;
            if (u > 0) wait(&empty[s], (u & 1) ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(patch) : "memory");
            const int tile = (blockIdx.x + 148 * i) % (32 * 28);
            const int n = tile / 28, p0 = (tile % 28) * 2;
            const uint32_t dst = su32(base + (size_t)s * patch);
            if (!per_row) {
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                    ::"r"(dst), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(w0), "r"(p0 - 1), "r"(n) : "memory");
            } else {
                for (int r = 0; r < rows; ++r)
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                        ::"r"(dst + r * 128 * slots), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(w0), "r"(p0 - 1 + r), "r"(n)
                        : "memory");
            }
        }
    }
    if (w == 7 && l == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            wait(&full[s], ph);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            if (++s == S) { s = 0; ph ^= 1; }
        }
        out[blockIdx.x] = gt() - t0;
    }
}

typedef CUresult (*EncT)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const size_t N = 32, H = 56, W = 56, C = 64;
    void* X;
    cudaMalloc(&X, N * H * W * C * 2);
    cudaMemset(X, 0, N * H * W * C * 2);
    EncT et;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&et, cudaEnableDefault, &q);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8);
    struct V { int rows, slots, w0, per_row; };
    const V vs[] = {{6, 64, -1, 0}, {6, 64, 0, 0}, {6, 56, 0, 0}, {4, 64, -1, 0}, {2, 64, -1, 0},
                    {6, 64, -1, 1}, {6, 56, 0, 1}, {4, 64, -1, 1}};
    for (const V& v : vs) {
        CUtensorMap tm;
        cuuint64_t dims[4] = {C, W, H, N}, str[3] = {C * 2, W * C * 2, H * W * C * 2};
        cuuint32_t box[4] = {64, (cuuint32_t)v.slots, (cuuint32_t)(v.per_row ? 1 : v.rows), 1}, es[4] = {1, 1, 1, 1};
        CUresult r = et(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int patch = 128 * v.slots * v.rows;
        for (int S : {1, 2, 4}) {
            const int smem = S * patch + 2048;
            if (smem > 232448) continue;
            const int iters = 64;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k<<<148, 256, smem>>>(tm, v.rows, v.slots, v.w0, v.per_row, S, 8, out);
            cudaDeviceSynchronize();
            k<<<148, 256, smem>>>(tm, v.rows, v.slots, v.w0, v.per_row, S, iters, out);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
            double tot = 0;
            for (int i = 0; i < 148; ++i) tot += h[i];
            tot /= 148;
            printf("box {64,%2d,%d,1}%s w0=%2d S=%d: %.3f us/patch  %6.1f GB/s/SM  %7.1f GB/s chip (%s)\n", v.slots,
                   v.per_row ? 1 : v.rows, v.per_row ? " x rows" : "       ", v.w0, S, tot / iters / 1e3,
                   iters * (double)patch / tot, 148.0 * iters * patch / tot, cudaGetErrorString(e));
        }
    }
    return 0;
}
