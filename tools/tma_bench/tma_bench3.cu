// Microbenchmark 3: TMA throughput per SM for the conv A operand:
//   mode 0: 2-D tiled box {64 ch, 128 rows} over the NHWC tensor viewed as [N*H*W][C]
//   mode 1: 4-D tiled box {64 ch, 64 w, 2 h, 1 n} (a 2-row output patch, OOB zero fill)
//   mode 2: im2col box, 128 pixels x 64 channels, 3x3 pad 1 (the current conv producer)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ bool tw(uint32_t a, uint32_t par) { uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(a), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) { while (!tw(su32(b), par)) {} }
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap tm, int mode, int S, int iters, int P, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  const int stage_bytes = 16384;
  uint64_t* full = (uint64_t*)(base + S * stage_bytes);
  uint64_t* empty = full + 16;
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&full[s]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&empty[s]))); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint64_t t0 = gt();
  if (w < P && l == 0) {
    for (int i = w; i < iters; i += P) {
      int s = i % S; int u = i / S;
      if (u > 0) wait(&empty[s], (u & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(stage_bytes) : "memory");
      int tile = (blockIdx.x + 148 * (i / 9)) % 784, tap = i % 9, r = tap / 3, sx = tap % 3;
      int n = tile / 28, p0 = (tile % 28) * 2;          // 2-row patch of a 56x56 image
      uint32_t dst = su32(base + s * stage_bytes);
      if (mode == 0) {
        int row = tile * 128;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     :: "r"(dst), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(row) : "memory");
      } else if (mode == 1) {
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                     :: "r"(dst), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(sx - 1), "r"(p0 + r - 1), "r"(n) : "memory");
      } else {
        int m0 = tile * 128, nn = m0 / 3136, rem = m0 % 3136, pp = rem / 56, qq = rem % 56;
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};"
                     :: "r"(dst), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(qq - 1), "r"(pp - 1), "r"(nn), "h"((uint16_t)sx), "h"((uint16_t)r) : "memory");
      }
    }
  }
  if (w == 7 && l == 0) {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait(&full[s], ph);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[s])) : "memory");
      if (++s == S) { s = 0; ph ^= 1; }
    }
    out[blockIdx.x] = gt() - t0;
  }
}
typedef CUresult (*EncT)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncI)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const size_t N = 32, H = 56, W = 56, C = 64;
  void* X; cudaMalloc(&X, N * H * W * C * 2); cudaMemset(X, 0, N * H * W * C * 2);
  EncT et; EncI ei; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&et, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&ei, cudaEnableDefault, &q);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  const char* names[3] = {"2-D tiled {64ch,128rows}", "4-D tiled {64ch,64w,2h,1n} patch", "im2col 128px x 64ch"};
  for (int mode = 0; mode < 3; ++mode) {
    CUtensorMap tm;
    cuuint32_t es4[4] = {1, 1, 1, 1};
    if (mode == 0) {
      cuuint64_t dims[2] = {C, N * H * W}, str[1] = {C * 2}; cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
      et(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (mode == 1) {
      cuuint64_t dims[4] = {C, W, H, N}, str[3] = {C * 2, W * C * 2, H * W * C * 2}; cuuint32_t box[4] = {64, 64, 2, 1};
      et(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, X, dims, str, box, es4, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[4] = {C, W, H, N}, str[3] = {C * 2, W * C * 2, H * W * C * 2}; int lo[2] = {-1, -1}, hi[2] = {-1, -1};
      ei(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, X, dims, str, lo, hi, 64, 128, es4, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int P : {1, 2, 4}) for (int S : {8, 12}) {
      int smem = S * 16384 + 2048, iters = 900;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k<<<148, 256, smem>>>(tm, mode, S, 36, P, out); cudaDeviceSynchronize();
      k<<<148, 256, smem>>>(tm, mode, S, iters, P, out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<unsigned long long> h(148); cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
      double tot = 0; for (int i = 0; i < 148; ++i) tot += h[i]; tot /= 148;
      printf("%-36s P=%d S=%2d: %6.1f GB/s/SM  %.3f us/stage (%s)\n", names[mode], P, S, iters * 16384.0 / tot, tot / iters / 1e3, cudaGetErrorString(e));
    }
  }
  return 0;
}
