// Microbenchmark 2: does TMA issue rate scale with the number of issuing warps?
// P producer warps each issue nbox/P of the stage's boxes (full barrier count = P).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ bool tw(uint32_t a, uint32_t par) { uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(a), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) { while (!tw(su32(b), par)) {} }
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap tm, int S, int nbox, int rows, int iters, int P, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  const int box_bytes = rows * 128, stage_bytes = box_bytes * nbox;
  uint64_t* full = (uint64_t*)(base + S * stage_bytes);
  uint64_t* empty = full + 16;
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&full[s])), "r"(P)); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&empty[s]))); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint64_t t0 = gt();
  if (w < P && l == 0) {
    int s = 0; uint32_t ph = 0;
    const int per = nbox / P;
    for (int i = 0; i < iters; ++i) {
      if (i >= S) wait(&empty[s], ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(per * box_bytes) : "memory");
      for (int bb = 0; bb < per; ++bb) {
        int b = w * per + bb;
        int x = ((blockIdx.x * 7 + i * 3 + b) % 64) * 64, y = ((blockIdx.x * 13 + i) % 32) * rows;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     :: "r"(su32(base + s * stage_bytes + b * box_bytes)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(x), "r"(y) : "memory");
      }
      if (++s == S) { s = 0; ph ^= 1; }
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
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* A; size_t MB = 64; cudaMalloc(&A, 8192ull * 8192 * 2); cudaMemset(A, 0, 8192ull * 8192 * 2);
  Enc enc; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  // {S, nbox, rows, P}
  int cfgs[][4] = {{8,2,128,1},{8,2,128,2},{6,4,64,1},{6,4,64,2},{6,4,64,4},{12,1,128,1},{12,2,64,2},{3,4,128,1},{3,4,128,2},{3,4,128,4}};
  for (auto& c : cfgs) {
    int S = c[0], nbox = c[1], rows = c[2], P = c[3];
    CUtensorMap tm; cuuint64_t dims[2] = {8192, 8192}, str[1] = {8192 * 2}; cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int smem = S * nbox * rows * 128 + 2048; int iters = 2000;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 256, smem>>>(tm, S, nbox, rows, 50, P, out); cudaDeviceSynchronize();
    k<<<148, 256, smem>>>(tm, S, nbox, rows, iters, P, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148); cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    double tot = 0; for (int i = 0; i < 148; ++i) tot += h[i]; tot /= 148;
    double bytes = (double)iters * nbox * rows * 128;
    printf("S=%2d nbox=%d rows=%3d P=%d (%3d KB/stage, %3d KB ring): %6.1f GB/s/SM, %.3f us/stage (%s)\n", S, nbox, rows, P,
           nbox * rows * 128 / 1024, S * nbox * rows * 128 / 1024, bytes / tot, tot / iters / 1e3, cudaGetErrorString(e));
  }
  return 0;
}
