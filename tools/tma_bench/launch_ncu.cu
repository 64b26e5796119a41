// Device-side launch cost under ncu (gpu__time_duration): an empty 148 x 256 kernel with 0 / 208 KB of
// dynamic SMEM, + a TMEM alloc/relinquish/dealloc of 128 columns, + 3 CUtensorMap and a 1 KB struct of
// __grid_constant__ parameters.  3 launches each.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc launch_ncu.cu -o /tmp/launch_ncu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "ptx.cuh"
using namespace xtc;
struct Big { CUtensorMap a, b, c; unsigned char pad[1024]; };
template <bool TMEM, bool BIG>
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ Big m, int* sink) {

    __shared__ uint32_t slot;
    if (TMEM) {
        if (threadIdx.x < 32) { ptx::tmem_alloc<1>(&slot, 128); ptx::tmem_relinquish<1>(); }
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
        if (threadIdx.x < 32) ptx::tmem_dealloc<1>(slot, 128);
    }
    if (BIG && threadIdx.x == 0 && m.pad[blockIdx.x & 1023] == 7) sink[0] = 1;
}
template <bool T, bool B>
void run(int smem, const Big& m, int* sink) {
    cudaFuncSetAttribute(k<T, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int i = 0; i < 3; ++i) k<T, B><<<148, 256, smem>>>(m, sink);
    cudaDeviceSynchronize();
}
int main() {
    int* sink; cudaMalloc(&sink, 8);
    Big m{}; 
    run<false, false>(0, m, sink);
    run<false, false>(208 * 1024, m, sink);
    run<true, false>(0, m, sink);
    run<true, false>(208 * 1024, m, sink);
    run<true, true>(208 * 1024, m, sink);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
