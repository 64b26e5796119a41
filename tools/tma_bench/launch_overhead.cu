// Launch-overhead microbenchmark: how long does an (almost) empty kernel take between two
// CUDA events, as a function of the launch configuration the tcgen05 kernels use?
//   variants: dynamic SMEM 0 / 100 KB / 206 KB, TMEM alloc+dealloc (256 cols), three
//   __grid_constant__ CUtensorMap parameters, 148 vs 25 CTAs.
// Each variant: 50 reps timed one by one (event pair per launch, a long device delay kernel
// in front so the host enqueue never starves the GPU) and 200 back-to-back launches between
// one event pair.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc launch_overhead.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#include "ptx.cuh"

using namespace xtc;

struct Maps { CUtensorMap a, b, c; };

__global__ void k_delay(unsigned long long ns) {
    const unsigned long long t0 = ptx::globaltimer();
    while (ptx::globaltimer() - t0 < ns) {}
}

// TMEM: 0 none, 1 alloc+relinquish+dealloc, 2 alloc+dealloc (no relinquish), 3 alloc 32 cols,
// 4 relinquish only, 5 alloc+relinquish+dealloc with no fences
template <int TMEM, bool MAPS>
__global__ void __launch_bounds__(256, 1) k_empty(const __grid_constant__ Maps m, int* sink) {
    extern __shared__ uint8_t smem[];
    __shared__ uint32_t slot;
    const uint32_t cols = TMEM == 3 ? 32 : 256;
    if constexpr (MAPS) {
        if (threadIdx.x == 0) { ptx::prefetch_tmap(&m.a); ptx::prefetch_tmap(&m.b); ptx::prefetch_tmap(&m.c); }
    }
    if constexpr (TMEM != 0) {
        if ((threadIdx.x >> 5) == 2) {
            if (TMEM != 4) ptx::tmem_alloc<1>(&slot, cols);
            if (TMEM != 2) ptx::tmem_relinquish<1>();
        }
        if (TMEM != 5) ptx::tc_fence_before();
        __syncthreads();
        if (TMEM != 5) ptx::tc_fence_after();
    }
    if (threadIdx.x == 0 && blockIdx.x == 100000) sink[0] = smem[0];
    if constexpr (TMEM != 0) {
        if (TMEM != 5) ptx::tc_fence_before();
        __syncthreads();
        if ((threadIdx.x >> 5) == 2 && TMEM != 4) {
            if (TMEM != 5) ptx::tc_fence_after();
            ptx::tmem_dealloc<1>(slot, cols);
        }
    }
}

template <int TMEM, bool MAPS>
static void run(const char* name, int grid, int smem, int* sink, const Maps& m) {
    auto k = k_empty<TMEM, MAPS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t st;
    cudaStreamCreate(&st);
    std::vector<cudaEvent_t> ev(102);
    for (auto& e : ev) cudaEventCreate(&e);
    for (int i = 0; i < 5; ++i) k<<<grid, 256, smem, st>>>(m, sink);
    k_delay<<<1, 1, 0, st>>>(2000000);
    for (int i = 0; i < 50; ++i) {
        cudaEventRecord(ev[2 * i], st);
        k<<<grid, 256, smem, st>>>(m, sink);
        cudaEventRecord(ev[2 * i + 1], st);
    }
    cudaStreamSynchronize(st);
    std::vector<float> t(50);
    for (int i = 0; i < 50; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
    std::sort(t.begin(), t.end());
    k_delay<<<1, 1, 0, st>>>(3000000);
    cudaEventRecord(ev[100], st);
    for (int i = 0; i < 200; ++i) k<<<grid, 256, smem, st>>>(m, sink);
    cudaEventRecord(ev[101], st);
    cudaStreamSynchronize(st);
    float tb = 0;
    cudaEventElapsedTime(&tb, ev[100], ev[101]);
    printf("%-34s grid %3d smem %6d: single launch med %.2f us (min %.2f)  back-to-back %.2f us/launch  %s\n", name, grid,
           smem, t[25] * 1e3, t[0] * 1e3, tb * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(st);
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4);
    Maps m;
    memset(&m, 0, sizeof m);
    for (int grid : {148}) {
        run<0, false>("empty", grid, 206 * 1024, sink, m);
        run<1, false>("alloc+relinquish+dealloc", grid, 206 * 1024, sink, m);
        run<2, false>("alloc+dealloc", grid, 206 * 1024, sink, m);
        run<3, false>("alloc 32 cols", grid, 206 * 1024, sink, m);
        run<4, false>("relinquish only", grid, 206 * 1024, sink, m);
        run<5, false>("no tcgen05 fences", grid, 206 * 1024, sink, m);
        run<0, false>("empty 0 smem", grid, 0, sink, m);
        run<1, false>("alloc.. 0 smem", grid, 0, sink, m);
    }
    return 0;
}
