// Microbenchmark: cost of reading %globaltimer and %clock64 from a warp (cycles per read),
// and of a 9-iteration trivial loop with / without a %globaltimer read per iteration.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2512_16512_b200/csrc timer_cost.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

__global__ void k(unsigned long long* out, int n) {
    if (threadIdx.x != 0) return;
    unsigned long long acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc += xtc::ptx::globaltimer();
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) acc += clock64();
    long long t2 = clock64();
    volatile int sink = 0;
    for (int i = 0; i < n; ++i) sink = sink + i;
    long long t3 = clock64();
    out[0] = (t1 - t0) / n;
    out[1] = (t2 - t1) / n;
    out[2] = (t3 - t2) / n;
    out[3] = acc;
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 32);
    unsigned long long h[4];
    for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 32>>>(d, 1000);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    }
    printf("cycles per %%globaltimer read: %llu\ncycles per clock64 read: %llu\ncycles per trivial loop iteration (volatile): %llu\n",
           h[0], h[1], h[2]);
    return 0;
}
