// stream_k.cuh -- split applied to the flattened (output tile, k-block) loop:
// split_k_mode = XTC_SPLITK_STREAM ("stream-K").
//
// The persistent grid of G CTAs divides the I = tiles x kb_total iterations of the tile loop
// nest into G contiguous ranges [s_g, e_g), s_g = floor(I g / G): every CTA gets the same
// number of k-blocks (+-1) whatever the tile count, so no CTA idles for a partial last wave
// (the paper's "last block may contain fewer iterations", taken over the whole grid).
// A range can start and end inside a tile.  Per CTA:
//   * its first tile, when the range starts inside it (kb0 > 0), is a CONTRIBUTION: the
//     epilogue writes the fp32 partial to the CTA's slot of the workspace and publishes it
//     (per epilogue warp: fence, then flag[g][warp] = epoch of this launch);
//   * its last tile, when the range ends inside it (kb0 == 0, kb1 < kb_total), is OWNED: the
//     epilogue waits for the flags of the CTAs g+1 .. g_last that hold the rest of the tile's
//     k-blocks and adds their partials, in ascending k order, to its own accumulator before
//     the consumer and the single rounding;
//   * every other tile is complete and takes the normal epilogue.
// A contributor publishes at the start of its range and never waits, so the owner's waits
// cannot deadlock once all G CTAs are resident (G <= #SMs, cooperative launch).
#pragma once
#include <stdint.h>
#include "ptx.cuh"
#include "xtc_internal.h"

namespace xtc {

// [s, e) of CTA g (of G) over I iterations
__device__ __forceinline__ void sk_range(int64_t I, int64_t G, int64_t g, int64_t& s, int64_t& e) {
    s = I * g / G;
    e = I * (g + 1) / G;
}

// the CTA whose range holds iteration i
__device__ __forceinline__ int64_t sk_owner_of(int64_t I, int64_t G, int64_t i) {
    return ((i + 1) * G + I - 1) / I - 1;
}

__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// lane 0 of epilogue warp q of the owner: wait until every contributor c in (g, g_last] has
// published its warp-q rows for this launch
__device__ __forceinline__ void sk_wait(const uint32_t* flags, int64_t g, int64_t g_last, int q, uint32_t epoch) {
    for (int64_t c = g + 1; c <= g_last; ++c) {
        const uint32_t* f = flags + c * 4 + q;
        if (ld_acquire_gpu(f) == epoch) continue;
        const uint64_t t0 = ptx::globaltimer();
        uint32_t n = 0;
        while (ld_acquire_gpu(f) != epoch) {
            __nanosleep(32);
            if ((++n & 1023u) == 0 && ptx::globaltimer() - t0 > XTC_WATCHDOG_NS) {
                printf("xtc watchdog: stream-K partial of CTA %lld never published (block %d)\n", (long long)c,
                       blockIdx.x);
                __trap();
            }
        }
    }
}

// lane 0 of epilogue warp q of a contributor, after the warp's partial stores (+ __syncwarp)
__device__ __forceinline__ void sk_publish(uint32_t* flags, int64_t g, int q, uint32_t epoch) {
    ptx::fence_acq_rel_gpu();
    st_relaxed_gpu(flags + g * 4 + q, epoch);
}

}  // namespace xtc
