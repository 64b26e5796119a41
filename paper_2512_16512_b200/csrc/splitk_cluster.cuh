// splitk_cluster.cuh -- split with the reduction inside the contraction kernel:
// split_k_mode = XTC_SPLITK_CLUSTER.
//
// The split_k K segments of one output tile run on the split_k CTAs of ONE thread-block
// cluster (CTA rank s = segment s; a cluster is gang-scheduled, so all segments of a tile
// are resident together and may wait for each other).  Each CTA drains its TMEM partial
// into the fp32 workspace W[s][row][col] (the same layout as the ordered split-K), then
// signals every CTA of the cluster: each epilogue warp, after __syncwarp, has one lane fence
// (gpu scope) and arrive with release.cluster semantics on every CTA's signal barrier
// (4 x split_k arrivals complete a phase).  Once all split_k partials are in, CTA s reduces
// rows [s*rpc, (s+1)*rpc) of the tile, rpc = ceil(rows / split_k): W[0] + W[1] + ... in
// ascending segment order (the
// order of the separate reduction kernel, so both modes give bit-identical results),
// applies the fused consumer to the complete sum and rounds once.  No second kernel
// launch, and each CTA reads back only 1/split_k of the tile's partial planes.
//
// Two signal barriers alternate by tile parity: a CTA that finished tile i may already
// arrive for tile i+1 on a peer that is still waiting for a slower CTA's arrival for
// tile i; with one barrier that early arrival would complete the wrong phase.
#pragma once
#include <stdint.h>
#include "consumer.cuh"
#include "ptx.cuh"

namespace xtc {


struct ClusterSplitState {
    uint32_t parity = 0;                    // bit b: phase parity of signal barrier b
    int which = 0;                          // barrier of the next tile
};

// Called by all 128 epilogue threads (tid = 0..127) after their partial stores of this tile
// (direct stores, or -- tma_partials -- TMA stores issued by each warp's lane 0).
// rows [row0, row0 + nrows) of the output are the tile's valid rows (contiguous in C and W),
// cols [n0, n0 + ncols) its valid columns.
__device__ __forceinline__ void cluster_split_reduce(uint64_t* sig, ClusterSplitState& st, int ksc, int krank,
                                                     const float* __restrict__ W, int64_t M, int64_t ws_ld,
                                                     int64_t row0, int nrows, int64_t n0, int ncols, void* C,
                                                     int64_t ldc, bool out_bf16, int cons, const float* bias,
                                                     int tid, bool tma_partials, uint64_t* trace = nullptr) {
    // the warp's partial stores precede the signal: __syncwarp orders them before lane 0's
    // gpu-scope fence, and fence + relaxed cluster-scope arrives form the release (one fence for
    // all split_k arrives: a release.cluster arrive would pay a MEMBAR.ALL.GPU each)
    __syncwarp();
    uint64_t* bar = sig + st.which;
    if ((tid & 31) == 0) {
        if (tma_partials) {                  // this warp's TMA stores of its partial rows: complete,
            ptx::bulk_wait<0>();             // then ordered with the generic proxy of the readers
            ptx::fence_proxy_async_global();
        }
        ptx::fence_acq_rel_gpu();
        const uint32_t a = ptx::smem_u32(bar);
        for (int j = 0; j < ksc; ++j) ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(a, (uint32_t)j));
    }
    if (trace && tid == 0) trace[3] = ptx::globaltimer();       // XTC_TRACE: signal sent, peers' seen, done
    ptx::mbar_wait_cluster(bar, (st.parity >> st.which) & 1u);
    if (trace && tid == 0) trace[4] = ptx::globaltimer();
    st.parity ^= 1u << st.which;
    st.which ^= 1;

    const int rpc = (nrows + ksc - 1) / ksc;
    const int r_lo = krank * rpc;
    const int r_hi = min(nrows, r_lo + rpc);
    // 128 threads = (128 / gp) rows x gp four-column groups per pass, gp = pow2 >= groups: a warp
    // reads and writes whole row segments (coalesced); the segment sums are one short loop
    const int groups = (ncols + 3) >> 2;
    int gp = 1;
    while (gp < groups) gp <<= 1;
    const int g = tid & (gp - 1);
    const int rstep = 128 / gp;
    const int64_t plane = M * ws_ld;
    const int64_t col = n0 + 4 * g;
    const int cnt = min(4, ncols - 4 * g);
    const bool vec = ((ldc & 3) == 0) && ((n0 & 3) == 0) && cnt == 4 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
    if (gp <= 128 && cnt > 0) {
        for (int r = r_lo + tid / gp; r < r_hi; r += rstep) {
            const int64_t row = row0 + r;
            const float* src = W + row * ws_ld + col;
            float a[4];
            if (cnt == 4) {                                  // ws_ld is a multiple of 4: 16-byte loads
                float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
#pragma unroll 4
                for (int s = 1; s < ksc; ++s) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(src + s * plane));
                    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                }
                a[0] = acc.x; a[1] = acc.y; a[2] = acc.z; a[3] = acc.w;
            } else {
                for (int j = 0; j < cnt; ++j) {
                    float acc = __ldcg(src + j);
                    for (int s = 1; s < ksc; ++s) acc += __ldcg(src + s * plane + j);
                    a[j] = acc;
                }
            }
            const int64_t off = row * ldc + col;
            if (cons)
                for (int j = 0; j < cnt; ++j) a[j] = consume1(a[j], cons, bias, C, out_bf16, off + j, col + j);
            if (out_bf16) {
                uint16_t* dst = reinterpret_cast<uint16_t*>(C) + off;
                if (vec) *reinterpret_cast<uint2*>(dst) = make_uint2(ptx::pack_bf16x2(a[0], a[1]), ptx::pack_bf16x2(a[2], a[3]));
                else for (int j = 0; j < cnt; ++j) dst[j] = (uint16_t)(ptx::pack_bf16x2(a[j], 0.f) & 0xFFFFu);
            } else {
                float* dst = reinterpret_cast<float*>(C) + off;
                if (vec) *reinterpret_cast<float4*>(dst) = make_float4(a[0], a[1], a[2], a[3]);
                else for (int j = 0; j < cnt; ++j) dst[j] = a[j];
            }
        }
    }
    if (trace && tid == 0) trace[5] = ptx::globaltimer();
}

}  // namespace xtc
