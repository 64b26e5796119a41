// gemm_tc.cuh -- KB2/KB3: schedule-parametrised tcgen05 GEMM and implicit-GEMM
// conv2d for sm_100a (bf16 kind::f16 / tf32 kind::tf32, fp32 accumulate in TMEM).
//
// How the paper's primitives (Table I) appear in this kernel:
//   strip_mine  -> CTA tile 128 x tile_n x tile_k (CTA pair: 256 x tile_n); UMMA atom
//                  (128|256) x tile_n x 16 (8 for tf32)
//   interchange -> tile order (TileMap: MN / NM + grouped raster)
//   unroll      -> the tile_k / UMMA_K MMAs of one stage are issued back to back
//   vectorize   -> the innermost tile is one tcgen05.mma (the tensor core is the SIMD unit)
//   parallelize -> one CTA (pair) per tile, or persistent CTAs striding over tiles;
//                  cluster_m = 2 pairs two SMs on one 256-row tile (cta_group::2)
//   split       -> split_k contiguous K segments, fp32 partials + ordered reduction
//   pack        -> TMA -> `stages`-deep SMEM ring in the 128-byte-swizzled layout the
//                  UMMA reads ("copies the elements ... in the order of their access",
//                  P:549-557; the swizzle plays the role of the paper's anti-conflict pad)
//   bufferize   -> accumulator in TMEM (acc_buffers deep); output staged in SMEM and
//                  written back by TMA store ("copied to the output tensor, while modifying
//                  its ordering to fit the original layout")
//
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one thread;
// leader CTA only for pairs), warp 2 = TMEM allocator, warp 3 idle, warps 4..7 =
// epilogue (TMEM lane quarters).
//
// CTA pair (CG = 2): each CTA loads its own 128 rows of A and its tile_n/2 columns
// of B; both CTAs' TMA bytes are counted on the LEADER's full barrier; the leader's
// single thread issues cta_group::2 MMAs (M = 256) whose commits are multicast to
// the empty / tmem-full barriers of both CTAs; each CTA's epilogue drains its own
// 128 TMEM lanes and arrives on the leader's tmem-empty barrier.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <type_traits>
#include "consumer.cuh"
#include "ptx.cuh"
#include "splitk_cluster.cuh"
#include "stream_k.cuh"
#include "xtc_internal.h"

namespace xtc {

// xtc_run_multicast write-out: `nboxes` (1 or 4) staged boxes of 32 rows x 128 bytes at box0 (box b
// at box0 + b * kTcEpiStageBytes; row i at i * 128 with logical 16-byte chunk j at (j ^ (i & 7)) * 16,
// the 128-byte swizzle of the TMA-store staging) are read back by the whole warp and written as
// 16-byte vectors to rows row0.., columns col0.. of p.mc: with 4 boxes each warp instruction writes
// one 512-byte row segment, with 1 box four 128-byte rows.
__device__ __forceinline__ void mc_store_boxes(const TcParams& p, const uint8_t* box0, int nboxes, int64_t row0,
                                               int64_t col0, int lane) {
    const int os = p.out_bf16 ? 2 : 4;
    const int j = lane & 7;
    const int b = nboxes == 4 ? (lane >> 3) : 0;
    const int sub = nboxes == 4 ? 0 : (lane >> 3);
    const int step = nboxes == 4 ? 1 : 4;
    const int64_t c = col0 + (int64_t)b * (128 / os) + j * (16 / os);
    if (c >= p.N) return;
    uint8_t* const base = static_cast<uint8_t*>(p.mc);
    for (int i = sub; i < 32; i += step) {
        const uint4 w = *reinterpret_cast<const uint4*>(box0 + b * kTcEpiStageBytes + i * 128 + ((j ^ (i & 7)) << 4));
        void* dst = base + ((row0 + i) * p.mc_ld + c) * os;
        if (p.mc_mode == 2) {
            if (os == 2) ptx::multimem_st_v4_bf16x2(dst, w);
            else ptx::multimem_st_v4_f32(dst, w);
        } else {
            ptx::st_global_v4(dst, w);
        }
    }
}

// LEAN: no stream-K, cluster split-K, cluster_n multicast, split partials, atomics or fused
// gather / multicast write-out -- those paths compiled out (smaller code for the per-tile roles)
template <bool TF32, bool CONV, int CG, bool SPLIT3, int MS, bool LEAN = false>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, const TcParams p) {
    constexpr int ATOM = TF32 ? 32 : 64;     // elements per 128-byte row (A's K / B's N)
    constexpr int UMMA_K = TF32 ? 8 : 16;    // K per tcgen05.mma (32 bytes)
    // MS M-subtiles per CTA (tile_m = 128 * CG * MS): the CTA holds 128*MS rows of A, and each
    // k-step issues MS UMMAs (one per 128-row subtile) sharing the B operand into MS TMEM
    // accumulators of tile_n columns -- B is loaded once per MS*128 rows
    constexpr uint32_t A_ATOM_BYTES = 128 * MS * 128;
    constexpr int TILE_M = 128 * CG * MS;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    const int S = p.stages;
    // [resident B (b_resident only)][A ring][B ring (unless resident)][epilogue staging][barriers]
    const bool b_res = p.b_resident != 0;
    uint8_t* sBres = smem;
    uint8_t* sA = smem + (b_res ? (size_t)p.kb_total * p.b_stage_bytes : 0);
    uint8_t* sB = sA + (size_t)S * p.a_stage_bytes;
    // SPLIT3 (3xTF32): the lo rings (A_lo, B_lo) follow the B ring, p.lo_off bytes after their hi rings
    uint8_t* sC = sB + (b_res ? 0 : (size_t)S * p.b_stage_bytes) + (SPLIT3 ? (size_t)p.lo_off : 0);
    uint64_t* full = reinterpret_cast<uint64_t*>(sC + (p.buffer_c ? (p.ovl ? 2 * kTcEpiSmem : kTcEpiSmem) : 0));
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint64_t* tempty = tfull + 2;
    uint64_t* bfull = tempty + 2;            // resident B landed
    uint64_t* split = bfull + 1;             // SPLIT3: lo parts of stage s written (warps 2 and 3)
    uint64_t* ksig = split + 8;              // cluster split-K: partials-written signals (2, by tile parity)
    uint64_t* tready = ksig + 2;             // TMEM allocated (its address is in tmem_slot)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tready + 1);

    if (p.trace && blockIdx.x < kTraceCtas && threadIdx.x == 0)
        p.trace[(size_t)blockIdx.x * kTraceSlots] = ptx::globaltimer();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0u;
    // cluster_n (CG = 1): cn CTAs on adjacent N tiles of one M tile; CTA crank loads rows
    // [crank*128/cn, (crank+1)*128/cn) of every A stage and multicasts them to all cn CTAs
    const int cn = (!LEAN && CG == 1) ? p.cn : 1;
    const bool mcast = cn > 1;
    const uint32_t crank = mcast ? ptx::cluster_ctarank() : 0u;
    const uint16_t cmask = (uint16_t)((1u << cn) - 1u);
    // cluster split-K (split_k_mode XTC_SPLITK_CLUSTER, CG = 1, cn = 1): the ksc CTAs of a
    // cluster run the ksc K segments of one output tile; CTA rank = segment
    const int ksc = (!LEAN && CG == 1 && cn == 1 && p.ksc > 1) ? p.ksc : 1;
    const bool kclu = ksc > 1;
    const uint32_t krank = kclu ? ptx::cluster_ctarank() : 0u;
    const int64_t cluster_id = blockIdx.x / (CG * cn * ksc);
    const int64_t num_clusters = gridDim.x / (CG * cn * ksc);
    // The tiles this CTA (cluster) visits and the k-block range of each: data-parallel (strided
    // over the tile map; K segment from the split or the cluster rank), or stream-K (a contiguous
    // range of the flattened (tile, k-block) space, stream_k.cuh).  Every role walks the same list.
    const bool sk = !LEAN && p.sk != 0;
    const int n_gather = LEAN ? 0 : p.n_gather;    // fused all-gather destinations (xtc_run_gather)
    const int mc_mode = LEAN ? 0 : p.mc_mode;      // multicast write-out (xtc_run_multicast)
    const bool atomic_k = !LEAN && p.atomic != 0;    // atomic split-K
    int64_t sk_s = 0, sk_e = 0;
    if (sk) sk_range(p.sk_iters, num_clusters, cluster_id, sk_s, sk_e);
    const int64_t n_walk = sk ? (sk_e > sk_s ? (sk_e - 1) / p.kb_total - sk_s / p.kb_total + 1 : 0)
                              : (p.num_tiles > cluster_id ? (p.num_tiles - cluster_id + num_clusters - 1) / num_clusters
                                                          : 0);
    auto tile_at = [&](int64_t i, int& mb, int& nb, int& ks, int& kb0, int& kb1) -> int64_t {
        int64_t t;
        if (sk) {
            t = sk_s / p.kb_total + i;
            const int64_t base = t * p.kb_total;
            kb0 = (int)(sk_s > base ? sk_s - base : 0);
            kb1 = (int)(sk_e - base < p.kb_total ? sk_e - base : p.kb_total);
            tile_coords(p.tm, t, mb, nb, ks);
            ks = 0;
        } else {
            t = cluster_id + i * num_clusters;
            tile_coords(p.tm, t, mb, nb, ks);
            if (kclu) ks = (int)krank;
            kb0 = ks * p.kb_per_split;
            kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        }
        return t;
    };
    const int bn_cta = p.tile_n / CG;        // B columns this CTA loads

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        if (p.buffer_c) ptx::prefetch_tmap(&tmC);
    }
    if (warp == 1 && lane == 0) {
        // a multicast stage is free when all cn CTAs' MMAs have consumed it (cn commit arrivals)
        for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], (uint32_t)cn); }
        for (int a = 0; a < 2; ++a) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 4 * CG); }
        ptx::mbar_init(bfull, 1);
        if constexpr (SPLIT3) for (int s = 0; s < S; ++s) ptx::mbar_init(&split[s], 2);
        if (kclu) { ptx::mbar_init(&ksig[0], 4u * ksc); ptx::mbar_init(&ksig[1], 4u * ksc); }
        ptx::mbar_init(tready, 1);
        ptx::fence_mbarrier_init();
    }
    // Barriers first; the TMEM allocation (the first tcgen05 instruction, ~0.5-1 us on a cold
    // SM) is then taken by warp 2 while the producers already issue the first (HBM-cold)
    // stages.  Only the MMA issuer and the epilogue read the TMEM address: they wait on the
    // mbarrier tready, which warp 2 arrives on after the allocation.
    if (warp == 2 && p.debug_late_alloc) {
        ptx::tmem_alloc<CG>(tmem_slot, p.tmem_cols);
        ptx::tmem_relinquish<CG>();
        ptx::tc_fence_before();
    }
    if (CG == 2 || mcast || kclu) ptx::cluster_sync(); else __syncthreads();
    if (warp == 2 && p.debug_late_alloc) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tready);
    } else if (warp == 2) {
        ptx::tmem_alloc<CG>(tmem_slot, p.tmem_cols);
        ptx::tmem_relinquish<CG>();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tready);
    }
    auto tmem_address = [&]() -> uint32_t {     // warps 1 and 4..7, once, before any TMEM use
        ptx::mbar_wait(tready, 0);
        ptx::tc_fence_after();
        return *reinterpret_cast<volatile uint32_t*>(tmem_slot);
    };
    uint64_t* const trace = (p.trace && blockIdx.x < kTraceCtas) ? p.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
    if (trace && threadIdx.x == 0) trace[1] = ptx::globaltimer();
    int trace_k = 0;       // per-role counters (each role only touches its own slots)

    if (warp == 0 || ((warp == 2 || warp == 3) && warp - 1 < p.pack_warps)) {
        // ===================== TMA producer(s) (pack) =====================
        // pack_warps producers (warps 0, 2, 3) share the ring: the g-th k-block of this
        // CTA's tile sequence uses slot g % S and is issued by producer g % pack_warps.
        {
            const int pw = warp == 0 ? 0 : warp - 1;
            const int P = p.pack_warps;
            int g = 0;                    // k-blocks seen (trace index)
            int s = 0, rr = 0;            // slot g % S, producer g % P (incremental: no divisions)
            uint32_t use_par = 0;         // parity of (g / S)
            bool first_round = true;      // g < S: slot never filled before
            const uint32_t stage_bytes = p.a_stage_bytes + (b_res ? 0u : p.b_stage_bytes);
            const int n_a = p.tile_k / ATOM;
            const int n_b = bn_cta / ATOM;
            if (b_res && pw == 0) {
                // pack B once: every k-block of this CTA's B columns (single N tile, split_k 1)
                if (ptx::elect_one()) {
                    const uint32_t all = (uint32_t)p.kb_total * p.b_stage_bytes;
                    uint32_t bar_c = 0;
                    if constexpr (CG == 2) {
                        if (rank == 0) ptx::mbar_arrive_expect_tx(bfull, 2 * all);
                        bar_c = ptx::mapa_shared(ptx::smem_u32(bfull), 0);
                    } else {
                        ptx::mbar_arrive_expect_tx(bfull, all);
                    }
                    const int nc = bn_cta * (int)rank;
                    for (int kb = 0; kb < p.kb_total; ++kb)
                        if (p.b3d) {
                            uint8_t* dst = sBres + (size_t)kb * p.b_stage_bytes;
                            if constexpr (CG == 2) ptx::tma_load_3d_pair(&tmB, dst, bar_c, 0, kb * p.tile_k, nc / ATOM);
                            else ptx::tma_load_3d(&tmB, dst, bfull, 0, kb * p.tile_k, nc / ATOM);
                        } else
                        for (int b = 0; b < n_b; ++b) {
                            uint8_t* dst = sBres + (size_t)kb * p.b_stage_bytes + (size_t)b * p.tile_k * 128;
                            if constexpr (CG == 2) ptx::tma_load_2d_pair(&tmB, dst, bar_c, nc + b * ATOM, kb * p.tile_k);
                            else ptx::tma_load_2d(&tmB, dst, bfull, nc + b * ATOM, kb * p.tile_k);
                        }
                }
                __syncwarp();
            }
            for (int64_t it = 0; it < n_walk; ++it) {
                int mb, nb, ks, kb0, kb1;
                tile_at(it, mb, nb, ks, kb0, kb1);
                const int m0 = mb * TILE_M + 128 * MS * (int)rank;     // this CTA's 128*MS rows
                const int n0 = (nb * cn + (int)crank) * p.tile_n + bn_cta * (int)rank;  // this CTA's B columns
                int wq = 0, hp = 0, nimg = 0;
                if constexpr (CONV) {
                    const int pq = p.cg.P * p.cg.Q;
                    nimg = m0 / pq;
                    const int rem = m0 - nimg * pq;
                    const int pp = rem / p.cg.Q, qq = rem - pp * p.cg.Q;
                    hp = pp * p.cg.sh - p.cg.ph;      // filter-window origin of pixel m0
                    wq = qq * p.cg.sw - p.cg.pw;
                }
                // conv: (filter row r, filter col sx, channel c) of the next k-block, advanced
                // incrementally (no integer division in the issue loop)
                int c_run = 0, s_run = 0, r_run = 0;
                if constexpr (CONV) {
                    const int kc0 = kb0 * p.tile_k;
                    const int rs0 = kc0 / p.cg.C;
                    c_run = kc0 - rs0 * p.cg.C;
                    r_run = rs0 / p.cg.S;
                    s_run = rs0 - r_run * p.cg.S;
                }
                for (int kb = kb0; kb < kb1; ++kb) {
                    const int c_kb = c_run, s_kb = s_run, r_kb = r_run;
                    if constexpr (CONV) {
                        c_run += p.tile_k;
                        while (c_run >= p.cg.C) {
                            c_run -= p.cg.C;
                            if (++s_run == p.cg.S) { s_run = 0; ++r_run; }
                        }
                    }
                    const int cs = s;
                    const uint32_t cpar = use_par;
                    const bool mine = rr == pw, fresh = first_round;
                    trace_k = g < kTraceK ? g : kTraceK;
                    ++g;
                    if (++rr == P) rr = 0;
                    if (++s == S) { s = 0; use_par ^= 1u; first_round = false; }
                    if (!mine) continue;                       // warp-uniform
                    if (!fresh) ptx::mbar_wait(&empty[cs], cpar ^ 1u);   // first fill: the slot is free
                    if (trace && lane == 0 && trace_k < kTraceK) trace[8 + trace_k] = ptx::globaltimer();
                    // One lane issues while the other 31 wait at __syncwarp below: letting them
                    // run ahead into the next try_wait would suspend the warp (divergent paths
                    // of a warp are serialised) and throttle the issuing lane.
                    if (ptx::elect_one()) {
                    uint32_t bar_c = 0;
                    uint64_t* const fb = &full[cs];
                    if constexpr (CG == 2) {
                        if (rank == 0) ptx::mbar_arrive_expect_tx(fb, 2 * stage_bytes);
                        bar_c = ptx::mapa_shared(ptx::smem_u32(fb), 0);
                    } else {
                        ptx::mbar_arrive_expect_tx(fb, stage_bytes);
                    }
                    uint8_t* a_dst = sA + (size_t)cs * p.a_stage_bytes;
                    uint8_t* b_dst = sB + (size_t)cs * p.b_stage_bytes;
                    // 3-D maps: one TMA moves all atoms of the stage ({atom, rows, atom index} box
                    // lands as [atom][rows][128 B], the layout the UMMA descriptors walk)
                    const bool a_one = !CONV && p.a3d;
                    if (MS == 1 && mcast) {
                        // this CTA's 128/cn-row slice of every A atom, into the same offset of all cn CTAs
                        const int rows = 128 / cn;
                        for (int a = 0; a < n_a; ++a)
                            ptx::tma_load_2d_multicast(&tmA, a_dst + a * A_ATOM_BYTES + crank * rows * 128, fb,
                                                       kb * p.tile_k + a * ATOM, m0 + (int)crank * rows, cmask);
                    } else if (a_one) {
                        const int ka = kb * (p.tile_k / ATOM);
                        if constexpr (CG == 2) ptx::tma_load_3d_pair(&tmA, a_dst, bar_c, 0, m0, ka);
                        else ptx::tma_load_3d(&tmA, a_dst, fb, 0, m0, ka);
                    }
                    int c = c_kb, sx = s_kb, r = r_kb;       // conv: this atom's (r, s, c)
                    for (int a = 0; a < ((a_one || mcast) ? 0 : n_a); ++a) {
                        const int kc = kb * p.tile_k + a * ATOM;
                        if constexpr (CONV) {
                            if (a > 0) {
                                c += ATOM;
                                if (c == p.cg.C) {
                                    c = 0;
                                    if (++sx == p.cg.S) { sx = 0; ++r; }
                                }
                            }
                            if constexpr (CG == 2)
                                ptx::tma_load_im2col_4d_pair(&tmA, a_dst + a * A_ATOM_BYTES, bar_c, c, wq, hp, nimg,
                                                             (uint16_t)sx, (uint16_t)r);
                            else
                                ptx::tma_load_im2col_4d(&tmA, a_dst + a * A_ATOM_BYTES, fb, c, wq, hp, nimg,
                                                        (uint16_t)sx, (uint16_t)r);
                        } else {
                            if constexpr (CG == 2) ptx::tma_load_2d_pair(&tmA, a_dst + a * A_ATOM_BYTES, bar_c, kc, m0);
                            else ptx::tma_load_2d(&tmA, a_dst + a * A_ATOM_BYTES, fb, kc, m0);
                        }
                    }
                    if (!b_res && p.b3d) {
                        if constexpr (CG == 2) ptx::tma_load_3d_pair(&tmB, b_dst, bar_c, 0, kb * p.tile_k, n0 / ATOM);
                        else ptx::tma_load_3d(&tmB, b_dst, fb, 0, kb * p.tile_k, n0 / ATOM);
                    }
                    for (int b = 0; b < ((b_res || p.b3d) ? 0 : n_b); ++b) {
                        uint8_t* dst = b_dst + (size_t)b * p.tile_k * 128;
                        if constexpr (CG == 2) ptx::tma_load_2d_pair(&tmB, dst, bar_c, n0 + b * ATOM, kb * p.tile_k);
                        else ptx::tma_load_2d(&tmB, dst, fb, n0 + b * ATOM, kb * p.tile_k);
                    }
                    }   // elected lane
                    __syncwarp();
                }
            }
        }
    } else if (SPLIT3 && (warp == 2 || warp == 3)) {
        // ===================== 3xTF32 split: lo = a - tf32(a) =====================
        // kind::tf32 reads the hi part of an fp32 operand (the low 13 mantissa bits are
        // ignored); the lo part is written at the same offsets of the lo rings, so it
        // inherits the swizzled layout.  Warps 2 and 3 share each stage's A and B tiles.
        int s = 0;
        uint32_t ph = 0;
        const uint32_t lo_off = p.lo_off;
        auto split_buf = [&](uint8_t* hi, uint32_t bytes) {
            const uint4* src = reinterpret_cast<const uint4*>(hi);
            uint4* dst = reinterpret_cast<uint4*>(hi + lo_off);
            for (uint32_t i = (uint32_t)((warp - 2) * 32 + lane); i < bytes / 16; i += 64) {
                const uint4 x = src[i];
                uint4 l;
                l.x = __float_as_uint(__uint_as_float(x.x) - __uint_as_float(x.x & 0xFFFFE000u));
                l.y = __float_as_uint(__uint_as_float(x.y) - __uint_as_float(x.y & 0xFFFFE000u));
                l.z = __float_as_uint(__uint_as_float(x.z) - __uint_as_float(x.z & 0xFFFFE000u));
                l.w = __float_as_uint(__uint_as_float(x.w) - __uint_as_float(x.w & 0xFFFFE000u));
                dst[i] = l;
            }
        };
        for (int64_t it = 0; it < n_walk; ++it) {
            int mb, nb, ks, kb0, kb1;
            tile_at(it, mb, nb, ks, kb0, kb1);
            for (int kb = kb0; kb < kb1; ++kb) {
                ptx::mbar_wait(&full[s], ph);
                split_buf(sA + (size_t)s * p.a_stage_bytes, p.a_stage_bytes);
                split_buf(sB + (size_t)s * p.b_stage_bytes, p.b_stage_bytes);
                ptx::fence_proxy_async_smem();       // generic-proxy stores -> visible to the tensor core
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&split[s]);
                if (++s == S) { s = 0; ph ^= 1u; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (contraction) =====================
        const uint32_t tmem_base = tmem_address();
        // One elected lane runs each tile's whole k-loop (stage waits, UMMAs, commits); the
        // warp reconverges once per tile.  Loop bounds and strides are pinned in registers
        // and the atoms of a stage are a compile-time count (NA), so a stage is straight-line
        // code: with short UMMAs (N = 64: ~48 cycles) any per-stage branch or constant-bank
        // reload shows up directly in the tile time (profiles/r01_conv_halo_ab.txt).
        if (rank == 0) {
            const uint32_t b_lbo = (uint32_t)p.tile_k * 128u;   // stride between 128-byte N blocks of B
            // Descriptors of stage 0; stage s and each k-step only advance the 14-bit
            // start-address field (address >> 4), which never carries out of the field
            // because the whole SMEM window is < 256 KB.
            const uint64_t adesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sA), 16, 1024);
            // B is MN-major: LBO = stride between 128-byte N blocks, SBO = stride between
            // K-row groups (8 rows of 128 B for SW128; 4 rows for tf32's SW128_BASE32B)
            uint8_t* const b_base_ptr = b_res ? sBres : sB;
            const uint64_t bdesc0 = TF32 ? ptx::smem_desc_sw128(ptx::smem_u32(b_base_ptr), b_lbo, 512, 1)
                                         : ptx::smem_desc_sw128(ptx::smem_u32(b_base_ptr), b_lbo, 1024, 2);
            const uint32_t a_stage16 = ptx::pin(p.a_stage_bytes >> 4), b_stage16 = ptx::pin(p.b_stage_bytes >> 4);
            const uint32_t idesc = ptx::pin(p.idesc);
            const int Sring = ptx::pin(S), accb = ptx::pin(p.acc_buffers), tile_n = ptx::pin(p.tile_n);
            const uint32_t b_res_u = ptx::pin((uint32_t)(b_res ? 1 : 0));
            const uint32_t lo16 = ptx::pin(p.lo_off >> 4);     // SPLIT3: hi stage -> lo stage (16-byte units)
            if (b_res) ptx::mbar_wait(bfull, 0);     // resident B has landed (in both CTAs for a pair)
            // NA > 0: atoms per stage known at compile time; NA == 0: none (diagnostics);
            // NA < 0: runtime count n_a (other tile_k, and the traced variant)
            auto mma_loop = [&](auto na_c, auto trace_c, auto mc_c) {
                constexpr int NA = decltype(na_c)::value;
                constexpr bool TR = decltype(trace_c)::value;
                constexpr bool MC = decltype(mc_c)::value;   // cluster_n: stage release multicast to the cluster
                const int n_a = NA >= 0 ? NA : ptx::pin(p.tile_k / ATOM);
                int s = 0, acc = 0, tk = 0;
                uint32_t ph = 0, aph = 0;
                for (int64_t it = 0; it < n_walk; ++it) {
                    int mb, nb, ks, kb0, kb1;
                    tile_at(it, mb, nb, ks, kb0, kb1);
                    ptx::mbar_wait(&tempty[acc], aph ^ 1);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * MS * tile_n);
                        int s1 = s, tk1 = tk;
                        uint32_t ph1 = ph;
                        for (int kb = kb0; kb < kb1; ++kb) {
                            ptx::mbar_wait(&full[s1], ph1);
                            if constexpr (SPLIT3) ptx::mbar_wait(&split[s1], ph1);   // lo parts written
                            if constexpr (TR) {
                                if (tk1 < kTraceK) trace[8 + kTraceK + tk1] = ptx::globaltimer();
                                ++tk1;
                            }
                            ptx::tc_fence_after();
                            const uint64_t ad = adesc0 + (uint64_t)((uint32_t)s1 * a_stage16);
                            const uint64_t bd = bdesc0 + (uint64_t)((b_res_u ? (uint32_t)kb : (uint32_t)s1) * b_stage16);
                            const uint32_t acc0 = kb > kb0 ? 1u : 0u;
                            auto pass = [&](uint64_t ad_, uint64_t bd_, uint32_t first) {
#pragma unroll
                                for (int a = 0; a < (NA >= 0 ? NA : n_a); ++a) {
#pragma unroll
                                    for (int kk = 0; kk < ATOM / UMMA_K; ++kk) {
                                        const uint32_t krow = a * ATOM + kk * UMMA_K;
#pragma unroll
                                        for (int h = 0; h < MS; ++h)
                                            ptx::umma<TF32, CG>(d_tmem + (uint32_t)(h * tile_n),
                                                                ad_ + (uint64_t)((a * A_ATOM_BYTES + h * 128 * 128 + kk * 32) >> 4),
                                                                bd_ + (uint64_t)(krow * 8), idesc,
                                                                (a > 0 || kk > 0) ? 1u : first);
                                    }
                                }
                            };
                            if constexpr (SPLIT3) {
                                // small terms first: hi*lo + lo*hi, then hi*hi
                                pass(ad, bd + (uint64_t)lo16, acc0);
                                pass(ad + (uint64_t)lo16, bd, 1u);
                                pass(ad, bd, 1u);
                            } else {
                                pass(ad, bd, acc0);
                            }
                            if constexpr (MC) ptx::umma_commit_multicast(&empty[s1], cmask);   // ... in every CTA
                            else ptx::umma_commit<CG>(&empty[s1]);   // frees the SMEM slot(s) when these MMAs finish
                            if (++s1 == Sring) { s1 = 0; ph1 ^= 1u; }
                        }
                        ptx::umma_commit<CG>(&tfull[acc]);      // accumulator ready for the epilogue(s)
                    }
                    __syncwarp();
                    for (int kb = kb0; kb < kb1; ++kb)           // every lane tracks the ring position
                        if (++s == Sring) { s = 0; ph ^= 1u; }
                    if constexpr (TR) tk += kb1 - kb0;
                    if (++acc == accb) { acc = 0; aph ^= 1u; }
                }
            };
            using T0 = std::integral_constant<bool, false>;
            using T1 = std::integral_constant<bool, true>;
            const int n_a = p.tile_k / ATOM;
            bool issued = false;
            if constexpr (CG == 1 && !CONV && !SPLIT3) {
                if (mcast) {
                    if (trace) mma_loop(std::integral_constant<int, -1>{}, T1{}, T1{});
                    else if (n_a == 1) mma_loop(std::integral_constant<int, 1>{}, T0{}, T1{});
                    else if (n_a == 2) mma_loop(std::integral_constant<int, 2>{}, T0{}, T1{});
                    else mma_loop(std::integral_constant<int, -1>{}, T0{}, T1{});
                    issued = true;
                }
            }
            if (issued) {
            } else if (trace) mma_loop(std::integral_constant<int, -1>{}, T1{}, T0{});
            else if (p.debug_skip_mma & ~65536) mma_loop(std::integral_constant<int, 0>{}, T0{}, T0{});
            else if (n_a == 1) mma_loop(std::integral_constant<int, 1>{}, T0{}, T0{});
            else if (n_a == 2) mma_loop(std::integral_constant<int, 2>{}, T0{}, T0{});
            else if (n_a == 4) mma_loop(std::integral_constant<int, 4>{}, T0{}, T0{});
            else mma_loop(std::integral_constant<int, -1>{}, T0{}, T0{});
        }
    } else if (warp >= 4) {
        // ===================== epilogue (bufferize) =====================
        const uint32_t tmem_base = tmem_address();
        const int q = warp & 3;                        // TMEM lanes 32q..32q+31
        int acc = 0;
        uint32_t aph = 0;
        int buf = 0;
        ClusterSplitState kst;
        uint8_t* stage = sC + q * (kTcEpiStageBytes * kTcEpiBuffers);
        if (n_gather && lane == 0)
            for (int d = 0; d < n_gather; ++d) ptx::tmap_acquire(reinterpret_cast<const CUtensorMap*>(p.gather) + d);
        const bool to_ws = !LEAN && p.split_out != 0;
        const bool bf16_out = p.out_bf16 && !to_ws;
        for (int64_t it = 0; it < n_walk; ++it) {
            int mb, nb, ks, kb0, kb1;
            const int64_t t = tile_at(it, mb, nb, ks, kb0, kb1);
            const int m0t = mb * TILE_M + 128 * MS * (int)rank, n0 = (nb * cn + (int)crank) * p.tile_n;
            ptx::mbar_wait(&tfull[acc], aph);
            if (trace && warp == 4 && lane == 0 && trace_k < kTraceTiles) trace[8 + 2 * kTraceK + 2 * trace_k] = ptx::globaltimer();
            ptx::tc_fence_after();
            // stream-K: a tile this CTA's range starts inside is a contribution (its partial goes to the
            // CTA's workspace slot); one its range ends inside is owned (the later k-ranges' partials,
            // held by CTAs cluster_id+1 .. sk_last, are added in k order before the consumer)
            const bool sk_contrib = sk && kb0 > 0;
            const bool sk_own = sk && kb0 == 0 && kb1 < p.kb_total;
            int64_t sk_last = 0;
            if (sk_own) {
                sk_last = sk_owner_of(p.sk_iters, num_clusters, (t + 1) * p.kb_total - 1);
                if (trace && warp == 4 && lane == 0) trace[3] = ptx::globaltimer();   // XTC_TRACE: owner waits
                if (lane == 0) sk_wait(p.sk_flags, cluster_id, sk_last, q, p.sk_epoch);
                __syncwarp();
                if (trace && warp == 4 && lane == 0) trace[4] = ptx::globaltimer();
            }
            if constexpr (MS == 2 && !CONV) {
                if (p.ovl) {
                    // ---- overlapped epilogue: TMEM -> SMEM tile (subtile 1) + registers (subtile 0),
                    // TMEM released, then the TMA stores run while the next tile's MMAs do ----
                    uint8_t* big = sC + q * (4 * kTcEpiStageBytes);    // 4 boxes [32 rows][128 B] = 256 columns
                    // fused relu / bias on a 32-column chunk of output row `r`, before the rounding
                    auto consume = [&](uint32_t (&v)[32], int64_t r, int c) {
                        if (p.cons && r < p.M) {
                            const int64_t cc = (int64_t)n0 + c;
                            const int nc = (int)((p.N - cc) < 32 ? (p.N - cc) : 32);
                            if (nc > 0) apply_consumer32(v, p.cons, p.bias, p.C, true, r, p.ldc, cc, nc, true, true);
                        }
                    };
                    if (lane == 0) ptx::bulk_wait_read<0>();          // the previous tile's stores have read it
                    __syncwarp();
                    const uint32_t t_q = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * 2 * 256);
                    for (int c = 0; c < 256; c += 32) {
                        uint32_t v[32];
                        ptx::tmem_ld_32x32b_x32(t_q + (uint32_t)(256 + c), v);
                        ptx::tmem_ld_wait();
                        consume(v, m0t + 128 + 32 * q + lane, c);
                        uint8_t* rowp = big + (c >> 6) * kTcEpiStageBytes + lane * 128;
                        const int cbase = (c & 63) ? 4 : 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint4 w;
                            w.x = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
                            w.y = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                            w.z = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                            w.w = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                            *reinterpret_cast<uint4*>(rowp + (((cbase + j) ^ (lane & 7)) * 16)) = w;
                        }
                    }
                    uint32_t R[8][16];                                   // subtile 0, packed bf16x2
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        uint32_t v[32];
                        ptx::tmem_ld_32x32b_x32(t_q + (uint32_t)(32 * i), v);
                        ptx::tmem_ld_wait();
                        consume(v, m0t + 32 * q + lane, 32 * i);
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            R[i][j] = ptx::pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
                    }
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {                                     // TMEM free: the next tile's MMAs start
                        if constexpr (CG == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
                        else ptx::mbar_arrive(&tempty[acc]);
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    // the four 64-column boxes of 32 rows starting at `row`: to C, or (fused all-gather)
                    // to every destination at gather_row0 + row
                    auto store_rows = [&](int row) {
                        if (n_gather) {
                            const CUtensorMap* gm = reinterpret_cast<const CUtensorMap*>(p.gather);
                            for (int d = 0; d < n_gather; ++d)
                                for (int b = 0; b < 4; ++b)
                                    ptx::tma_store_3d(gm + d, big + b * kTcEpiStageBytes, n0 + 64 * b,
                                                      p.gather_row0 + row, 0);
                        } else {
                            for (int b = 0; b < 4; ++b)
                                ptx::tma_store_3d(&tmC, big + b * kTcEpiStageBytes, n0 + 64 * b, row, 0);
                        }
                        ptx::bulk_commit();
                    };
                    if (mc_mode) {                                     // subtile 1: rows m0t + 128 + 32q
                        mc_store_boxes(p, big, 4, p.gather_row0 + m0t + 128 + 32 * q, n0, lane);
                    } else if (lane == 0) {
                        store_rows(m0t + 128 + 32 * q);
                        ptx::bulk_wait_read<0>();                        // ... have read the SMEM tile
                    }
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        uint8_t* rowp = big + (i >> 1) * kTcEpiStageBytes + lane * 128;
                        const int cbase = (i & 1) ? 4 : 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint4 w = make_uint4(R[i][4 * j], R[i][4 * j + 1], R[i][4 * j + 2], R[i][4 * j + 3]);
                            *reinterpret_cast<uint4*>(rowp + (((cbase + j) ^ (lane & 7)) * 16)) = w;
                        }
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (mc_mode) {                                     // subtile 0: rows m0t + 32q
                        mc_store_boxes(p, big, 4, p.gather_row0 + m0t + 32 * q, n0, lane);
                        __syncwarp();                                    // read before the next tile's drain
                    } else if (lane == 0) {
                        store_rows(m0t + 32 * q);
                    }
                    if (trace && warp == 4 && lane == 0 && trace_k < kTraceTiles) trace[8 + 2 * kTraceK + 2 * trace_k++ + 1] = ptx::globaltimer();
                    if (++acc == p.acc_buffers) { acc = 0; aph ^= 1; }
                    continue;
                }
            }
            for (int h = 0; h < MS; ++h) {                 // M-subtiles: accumulator h holds rows m0t + 128h ..
            const int m0 = m0t + 128 * h;
            const int64_t row = (int64_t)m0 + 32 * q + lane;
            const uint32_t t_row = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)((acc * MS + h) * p.tile_n);
            for (int c = 0; c < p.tile_n; c += 32) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(t_row + c, v);
                ptx::tmem_ld_wait();
                // slot of tile_n/4 column groups x 128 rows (row = TMEM lane) of float4: a warp's 32 rows of one
                // group are 512 contiguous bytes, so partial stores and the owner's loads are coalesced
                if (sk_contrib) {
                    uint4* dst = reinterpret_cast<uint4*>(p.Wk + cluster_id * p.sk_slot) + (int64_t)(c / 4) * 128 + 32 * q + lane;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        dst[(int64_t)j * 128] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    continue;
                }
                if (sk_own) {                      // + the later k-ranges, ascending
                    for (int64_t g2 = cluster_id + 1; g2 <= sk_last; ++g2) {
                        const float4* src = reinterpret_cast<const float4*>(p.Wk + g2 * p.sk_slot) +
                                            (int64_t)(c / 4) * 128 + 32 * q + lane;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float4 w = __ldcg(src + (int64_t)j * 128);
                            v[4 * j] = __float_as_uint(__uint_as_float(v[4 * j]) + w.x);
                            v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + w.y);
                            v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + w.z);
                            v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + w.w);
                        }
                    }
                }
                if (p.cons && row < p.M) {         // fused consumer before the rounding
                    const int64_t cc = (int64_t)n0 + c;
                    const int nc = (int)((p.N - cc) < 32 ? (p.N - cc) : 32);
                    // atomic split-K: C is accumulated in place, the first segment adds the bias
                    if (nc > 0) apply_consumer32(v, p.cons, p.bias, p.C, bf16_out, row, p.ldc, cc, nc, !atomic_k,
                                                 !atomic_k || ks == 0);
                }
                if (p.buffer_c) {
                    // stage one 128-byte row per thread (swizzled), then one TMA store per warp
                    const bool first_half = !bf16_out || ((c & 63) == 0);
                    if (first_half) {
                        if (lane == 0) ptx::bulk_wait_read<1>();
                        __syncwarp();
                    }
                    uint8_t* rowp = stage + buf * kTcEpiStageBytes + lane * 128;
                    if (bf16_out) {
                        const int cbase = (c & 63) ? 4 : 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint4 w;
                            w.x = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
                            w.y = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                            w.z = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                            w.w = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                            const int phys = (cbase + j) ^ (lane & 7);
                            *reinterpret_cast<uint4*>(rowp + phys * 16) = w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            uint4 w = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                            const int phys = j ^ (lane & 7);
                            *reinterpret_cast<uint4*>(rowp + phys * 16) = w;
                        }
                    }
                    const bool last_half = !bf16_out || ((c & 63) == 32) || (c + 32 >= p.tile_n);
                    if (last_half) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (mc_mode) {
                            mc_store_boxes(p, stage + buf * kTcEpiStageBytes, 1, p.gather_row0 + m0 + 32 * q,
                                           bf16_out ? (n0 + (c & ~63)) : (n0 + c), lane);
                            __syncwarp();                        // read before the buffer is refilled
                        } else if (lane == 0) {
                            const int col = bf16_out ? (n0 + (c & ~63)) : (n0 + c);
                            if (n_gather) {
                                // fused all-gather: the staged chunk goes to every destination
                                // (this rank's C and its peers'), one bulk group for all
                                const CUtensorMap* gm = reinterpret_cast<const CUtensorMap*>(p.gather);
                                for (int d = 0; d < n_gather; ++d)
                                    ptx::tma_store_3d(gm + d, stage + buf * kTcEpiStageBytes, col,
                                                      p.gather_row0 + m0 + 32 * q, 0);
                            } else {
                                ptx::tma_store_3d(&tmC, stage + buf * kTcEpiStageBytes, col, m0 + 32 * q, to_ws ? ks : 0);
                            }
                            ptx::bulk_commit();
                        }
                        buf ^= 1;
                    }
                } else if (row < p.M) {
                    const int64_t col0 = (int64_t)n0 + c;
                    const int ncols = (int)((p.N - col0) < 32 ? (p.N - col0) : 32);
                    if (ncols > 0) {
                        if (to_ws) {
                            float* dst = p.Wk + ((int64_t)ks * p.M + row) * p.ws_ld + col0;
                            if (ncols == 32) {
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    reinterpret_cast<uint4*>(dst)[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                            } else {
                                #pragma unroll
                                for (int j = 0; j < 32; ++j) if (j < ncols) dst[j] = __uint_as_float(v[j]);
                            }
                        } else if (atomic_k) {
                            float* dst = reinterpret_cast<float*>(p.C) + row * p.ldc + col0;
                            #pragma unroll
                            for (int j = 0; j < 32; ++j) if (j < ncols) atomicAdd(dst + j, __uint_as_float(v[j]));
                        } else if (bf16_out) {
                            uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + col0;
                            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    uint4 w;
                                    w.x = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
                                    w.y = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                                    w.z = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                                    w.w = ptx::pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                                    reinterpret_cast<uint4*>(dst)[j] = w;
                                }
                            } else {
                                #pragma unroll
                                for (int j = 0; j < 32; ++j) if (j < ncols)
                                    dst[j] = (uint16_t)(ptx::pack_bf16x2(__uint_as_float(v[j]), 0.f) & 0xFFFFu);
                            }
                        } else {
                            float* dst = reinterpret_cast<float*>(p.C) + row * p.ldc + col0;
                            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    reinterpret_cast<uint4*>(dst)[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                            } else {
                                #pragma unroll
                                for (int j = 0; j < 32; ++j) if (j < ncols) dst[j] = __uint_as_float(v[j]);
                            }
                        }
                    }
                }
            }
            }   // M-subtiles
            if (sk_contrib) {                      // publish this warp's rows of the partial
                __syncwarp();
                if (lane == 0) sk_publish(p.sk_flags, cluster_id, q, p.sk_epoch);
                if (trace && warp == 4 && lane == 0) trace[5] = ptx::globaltimer();   // XTC_TRACE: published
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (trace && warp == 4 && lane == 0 && trace_k < kTraceTiles) trace[8 + 2 * kTraceK + 2 * trace_k++ + 1] = ptx::globaltimer();
            if (lane == 0) {                           // TMEM buffer free for the next tile
                if constexpr (CG == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
                else ptx::mbar_arrive(&tempty[acc]);
            }
            if (++acc == p.acc_buffers) { acc = 0; aph ^= 1; }
            if (kclu) {                                // the tile's K segments meet: ordered reduction
                const int64_t r0 = (int64_t)mb * TILE_M;
                const int64_t c0 = (int64_t)nb * p.tile_n;
                cluster_split_reduce(ksig, kst, ksc, (int)krank, p.Wk, p.M, p.ws_ld, r0,
                                     (int)(p.M - r0 < TILE_M ? p.M - r0 : TILE_M), c0,
                                     (int)(p.N - c0 < p.tile_n ? p.N - c0 : p.tile_n),
                                     p.C, p.ldc, p.out_bf16 != 0, p.cons_red, p.bias, (int)threadIdx.x - 128, p.buffer_c != 0, trace);
            }
        }
        // before the CTA exits its TMA stores must have READ the staging SMEM; their global writes complete
        // with the grid (what a later kernel or the host sees).  Waiting for the writes themselves put the
        // last tile's write latency on every launch's critical path.  (65536: A/B diagnostics, full wait.)
        if (p.buffer_c && lane == 0) {
            if (p.debug_skip_mma & 65536) ptx::bulk_wait<0>();
            else ptx::bulk_wait_read<0>();
        }
        if (trace && warp == 4 && lane == 0) trace[6] = ptx::globaltimer();   // XTC_TRACE: stores read
    }

    ptx::tc_fence_before();
    // (cluster_n: no CTA may exit while a peer can still multicast into its SMEM / barriers)
    if (CG == 2 || mcast || kclu) ptx::cluster_sync(); else __syncthreads();
    if (trace && threadIdx.x == 0) trace[2] = ptx::globaltimer();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<CG>(*reinterpret_cast<volatile uint32_t*>(tmem_slot), p.tmem_cols);
        if (trace && lane == 0) trace[7] = ptx::globaltimer();                // XTC_TRACE: TMEM released
    }
}

// ------------------------------------------------------------------ launch --
template <bool TF32, bool CONV, int CG, bool SPLIT3, int MS>
cudaError_t launch_tc_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                               const TcParams& p, int grid, int smem, cudaStream_t st) {
    // the lean variant for plain bf16 plans (no split / stream-K / multicast / gather)
    const bool lean = !TF32 && !SPLIT3 && !p.sk && p.ksc <= 1 && p.cn <= 1 && !p.split_out && !p.atomic &&
                      !p.n_gather && !p.mc_mode;
    auto k = lean ? tc_gemm_kernel<TF32, CONV, CG, SPLIT3, MS, !TF32 && !SPLIT3>
                  : tc_gemm_kernel<TF32, CONV, CG, SPLIT3, MS, false>;
    cudaError_t e = ensure_smem_attr(k, smem);
    if (e != cudaSuccess) return e;
    const int ksc = (CG == 1 && p.cn <= 1 && p.ksc > 1) ? p.ksc : 1;
    if (CG == 1 && p.cn <= 1 && ksc == 1 && !p.sk) {
        k<<<grid, kTcThreads, smem, st>>>(a, b, c, p);
    } else {
        if (ksc > 8) {
            e = ensure_nonportable_cluster(k);
            if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kTcThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        if (p.sk) {                 // stream-K owners wait for later CTAs: all of them must be resident
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = getenv("XTC_SK_NOCOOP") ? 0 : 1;   // (diagnostics: A/B of the attribute)
        } else {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = CG * (p.cn > 1 ? p.cn : 1) * ksc;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
        }
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, k, a, b, c, p);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

// The variants are instantiated in their own translation units (gemm_tc_*.cu) so that
// nvcc compiles them in parallel; gemm_tc.cu only dispatches.
#define XTC_TC_VARIANT(TF32, CONV, CG, SPLIT3, MS)                                                          \
    template cudaError_t launch_tc_t<TF32, CONV, CG, SPLIT3, MS>(const CUtensorMap&, const CUtensorMap&,   \
                                                                 const CUtensorMap&, const TcParams&, int, \
                                                                 int, cudaStream_t);
#define XTC_TC_EXTERN(TF32, CONV, CG, SPLIT3, MS) extern XTC_TC_VARIANT(TF32, CONV, CG, SPLIT3, MS)

}  // namespace xtc
