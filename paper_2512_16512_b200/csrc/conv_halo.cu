// conv_halo.cu -- KB3h: stride-1 conv2d as implicit GEMM with the input packed once per
// output tile (schedule knob pack_halo = 1), sm_100a tcgen05 (bf16 kind::f16 / tf32).
//
// The paper's pack primitive copies "the elements used below a given loop
// level ... in the order of their access".  The im2col kernel (gemm_tc.cu) packs at the
// k-block level: every filter tap (r, s) re-loads a 128 x C pixel block through the TMA
// im2col unit, 9 loads per tile for a 3x3 filter.  Here the pack sits at the output-tile
// level, above the (r, s, c) reduction loops: the tile's input window (tile rows + R - 1
// rows of Wp pixel slots, zero-filled outside the image by TMA) is loaded once, and tap
// (r, s) of virtual row v is patch row v + r*Wp + s -- the UMMA A operand of that tap is
// the patch advanced by (r*Wp + s) 128-byte rows.  The 128-byte swizzle is anchored to
// absolute SMEM addresses, so such views need no descriptor base offset
// (profiles/r01_umma_row_shift_microtest.txt).
//
// Virtual rows: a 128-row UMMA tile is 128/Wp output rows x Wp slots, Wp the power of two
// >= Q + S - 1.  Slots q >= Q and rows p >= P hold don't-care values and are never
// written: the TMA store box {f, q, p, n} is clipped at the tensor edges, direct stores
// test the bounds.
//
// Warp roles (256 threads): warp 0 = patch producer, warp 3 = B (filter) producer (ring,
// or the whole filter once with b_resident), warp 1 = MMA issuer, warp 2 = TMEM
// allocator, warps 4..7 = epilogue (TMEM lane quarters).
#include <cuda.h>
#include <cuda_runtime.h>
#include "consumer.cuh"
#include "ptx.cuh"
#include "splitk_cluster.cuh"
#include "stream_k.cuh"
#include "xtc_internal.h"

namespace xtc {

// LEAN: the split-free variant (no split_k partials, no cluster split-K, no stream-K): those paths
// are compiled out, which shrinks the code the per-tile roles walk (ncu: 18 % of the L56 kernel's
// warp samples were stalled on instruction fetch, 'no_instructions', in the full variant)
template <bool TF32, int MSUB, int CL, bool PAIR = false, bool LEAN = false>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_conv_halo_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmY, const TcParams p) {
    constexpr int ATOM = TF32 ? 32 : 64;     // channels per 128-byte row
    constexpr int UMMA_K = TF32 ? 8 : 16;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t pad = (1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    const bool b_res = p.b_resident != 0;
    const int S = p.stages;
    // [B: all k-blocks (b_resident) or an S-stage ring][patch buffers][epilogue staging][barriers]
    uint8_t* sB = smem;
    uint8_t* sP = sB + (size_t)(b_res ? p.kb_total : S) * p.b_stage_bytes;
    uint8_t* sC = sP + (size_t)p.nbuf * p.patch_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sC + (p.buffer_c ? kTcEpiSmem : 0));
    uint64_t* empty = full + 8;
    uint64_t* pfull = empty + 8;
    uint64_t* pempty = pfull + kHaloMaxPatchBufs;
    uint64_t* tfull = pempty + kHaloMaxPatchBufs;
    uint64_t* tempty = tfull + 2;
    uint64_t* bfull = tempty + 2;                // resident filter: one barrier per k-block
    uint64_t* ksig = bfull + kHaloMaxResidentKb; // cluster split-K: partials-written signals (2, by tile parity)
    uint64_t* tready = ksig + 2;                 // TMEM allocated (its address is in tmem_slot)
    uint64_t* tlast = tready + 1;                // the CTA's last tile accumulated (one phase: warps 0..3 drain
                                                 // half of it; tfull's parity would alias earlier tiles)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tlast + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // CL = 2: a cluster of two CTAs on M tiles 2j, 2j+1 (same N tile) shares the filter ring:
    // each fetches half of every stage and TMA-multicasts it to both.
    // PAIR (CL = 2, inner_m 256): the same two CTAs form a cta_group::2 pair.  Each packs its
    // own patch and half of the filter columns, all completing on the leader's barriers; the
    // leader (rank 0) issues M = 256 UMMAs (A rows from both patches, B columns from both
    // filter halves, at identical SMEM offsets) whose commits are multicast to both CTAs, and
    // both epilogues drain their own TMEM, then arrive on the leader's tempty.
    static_assert(!PAIR || (CL == 2 && MSUB == 1), "the CTA pair is a 2-CTA cluster, one UMMA tile per CTA");
    constexpr int CG = PAIR ? 2 : 1;
    const uint32_t rank = (CL == 2) ? ptx::cluster_ctarank() : 0u;
    // cluster split-K (split_k_mode XTC_SPLITK_CLUSTER, CL = 1): the ksc CTAs of a cluster run
    // the ksc K segments (runs of filter taps / channel planes) of one output tile
    const int ksc = (!LEAN && CL == 1 && p.ksc > 1) ? p.ksc : 1;
    const bool kclu = ksc > 1;
    const uint32_t krank = kclu ? ptx::cluster_ctarank() : 0u;
    const int64_t cluster_id = blockIdx.x / (CL * ksc);
    const int64_t num_clusters = gridDim.x / (CL * ksc);
    // XTC_TRACE (diagnostics): slot 0 entry, 1 setup done, 2 exit; 8+j patch j issued,
    // 8+kTraceK+j patch j seen by the MMA warp, 8+2kTraceK+2j(+1) epilogue of tile j start/end
    uint64_t* const trace = (p.trace && blockIdx.x < kTraceCtas) ? p.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
    if (trace && threadIdx.x == 0) trace[0] = ptx::globaltimer();
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmX);
        ptx::prefetch_tmap(&tmB);
        if (p.buffer_c) ptx::prefetch_tmap(&tmY);
    }
    // early start: after the barrier inits (made visible CTA-wide, or cluster-wide for a CTA pair /
    // multicast cluster / cluster split, whose TMAs and arrives target the peers' barriers) the two
    // producer warps (0: patches, 3: filter) start loading at once and walk their tiles without the
    // SMEM tile table; only the TMEM users (warps 1, 2, 4..7) build the table and meet at a named
    // barrier.  (Trace at L56 N=32 before: the setup barrier at 0.8 us, the first patch issued at
    // 1.18 us, its data at 2.46 us.)
    const bool early = !(p.debug_skip_mma & 8192);   // (8192: A/B diagnostics)
    if (warp == 1 && lane == 0) {
        // a multicast stage is free only when the MMAs of every CTA in the cluster have read it
        for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], PAIR ? 1 : CL); }
        for (int i = 0; i < kHaloMaxPatchBufs; ++i) {
            ptx::mbar_init(&pfull[i], 1);
            ptx::mbar_init(&pempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4 * CG);
        }
        for (int i = 0; i < kHaloMaxResidentKb; ++i) ptx::mbar_init(&bfull[i], 1);
        if (kclu) { ptx::mbar_init(&ksig[0], 4u * ksc); ptx::mbar_init(&ksig[1], 4u * ksc); }
        ptx::mbar_init(tready, 1);
        ptx::mbar_init(tlast, 1);
        ptx::fence_mbarrier_init();
    }
    // barriers first (peers' barriers exist before multicasts); the TMEM allocation is then
    // taken by warp 2 while warps 0 and 3 already issue the patch and filter loads, and only
    // the TMEM users (warps 1, 4..7) wait for it on the mbarrier tready
    if (warp == 2 && p.debug_late_alloc) {
        ptx::tmem_alloc<CG>(tmem_slot, p.tmem_cols);
        ptx::tmem_relinquish<CG>();
        ptx::tc_fence_before();
    }
    // tile id -> (image, first output row, first output channel)
    // (compact rows: tile j of an image = virtual rows v0 = j*128*MSUB ...; p0 = v0 / Wc is the output
    // row whose padded window starts the patch, off = v0 - p0*Wc the tile's first slot in it)
    auto decode = [&](int64_t t, int& nimg, int& p0, int& n0, int& ks, int& off) {
        int mb, nb;
        tile_coords(p.tm, t, mb, nb, ks);
        if (kclu) ks = (int)krank;
        if (PAIR && p.compact) {
            // compact rows + CTA pair: pair tile mb = (image pair i, tile j); rank r takes image 2i + r, tile j, so
            // both CTAs' A views start at the same slot offset (the leader's descriptors address both patches)
            const int ip = mb / p.tpi, j = mb - ip * p.tpi;
            nimg = 2 * ip + (int)rank;
            const int v0 = j * 128 * MSUB;
            p0 = v0 / p.wp;
            off = v0 - p0 * p.wp;
            n0 = nb * p.tile_n;
            return;
        }
        mb = mb * CL + (int)rank;                    // CL = 2: the loop runs over M-tile pairs
        nimg = mb / p.tpi;
        if (p.compact) {
            const int v0 = (mb - nimg * p.tpi) * 128 * MSUB;
            p0 = v0 / p.wp;
            off = v0 - p0 * p.wp;
        } else {
            p0 = (mb - nimg * p.tpi) * p.rt * MSUB;
            off = 0;
        }
        n0 = nb * p.tile_n;
    };
    // the tiles this CTA visits and the k-block range of each: data-parallel (strided over the tile
    // map; K segment from the split or the cluster rank), or stream-K (stream_k.cuh)
    const bool sk = !LEAN && p.sk != 0;
    int64_t sk_s = 0, sk_e = 0;
    if (sk) sk_range(p.sk_iters, num_clusters, cluster_id, sk_s, sk_e);
    const int64_t n_walk = sk ? (sk_e > sk_s ? (sk_e - 1) / p.kb_total - sk_s / p.kb_total + 1 : 0)
                              : (p.num_tiles > cluster_id ? (p.num_tiles - cluster_id + num_clusters - 1) / num_clusters
                                                          : 0);
    auto walk_at = [&](int64_t i, int& kb0, int& kb1) -> int64_t {
        int64_t t;
        if (sk) {
            t = sk_s / p.kb_total + i;
            const int64_t base = t * p.kb_total;
            kb0 = (int)(sk_s > base ? sk_s - base : 0);
            kb1 = (int)(sk_e - base < p.kb_total ? sk_e - base : p.kb_total);
        } else {
            t = cluster_id + i * num_clusters;
            int mb, nb, ks;
            tile_coords(p.tm, t, mb, nb, ks);
            if (kclu) ks = (int)krank;
            kb0 = ks * p.kb_per_split;
            kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        }
        return t;
    };
    auto load_b = [&](uint8_t* dst, uint64_t* bar, int kb, int n0) {
        if (p.b3d) {
            ptx::tma_load_3d(&tmB, dst, bar, 0, kb * p.tile_k, n0 / ATOM);
        } else {
            for (int b = 0; b < p.tile_n / ATOM; ++b)
                ptx::tma_load_2d(&tmB, dst + (size_t)b * p.tile_k * 128, bar, n0 + b * ATOM, kb * p.tile_k);
        }
    };
    // The CTA's tile walk decoded ONCE into an SMEM table (first kTileTable tiles) before the setup
    // barrier, every thread one entry: each role then reads a tile's (image, row, channel, K range)
    // with two LDS instead of re-running the divisions of tile_coords / decode / walk_at per tile
    // (measured ~1100 cycles per tile per role in XTC_TRACE phase totals).
    TileInfo* const tinfo = reinterpret_cast<TileInfo*>((reinterpret_cast<uintptr_t>(tmem_slot) + 4 + 15) & ~uintptr_t(15));
    const bool producer = warp == 0 || warp == 3;
    if (early) {                                 // the barrier inits are visible; producers go
        if (CL == 2 || kclu) ptx::cluster_sync();
        else __syncthreads();
    }
    if (!(early && producer)) {
        // early: the 192 threads of warps 1, 2, 4..7 fill the table; else all 256
        const int ti0 = early ? (warp < 3 ? (int)threadIdx.x - 32 : (int)threadIdx.x - 64) : (int)threadIdx.x;
        const int tstep = early ? (int)blockDim.x - 64 : (int)blockDim.x;
        for (int i = ti0; i < n_walk && i < kTileTable; i += tstep) {
            TileInfo ti;
            ti.t = (int32_t)walk_at(i, ti.kb0, ti.kb1);
            decode(ti.t, ti.nimg, ti.p0, ti.n0, ti.ks, ti.off);
            tinfo[i] = ti;
        }
    }
    if (early) {
        if (!producer) ptx::named_bar_sync(1, blockDim.x - 64);
    } else if (CL == 2 || kclu) {
        ptx::cluster_sync();
    } else {
        __syncthreads();
    }
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
    auto tmem_address = [&]() -> uint32_t {
        ptx::mbar_wait(tready, 0);
        ptx::tc_fence_after();
        return *reinterpret_cast<volatile uint32_t*>(tmem_slot);
    };
    const int sfold = p.sfold > 1 ? p.sfold : 1;  // s-fold: accumulator blocks s = 0..S-1 of tile_n columns
    const int acc_cols = MSUB * p.tile_n * sfold;  // TMEM columns of one accumulator buffer
    // the CTA's LAST tile is drained by all 8 warps: warps 4..7 take columns [0, tile_n/2), warps 0..3 --
    // idle by then -- the upper half of the same TMEM lane quarters (warp w reads lanes 32(w%4)..).  Direct
    // stores only (no staging SMEM for warps 0..3), one CTA per tile, no split / stream-K / s-fold.  The
    // one-tile-per-CTA shapes (L14, small batches) pay their whole epilogue after the last MMA.
    const bool split_last = !(p.debug_skip_mma & 0x20000) && CL == 1 && !kclu && !sk && sfold == 1 && p.buffer_c == 0 &&
                            !p.split_out && !p.atomic && p.tile_n >= 64 && (p.tile_n & 63) == 0 && n_walk > 0;
    if (trace && threadIdx.x == 0) trace[1] = ptx::globaltimer();
    int tj = 0;                                  // per-role tile counter for the trace

    // the producers of an early start walk their tiles directly (the table may not be filled yet)
    auto tile_at = [tinfo, &walk_at, &decode, early, producer](int64_t it, TileInfo& ti) {
        if (it < kTileTable && !(early && producer)) {
            ti = tinfo[it];
        } else {
            ti.t = (int32_t)walk_at(it, ti.kb0, ti.kb1);
            decode(ti.t, ti.nimg, ti.p0, ti.n0, ti.ks, ti.off);
        }
    };
    // PAIR: this CTA's half of the filter columns (128-byte blocks nblk0 ...), completing on the
    // leader's barrier bar_c
    auto load_b_pair = [&](uint8_t* dst, uint32_t bar_c, int kb, int nblk0) {
        if (p.b64) {                                 // tile_n = one atom: this CTA's 32-column, 64-byte half
            ptx::tma_load_2d_pair(&tmB, dst, bar_c, nblk0 * ATOM + (int)rank * (ATOM / 2), kb * p.tile_k);
        } else if (p.b3d) {
            ptx::tma_load_3d_pair(&tmB, dst, bar_c, 0, kb * p.tile_k, nblk0);
        } else {
            for (int b = 0; b < p.tile_n / ATOM / 2; ++b)
                ptx::tma_load_2d_pair(&tmB, dst + (size_t)b * p.tile_k * 128, bar_c, (nblk0 + b) * ATOM, kb * p.tile_k);
        }
    };

    if (warp == 0) {
        // ===================== patch producer (pack at the tile level) =====================
        int pb = 0;
        uint32_t use_par = 0;
        bool first_round = true;
        for (int64_t it = 0; it < ((p.debug_skip_mma & 1024) ? 0 : n_walk); ++it) {
            TileInfo ti;
            tile_at(it, ti);
            const int nimg = ti.nimg, p0 = ti.p0;
            const int cb = pb;
            const uint32_t cpar = use_par;
            const bool fresh = first_round;
            if (++pb == p.nbuf) { pb = 0; use_par ^= 1u; first_round = false; }
            if (!fresh) {
                if (p.debug_skip_mma & 128) ptx::mbar_wait_sleep(&pempty[cb], cpar ^ 1u);
                else ptx::mbar_wait(&pempty[cb], cpar ^ 1u);
            }
            if (trace && lane == 0 && tj < kTraceK) trace[8 + tj] = ptx::globaltimer();
            ++tj;
            if (p.debug_skip_mma & 2) {
                if (ptx::elect_one()) ptx::mbar_arrive(&pfull[cb]);
            } else if (ptx::elect_one()) {
                uint8_t* dst = sP + (size_t)cb * p.patch_bytes;
                // box {ATOM channels, Wp slots, rows, 1} at (plane, -pad_w, p0 - pad_h, n): the zero
                // padding and the slots beyond the image are TMA's out-of-bounds zero fill
                if constexpr (PAIR) {                 // both patches complete on the leader's barrier
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&pfull[cb], 2 * p.patch_tx);
                    const uint32_t bar_c = ptx::mapa_shared(ptx::smem_u32(&pfull[cb]), 0);
                    for (int pl = 0; pl < p.planes; ++pl)
                        ptx::tma_load_4d_pair(&tmX, dst + (size_t)pl * p.plane_bytes, bar_c, pl * ATOM, -p.cg.pw,
                                              p0 - p.cg.ph, nimg);
                } else {
                    ptx::mbar_arrive_expect_tx(&pfull[cb], p.patch_tx);
                    for (int pl = 0; pl < p.planes; ++pl)
                        ptx::tma_load_4d(&tmX, dst + (size_t)pl * p.plane_bytes, &pfull[cb], pl * ATOM, -p.cg.pw,
                                         p0 - p.cg.ph, nimg);
                }
            }
            __syncwarp();
        }
    } else if (warp == 3) {
        // ===================== filter (B) producer =====================
        if (b_res) {
            if (ptx::elect_one()) {
                // one barrier per k-block: the first tile's MMAs start when k-block 0 lands
                for (int kb = 0; kb < p.kb_total; ++kb) {
                    if constexpr (PAIR) {             // my half of the columns, on the leader's barrier
                        if (rank == 0) ptx::mbar_arrive_expect_tx(&bfull[kb], 2 * p.b_stage_bytes);
                        load_b_pair(sB + (size_t)kb * p.b_stage_bytes, ptx::mapa_shared(ptx::smem_u32(&bfull[kb]), 0),
                                    kb, (int)rank * (p.tile_n / ATOM / 2));
                    } else {
                        ptx::mbar_arrive_expect_tx(&bfull[kb], p.b_stage_bytes);
                        load_b(sB + (size_t)kb * p.b_stage_bytes, &bfull[kb], kb, 0);
                    }
                }
            }
            __syncwarp();
        } else {
            int s = 0;
            uint32_t use_par = 0;
            bool first_round = true;
            for (int64_t it = 0; it < n_walk; ++it) {
                TileInfo ti;
                tile_at(it, ti);
                const int kb0 = ti.kb0, kb1 = ti.kb1, n0 = ti.n0;
                for (int kb = kb0; kb < kb1; ++kb) {
                    const int cs = s;
                    const uint32_t cpar = use_par;
                    const bool fresh = first_round;
                    if (++s == S) { s = 0; use_par ^= 1u; first_round = false; }
                    if (!fresh) ptx::mbar_wait(&empty[cs], cpar ^ 1u);
                    if (PAIR && ptx::elect_one()) {
                        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[cs], 2 * p.b_stage_bytes);
                        load_b_pair(sB + (size_t)cs * p.b_stage_bytes, ptx::mapa_shared(ptx::smem_u32(&full[cs]), 0),
                                    kb, n0 / ATOM + (int)rank * (p.tile_n / ATOM / 2));
                    } else if (!PAIR && ptx::elect_one()) {
                        ptx::mbar_arrive_expect_tx(&full[cs], p.b_stage_bytes);   // both halves land here
                        if constexpr (CL == 2) {
                            // my half of the stage's 128-byte N blocks, written into both CTAs
                            const int half = p.tile_n / ATOM / 2;
                            ptx::tma_load_3d_multicast(&tmB, sB + (size_t)cs * p.b_stage_bytes +
                                                                 (size_t)rank * half * p.tile_k * 128,
                                                       &full[cs], 0, kb * p.tile_k, n0 / ATOM + (int)rank * half, 0x3);
                        } else {
                            load_b(sB + (size_t)cs * p.b_stage_bytes, &full[cs], kb, n0);
                        }
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (contraction over r, s, c) =====================
        // ONE elected lane runs the whole tile walk -- ring / patch / accumulator waits, UMMAs and
        // commits.  Between two tiles it touches nothing but the two hand-off barriers: no tile-table
        // reads (unless the tile has a K segment: split / stream-K / cluster split), no divisions, no
        // warp reconvergence.  The UMMA queue holds only a few N = 64 UMMAs (~50 cycles each), so
        // bookkeeping on this thread at a tile boundary idles the tensor pipe (measured at L56 N=32:
        // ~860 cycles per tile when the warp reconverged and re-read the tile table per tile).
        const uint32_t tmem_base = tmem_address();
        const uint32_t b_lbo = (uint32_t)p.tile_k * 128u;
        const uint64_t adesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sP), 16, 1024);
        // B (MN-major): 128-byte swizzle rows of one 64-column atom (8-row groups 1024 bytes apart), or
        // for the pair's 64-byte halves the SW64 layout (layout type 4, 8-row groups 512 bytes apart)
        const uint64_t bdesc0 = TF32 ? ptx::smem_desc_sw128(ptx::smem_u32(sB), b_lbo, 512, 1)
                              : p.b64 ? ptx::smem_desc_sw128(ptx::smem_u32(sB), b_lbo / 2, 512, 4)
                                      : ptx::smem_desc_sw128(ptx::smem_u32(sB), b_lbo, 1024, 2);
        const uint32_t brow16 = ptx::pin(p.b64 ? 4u : 8u);   // 16-byte units per filter k-row in SMEM
        // every loop bound and stride pinned in a register; an atom's MSUB x (ATOM/UMMA_K) UMMAs
        // are straight-line code
        const uint32_t b_stage16 = ptx::pin(p.b_stage_bytes >> 4);
        const uint32_t plane16 = ptx::pin(p.plane_bytes >> 4);
        const uint32_t patch16 = ptx::pin(p.patch_bytes >> 4);
        const int n_atoms = ptx::pin(p.tile_k / ATOM);
        const int R_S = ptx::pin(p.cg.S), planes = ptx::pin(p.planes);
        const uint32_t tile_n = ptx::pin((uint32_t)p.tile_n);
        // A offset change (16-byte units) when the atom index wraps the channel planes, and
        // when it also wraps the filter columns (next filter row: + Wp rows)
        const uint32_t d_plane = plane16;
        const uint32_t d_col = ptx::pin(8u - (uint32_t)(p.planes - 1) * plane16);
        const uint32_t d_row = ptx::pin((uint32_t)p.wp * 8u - (uint32_t)(p.planes - 1) * plane16 -
                                        (uint32_t)(p.cg.S - 1) * 8u);
        const int kb_total = ptx::pin((p.debug_skip_mma & 33) ? 0 : p.kb_total);
        const int Sring = ptx::pin(S);
        const uint32_t idesc = ptx::pin(p.idesc);
        const bool plain_arrive = (p.debug_skip_mma & 16) != 0;
        const bool wait_tempty = !(p.debug_skip_mma & 64);
        // diagnostics (1024, with 64): free run -- no per-tile waits or commits, one commit at the end
        const bool free_run = (p.debug_skip_mma & 1024) != 0;
        // every tile spans all k-blocks unless a split / stream-K / cluster split gives it a K segment
        const bool fullk = !sk && !kclu && p.kb_per_split >= p.kb_total;
        const int64_t n_mma = (PAIR && rank != 0) ? 0 : n_walk;
        if (ptx::elect_one()) {
            if (b_res && !(PAIR && rank != 0))        // the resident filter (per-k-block barriers)
                for (int kb = 0; kb < p.kb_total; ++kb) ptx::mbar_wait(&bfull[kb], 0);
            const bool mphs = trace != nullptr;        // XTC_TRACE: MMA-warp wait / issue cycle totals
            uint64_t m_wait = 0, m_issue = 0, mck = mphs ? clock64() : 0;
            int s = 0, acc = 0, pb = 0;
            uint32_t ph = 0, aph = 0, pph = 0;
            for (int64_t it = 0; it < n_mma; ++it) {
                if (wait_tempty && !free_run) ptx::mbar_wait(&tempty[acc], aph ^ 1u);
                if (!free_run) ptx::mbar_wait(&pfull[pb], pph);
                if (mphs) { const uint64_t c2 = clock64(); m_wait += c2 - mck; mck = c2; }
                if (trace && tj < kTraceK) trace[8 + kTraceK + tj] = ptx::globaltimer();
                ++tj;
                if (!(p.debug_skip_mma & 4096)) ptx::tc_fence_after();
                int kb0 = 0, kb1 = kb_total, toff = 0;
                if (!fullk || p.compact) {             // this tile's k-block range (split_k / stream-K), row offset
                    TileInfo ti;
                    tile_at(it, ti);
                    kb0 = ti.kb0;
                    kb1 = min(ti.kb1, kb_total);       // (kb_total 0: diagnostics without MMAs)
                    toff = ti.off;
                }
                const uint32_t d0 = tmem_base + (uint32_t)(acc * acc_cols);
                // compact rows: virtual row 0 of the tile is patch row toff (8 x 16 bytes per 128-byte row)
                const uint64_t apatch = adesc0 + (uint64_t)((uint32_t)pb * patch16 + (uint32_t)toff * 8u);
                // the next 128-byte atom: channel plane pl, filter column sx, A offset aoff
                // (16-byte units) = pl*plane16 + (r*Wp + sx)*8, starting at the segment's first atom
                int pl = 0, sx = 0;
                uint32_t aoff = 0;
                if (kb0 > 0) {
                    const int j0 = kb0 * n_atoms, tap0 = j0 / planes;
                    pl = j0 - tap0 * planes;
                    sx = tap0 % R_S;
                    aoff = (uint32_t)pl * plane16 + (uint32_t)((tap0 / R_S) * p.wp + sx) * 8u;
                }
                uint32_t accf = 0;                    // 0 for the tile's first UMMA (overwrite)
                const uint32_t aoff_mask = (p.debug_skip_mma & 256) ? 0u : 0xffffffffu;   // diagnostics: no tap shifts
                auto atom = [&](uint64_t bd) {
                    const uint64_t ad = apatch + (uint64_t)(aoff & aoff_mask);
#pragma unroll
                    for (int ms = 0; ms < MSUB; ++ms)
#pragma unroll
                        for (int kk = 0; kk < ATOM / UMMA_K; ++kk)
                            ptx::umma<TF32, CG>(d0 + (uint32_t)ms * tile_n, ad + (uint64_t)(ms * 1024 + kk * 2),
                                               bd + (uint64_t)((uint32_t)(kk * UMMA_K) * brow16), idesc, kk ? 1u : accf);
                    accf = 1u;
                    const bool pw = ++pl == planes;             // plane wraps: next filter column
                    pl = pw ? 0 : pl;
                    sx += pw ? 1 : 0;
                    const bool sw = sx == R_S;                  // column wraps: next filter row
                    sx = sw ? 0 : sx;
                    aoff += pw ? (sw ? d_row : d_col) : d_plane;
                };
                if (sfold > 1 && kb1 > kb0) {
                    // s-fold: per filter row r, channel plane pl and 16-deep step kk ONE UMMA of N = S x
                    // tile_n on the patch view of row r (no s shift); its B operand is the row's S resident
                    // taps, N blocks C x 128 bytes apart (row (r*S + s)*C + c of the RSCF filter)
                    const uint64_t bfold = ptx::smem_desc_sw128(ptx::smem_u32(sB), (uint32_t)p.cg.C * 128u, 1024, 2);
                    const int R_R = ptx::pin(p.cg.R), C_ = ptx::pin(p.cg.C);
                    for (int r = 0; r < R_R; ++r) {
                        const uint64_t ar = apatch + (uint64_t)((uint32_t)r * (uint32_t)p.wp * 8u);
                        const uint64_t brow = bfold + (uint64_t)((uint32_t)(r * R_S * C_) * 8u);
                        for (int pl2 = 0; pl2 < planes; ++pl2) {
                            const uint64_t ad = ar + (uint64_t)((uint32_t)pl2 * plane16);
                            const uint64_t bd = brow + (uint64_t)((uint32_t)(pl2 * ATOM) * 8u);
#pragma unroll
                            for (int kk = 0; kk < ATOM / UMMA_K; ++kk)
                                ptx::umma<TF32, CG>(d0, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * UMMA_K * 8), idesc,
                                                   (r | pl2 | kk) ? 1u : 0u);
                        }
                    }
                } else if (b_res) {
                    // resident filter: k-block kb of B at kb * b_stage16, atom a at a*ATOM rows
                    const int reps = (p.debug_skip_mma & 512) ? 2 : 1;   // diagnostics: every UMMA twice
                    for (int rep = 0; rep < reps; ++rep)
                    for (int kb = kb0; kb < kb1; ++kb) {
                        const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)kb * b_stage16);
                        for (int a = 0; a < n_atoms; ++a) atom(bd + (uint64_t)((uint32_t)(a * ATOM) * brow16));
                    }
                } else {
                    for (int kb = kb0; kb < kb1; ++kb) {
                        ptx::mbar_wait(&full[s], ph);
                        ptx::tc_fence_after();
                        const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)s * b_stage16);
                        for (int a = 0; a < n_atoms; ++a) atom(bd + (uint64_t)((uint32_t)(a * ATOM) * brow16));
                        if constexpr (PAIR) ptx::umma_commit<2>(&empty[s]);
                        else if constexpr (CL == 2) ptx::umma_commit_multicast(&empty[s], 0x3);
                        else ptx::umma_commit<1>(&empty[s]);
                        if (++s == Sring) { s = 0; ph ^= 1u; }
                    }
                }
                if (free_run) {
                    if (p.debug_skip_mma & 2048) { ptx::umma_commit<CG>(&pempty[pb]); ptx::umma_commit<CG>(&tempty[acc]); }
                    if (it + 1 == n_mma) { ptx::umma_commit<CG>(&tfull[0]); ptx::mbar_wait(&tfull[0], 0); }
                } else if (plain_arrive) {            // diagnostics: plain arrives (valid only without MMAs)
                    ptx::mbar_arrive(&pempty[pb]);
                    ptx::mbar_arrive(&tfull[acc]);
                    if (split_last && it + 1 == n_mma) ptx::mbar_arrive(tlast);
                } else {
                    ptx::umma_commit<CG>(&pempty[pb]);    // patch buffer(s) free once these MMAs finish
                    ptx::umma_commit<CG>(&tfull[acc]);
                    if (split_last && it + 1 == n_mma) ptx::umma_commit<CG>(tlast);
                }
                if (mphs) {
                    const uint64_t c2 = clock64();
                    m_issue += c2 - mck; mck = c2;
                    trace[kTracePhase + 6] = m_wait; trace[kTracePhase + 7] = m_issue;
                }
                if (++pb == p.nbuf) { pb = 0; pph ^= 1u; }
                if (++acc == p.acc_buffers) { acc = 0; aph ^= 1u; }
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ===================== epilogue (bufferize) =====================
        const uint32_t tmem_base = tmem_address();
        const int q = warp & 3;
        int acc = 0, buf = 0;
        uint32_t aph = 0;
        ClusterSplitState kst;
        uint8_t* stage = sC + q * (kTcEpiStageBytes * kTcEpiBuffers);
        const bool bf16_out = p.out_bf16 != 0;
        const int P = p.cg.P, Q = p.cg.Q;
        // s-fold exchange: [round parity][warp][row s(s-1)/2 + i][32 fp32] after the SMEM tile table
        float* const xbuf = reinterpret_cast<float*>(tinfo + kTileTable);
        const int xrows = sfold * (sfold - 1) / 2;
        uint32_t xround = 0;
        // tile-invariant virtual-row -> (row, slot) splits of this warp / thread (Wp is a power of two)
        int e_row0[MSUB], e_q0[MSUB], e_row[MSUB], e_q[MSUB];
#pragma unroll
        for (int ms = 0; ms < MSUB; ++ms) {
            const int v0 = ms * 128 + 32 * q, v = v0 + lane;
            e_row0[ms] = v0 / p.wp; e_q0[ms] = v0 % p.wp;
            e_row[ms] = v / p.wp; e_q[ms] = v % p.wp;
        }
        const bool phs = trace && warp == 4 && lane == 0;      // XTC_TRACE epilogue phase totals
        uint64_t ph_t[6] = {0, 0, 0, 0, 0, 0};
        uint64_t ck = phs ? clock64() : 0;
        auto lap = [&](int k) { if (phs) { const uint64_t c2 = clock64(); ph_t[k] += c2 - ck; ck = c2; } };
        for (int64_t it = 0; it < ((p.debug_skip_mma & 64) ? 0 : n_walk); ++it) {
            TileInfo ti;
            tile_at(it, ti);
            const int kb0 = ti.kb0, kb1 = ti.kb1, nimg = ti.nimg, p0 = ti.p0, n0 = ti.n0, ks = ti.ks;
            const int64_t t = ti.t;
            lap(1);
            if (p.debug_skip_mma & 128) ptx::mbar_wait_sleep(&tfull[acc], aph);
            else ptx::mbar_wait(&tfull[acc], aph);
            lap(0);
            if (trace && warp == 4 && lane == 0 && tj < kTraceTiles) trace[8 + 2 * kTraceK + 2 * tj] = ptx::globaltimer();
            ptx::tc_fence_after();
            // stream-K (stream_k.cuh): contribution -> this CTA's slot [128*MSUB virtual rows][tile_n];
            // owned -> + the later k-ranges' partials (CTAs cluster_id+1 .. sk_last), ascending
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
            for (int ms = 0; ms < ((p.debug_skip_mma & 8) ? 0 : MSUB); ++ms) {
                const int v = ms * 128 + 32 * q + lane;        // this thread's virtual row
                int prow0 = p0 + e_row0[ms], q0 = e_q0[ms];
                int prow = p0 + e_row[ms], qcol = e_q[ms];
                if (p.compact) {                               // the tile starts at slot off of patch row 0
                    const int w0 = ti.off + ms * 128 + 32 * q, w = w0 + lane;
                    const int r0 = w0 / p.wp, r = w / p.wp;
                    prow0 = p0 + r0; q0 = w0 - r0 * p.wp;
                    prow = p0 + r; qcol = w - r * p.wp;
                }
                const bool valid = prow < P && qcol < Q;
                const bool any_valid = prow0 < P;              // rows grow with the lane index
                const uint32_t t_row = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * acc_cols + ms * p.tile_n);
                const int c_end = (split_last && it + 1 == n_walk) ? p.tile_n / 2 : p.tile_n;
                for (int c = 0; c < c_end; c += 32) {
                    uint32_t vals[32];
                    lap(4);
                    ptx::tmem_ld_32x32b_x32(t_row + c, vals);
                    ptx::tmem_ld_wait();
                    if (sfold > 1) {
                        // s-fold: + block sx of virtual row v + sx, sx = 1..S-1 (S <= 4) in ascending order.
                        // All blocks are loaded and the rows the warp below needs (its last lanes' v + sx =
                        // this warp's rows 0..sx-1) published before ONE named barrier per chunk; rows of
                        // this warp come by shuffle.  Only when an output row spans warps (Wp > 32); else
                        // those lanes' slots are >= Q and never stored.
                        const bool xchg = p.wp > 32;
                        float* xb = xbuf + (size_t)(((xround & 1) * 4) * xrows) * 32;
                        ++xround;
                        uint32_t wb[3][32];
#pragma unroll
                        for (int sx = 1; sx < 4; ++sx)
                            if (sx < sfold) ptx::tmem_ld_32x32b_x32(t_row + (uint32_t)(sx * p.tile_n) + c, wb[sx - 1]);
                        ptx::tmem_ld_wait();
                        if (xchg) {
#pragma unroll
                            for (int sx = 1; sx < 4; ++sx)
                                if (sx < sfold && q > 0 && lane < sx) {
                                    float4* dst = reinterpret_cast<float4*>(
                                        xb + (size_t)(((q - 1) * xrows) + sx * (sx - 1) / 2 + lane) * 32);
#pragma unroll
                                    for (int j = 0; j < 8; ++j)
                                        dst[j] = make_float4(__uint_as_float(wb[sx - 1][4 * j]), __uint_as_float(wb[sx - 1][4 * j + 1]),
                                                             __uint_as_float(wb[sx - 1][4 * j + 2]), __uint_as_float(wb[sx - 1][4 * j + 3]));
                                }
                            ptx::named_bar_sync(3, 128);
                        }
#pragma unroll
                        for (int sx = 1; sx < 4; ++sx) {
                            if (sx >= sfold) break;
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                wb[sx - 1][j] = __float_as_uint(__shfl_down_sync(0xffffffffu, __uint_as_float(wb[sx - 1][j]), sx));
                            if (xchg && q < 3 && lane >= 32 - sx) {          // divergent: the last sx lanes
                                const float4* src = reinterpret_cast<const float4*>(
                                    xb + (size_t)((q * xrows) + sx * (sx - 1) / 2 + (lane - (32 - sx))) * 32);
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    const float4 o = src[j];
                                    wb[sx - 1][4 * j] = __float_as_uint(o.x); wb[sx - 1][4 * j + 1] = __float_as_uint(o.y);
                                    wb[sx - 1][4 * j + 2] = __float_as_uint(o.z); wb[sx - 1][4 * j + 3] = __float_as_uint(o.w);
                                }
                            }
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                vals[j] = __float_as_uint(__uint_as_float(vals[j]) + __uint_as_float(wb[sx - 1][j]));
                        }
                    }
                    lap(2);
                    // stream-K partial slot, column-group major: float4 (col/4, virtual row v) at (col/4)*128*MSUB + v,
                    // so a warp's 32 rows of one 4-column group are 512 contiguous bytes (coalesced both ways; a
                    // row-major slot made every 16-byte access of a warp touch 32 lines)
                    if (sk_contrib) {
                        uint4* dst = reinterpret_cast<uint4*>(p.Wk + cluster_id * p.sk_slot) + (int64_t)(c / 4) * (128 * MSUB) + v;
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            dst[(int64_t)j * (128 * MSUB)] = make_uint4(vals[4 * j], vals[4 * j + 1], vals[4 * j + 2], vals[4 * j + 3]);
                        continue;
                    }
                    if (sk_own) {
                        for (int64_t g2 = cluster_id + 1; g2 <= sk_last; ++g2) {
                            const float4* src = reinterpret_cast<const float4*>(p.Wk + g2 * p.sk_slot) +
                                                (int64_t)(c / 4) * (128 * MSUB) + v;
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const float4 w = __ldcg(src + (int64_t)j * (128 * MSUB));
                                vals[4 * j] = __float_as_uint(__uint_as_float(vals[4 * j]) + w.x);
                                vals[4 * j + 1] = __float_as_uint(__uint_as_float(vals[4 * j + 1]) + w.y);
                                vals[4 * j + 2] = __float_as_uint(__uint_as_float(vals[4 * j + 2]) + w.z);
                                vals[4 * j + 3] = __float_as_uint(__uint_as_float(vals[4 * j + 3]) + w.w);
                            }
                        }
                    }
                    if (!any_valid || (p.debug_skip_mma & 4)) continue;   // warp-uniform
                    if (p.cons && valid) {            // fused consumer before the rounding
                        const int64_t m = ((int64_t)nimg * P + prow) * Q + qcol;
                        const int64_t cc = (int64_t)n0 + c;
                        const int nc = (int)((p.N - cc) < 32 ? (p.N - cc) : 32);
                        if (nc > 0) apply_consumer32(vals, p.cons, p.bias, p.C, bf16_out, m, p.ldc, cc, nc);
                    }
                    if (p.buffer_c) {
                        // one 128-byte staging row per thread (virtual row order = the TMA box's
                        // [p][q] order), then one clipped 4-D TMA store per warp
                        const bool first_half = !bf16_out || ((c & 63) == 0);
                        if (first_half) {
                            if (lane == 0) ptx::bulk_wait_read<1>();
                            __syncwarp();
                            lap(3);
                        }
                        uint8_t* rowp = stage + buf * kTcEpiStageBytes + lane * 128;
                        if (bf16_out) {
                            const int cbase = (c & 63) ? 4 : 0;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                uint4 w;
                                w.x = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 0]), __uint_as_float(vals[8 * j + 1]));
                                w.y = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 2]), __uint_as_float(vals[8 * j + 3]));
                                w.z = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 4]), __uint_as_float(vals[8 * j + 5]));
                                w.w = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 6]), __uint_as_float(vals[8 * j + 7]));
                                *reinterpret_cast<uint4*>(rowp + (((cbase + j) ^ (lane & 7)) * 16)) = w;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) * 16)) =
                                    make_uint4(vals[4 * j], vals[4 * j + 1], vals[4 * j + 2], vals[4 * j + 3]);
                        }
                        const bool last_half = !bf16_out || ((c & 63) == 32) || (c + 32 >= p.tile_n);
                        if (last_half) {
                            ptx::fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) {
                                const int col = bf16_out ? (n0 + (c & ~63)) : (n0 + c);
                                ptx::tma_store_4d(&tmY, stage + buf * kTcEpiStageBytes, col, q0, prow0, nimg);
                                ptx::bulk_commit();
                            }
                            buf ^= 1;
                        }
                    } else if (valid) {
                        const int64_t m = ((int64_t)nimg * P + prow) * Q + qcol;
                        const int64_t col0 = (int64_t)n0 + c;
                        const int ncols = (int)((p.N - col0) < 32 ? (p.N - col0) : 32);
                        if (!LEAN && p.split_out) {         // split_k: this segment's fp32 partial sums
                            float* dst = p.Wk + ((int64_t)ks * p.M + m) * p.ws_ld + col0;
                            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    reinterpret_cast<uint4*>(dst)[j] =
                                        make_uint4(vals[4 * j], vals[4 * j + 1], vals[4 * j + 2], vals[4 * j + 3]);
                            } else {
                                #pragma unroll
                                for (int j = 0; j < 32; ++j) if (j < ncols) dst[j] = __uint_as_float(vals[j]);
                            }
                        } else if (bf16_out) {
                            uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + m * p.ldc + col0;
                            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    uint4 w;
                                    w.x = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 0]), __uint_as_float(vals[8 * j + 1]));
                                    w.y = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 2]), __uint_as_float(vals[8 * j + 3]));
                                    w.z = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 4]), __uint_as_float(vals[8 * j + 5]));
                                    w.w = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 6]), __uint_as_float(vals[8 * j + 7]));
                                    reinterpret_cast<uint4*>(dst)[j] = w;
                                }
                            } else {
                                #pragma unroll
                                for (int j = 0; j < 32; ++j) if (j < ncols)
                                    dst[j] = (uint16_t)(ptx::pack_bf16x2(__uint_as_float(vals[j]), 0.f) & 0xFFFFu);
                            }
                        } else {
                            float* dst = reinterpret_cast<float*>(p.C) + m * p.ldc + col0;
                            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    reinterpret_cast<uint4*>(dst)[j] =
                                        make_uint4(vals[4 * j], vals[4 * j + 1], vals[4 * j + 2], vals[4 * j + 3]);
                            } else {
                                #pragma unroll
                                for (int j = 0; j < 32; ++j) if (j < ncols) dst[j] = __uint_as_float(vals[j]);
                            }
                        }
                    }
                }
            }
            if (sk_contrib) {                          // publish this warp's rows of the partial
                __syncwarp();
                if (lane == 0) sk_publish(p.sk_flags, cluster_id, q, p.sk_epoch);
                if (trace && warp == 4 && lane == 0) trace[5] = ptx::globaltimer();   // XTC_TRACE: published
            }
            ptx::tc_fence_before();
            __syncwarp();
            lap(4);
            if (trace && warp == 4 && lane == 0 && tj < kTraceTiles) trace[8 + 2 * kTraceK + 2 * tj + 1] = ptx::globaltimer();
            ++tj;
            if (lane == 0) {
                if constexpr (PAIR) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
                else ptx::mbar_arrive(&tempty[acc]);
            }
            if (++acc == p.acc_buffers) { acc = 0; aph ^= 1u; }
            if (kclu) {
                // the tile's valid output rows are contiguous in y: image nimg, rows p0 .. p0+rt*MSUB-1 (< P)
                const int p1 = min(P, p0 + p.rt * MSUB);
                cluster_split_reduce(ksig, kst, ksc, (int)krank, p.Wk, p.M, p.ws_ld, ((int64_t)nimg * P + p0) * Q,
                                     (p1 - p0) * Q, n0, (int)((p.N - n0) < p.tile_n ? (p.N - n0) : p.tile_n), p.C, p.ldc,
                                     bf16_out, p.cons_red, p.bias, (int)threadIdx.x - 128, false, trace);
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
        if (phs) {
            lap(4);
            for (int k = 0; k < 5; ++k) trace[kTracePhase + k] = ph_t[k];
            trace[kTracePhase + 5] = (uint64_t)tj;
        }
    }

    if (split_last && warp < 4 && !(p.debug_skip_mma & (64 | 8))) {
        const uint32_t tmem_base = tmem_address();
        const int64_t it = n_walk - 1;
        const int acc = (int)(it % p.acc_buffers);
        const uint32_t aph = (uint32_t)((it / p.acc_buffers) & 1);
        TileInfo ti;
        tile_at(it, ti);
        (void)aph;
        ptx::mbar_wait(tlast, 0);                  // the last tile's MMAs are complete
        ptx::tc_fence_after();
        const int q = warp, P = p.cg.P, Q = p.cg.Q;
        const bool bf16_out = p.out_bf16 != 0;
#pragma unroll 1
        for (int ms = 0; ms < MSUB; ++ms) {
            const int w = ti.off + ms * 128 + 32 * q + lane;   // this thread's row (pow2 rows: off = 0)
            const int r = w / p.wp;
            const int prow = ti.p0 + r, qcol = w - r * p.wp;
            const bool valid = prow < P && qcol < Q;
            const int64_t m = ((int64_t)ti.nimg * P + prow) * Q + qcol;
            const uint32_t t_row = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * acc_cols + ms * p.tile_n);
#pragma unroll 1
            for (int c = p.tile_n / 2; c < p.tile_n; c += 32) {
                uint32_t vals[32];
                ptx::tmem_ld_32x32b_x32(t_row + c, vals);
                ptx::tmem_ld_wait();
                if (!valid) continue;
                const int64_t col0 = (int64_t)ti.n0 + c;
                const int ncols = (int)((p.N - col0) < 32 ? (p.N - col0) : 32);
                if (ncols <= 0) continue;
                if (p.cons) apply_consumer32(vals, p.cons, p.bias, p.C, bf16_out, m, p.ldc, col0, ncols);
                if (bf16_out) {
                    uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + m * p.ldc + col0;
                    if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint4 o;
                            o.x = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 0]), __uint_as_float(vals[8 * j + 1]));
                            o.y = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 2]), __uint_as_float(vals[8 * j + 3]));
                            o.z = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 4]), __uint_as_float(vals[8 * j + 5]));
                            o.w = ptx::pack_bf16x2(__uint_as_float(vals[8 * j + 6]), __uint_as_float(vals[8 * j + 7]));
                            reinterpret_cast<uint4*>(dst)[j] = o;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) if (j < ncols)
                            dst[j] = (uint16_t)(ptx::pack_bf16x2(__uint_as_float(vals[j]), 0.f) & 0xFFFFu);
                    }
                } else {
                    float* dst = reinterpret_cast<float*>(p.C) + m * p.ldc + col0;
                    if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            reinterpret_cast<uint4*>(dst)[j] = make_uint4(vals[4 * j], vals[4 * j + 1], vals[4 * j + 2], vals[4 * j + 3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) if (j < ncols) dst[j] = __uint_as_float(vals[j]);
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    if (CL == 2 || kclu) ptx::cluster_sync(); else __syncthreads();   // no CTA exits while a peer may still signal it
    if (trace && threadIdx.x == 0) trace[2] = ptx::globaltimer();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<CG>(*reinterpret_cast<volatile uint32_t*>(tmem_slot), p.tmem_cols);
        if (trace && lane == 0) trace[7] = ptx::globaltimer();                // XTC_TRACE: TMEM released
    }
}

template <bool TF32, int MSUB, int CL, bool PAIR = false>
static cudaError_t launch_halo_t(const CUtensorMap& x, const CUtensorMap& b, const CUtensorMap& y, const TcParams& p,
                                 int grid, int smem, cudaStream_t st) {
    // the lean variant for split-free bf16 plans (the BASELINE layers' schedules)
    const bool lean = !TF32 && !p.sk && p.ksc <= 1 && !p.split_out && !p.atomic;
    auto k = lean ? tc_conv_halo_kernel<TF32, MSUB, CL, PAIR, !TF32> : tc_conv_halo_kernel<TF32, MSUB, CL, PAIR, false>;
    cudaError_t e = ensure_smem_attr(k, smem);
    if (e != cudaSuccess) return e;
    const int ksc = (CL == 1 && p.ksc > 1) ? p.ksc : 1;
    if (CL == 1 && ksc == 1 && !p.sk) {
        k<<<grid, kTcThreads, smem, st>>>(x, b, y, p);
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
            attr[0].val.clusterDim.x = CL * ksc;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
        }
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, k, x, b, y, p);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

template <bool TF32, int MSUB>
static cudaError_t launch_halo_cl(const CUtensorMap& x, const CUtensorMap& b, const CUtensorMap& y, const TcParams& p,
                                  int grid, int smem, cudaStream_t st) {
    return p.cl == 2 ? launch_halo_t<TF32, MSUB, 2>(x, b, y, p, grid, smem, st)
                     : launch_halo_t<TF32, MSUB, 1>(x, b, y, p, grid, smem, st);
}

cudaError_t launch_tc_conv_halo(bool tf32, const CUtensorMap& x, const CUtensorMap& b, const CUtensorMap& y,
                                const TcParams& p, int grid, int smem, cudaStream_t st) {
    // MSUB (128-row UMMA tiles per patch) is a template parameter: the per-atom UMMA
    // sequence is straight-line code
    if (p.pair)
        return tf32 ? launch_halo_t<true, 1, 2, true>(x, b, y, p, grid, smem, st)
                    : launch_halo_t<false, 1, 2, true>(x, b, y, p, grid, smem, st);
    if (p.msub == 2)
        return tf32 ? launch_halo_cl<true, 2>(x, b, y, p, grid, smem, st) : launch_halo_cl<false, 2>(x, b, y, p, grid, smem, st);
    return tf32 ? launch_halo_cl<true, 1>(x, b, y, p, grid, smem, st) : launch_halo_cl<false, 1>(x, b, y, p, grid, smem, st);
}

}  // namespace xtc
