// planner.cpp -- a2: schedule application = legality + launch-plan derivation.
//
// The paper's Scheduler "records the scheduling API calls and builds an
// internal representation of the schedule", which the Compiler then applies
// (P:751-755).  On B200 the "compiled" artefact is a launch plan
// for one of the pre-built sm_100a kernel variants: grid / cluster, SMEM
// bytes, TMEM columns, split-K workspace.  Everything here is host integer
// work (no CUDA calls), so it is testable without a GPU.
//
// Legality rules:
//   tcgen05 : UMMA M in {128 (cta_group::1), 256 (cta_group::2)}; N multiple of
//             the 128-byte swizzle atom of B (64 bf16 / 32 tf32 columns) and <= 256;
//             tile_k multiple of the A swizzle atom (64 bf16 / 32 tf32), <= 256;
//             stages 2..8; SMEM <= 232448 B (sm_100 opt-in limit); TMEM columns
//             (pow2 >= 32 of acc_buffers * tile_n) <= 512; TMA row pitches % 16 B.
//   SIMT    : fp32 inputs; inner tile TM,TN in {1,2,4,8}; (tile/inner) threads
//             in [1,1024]; unroll divides tile_k; vector_n 4 needs TN%4.
//   split   : every K segment holds >= 1 k-block; atomic split-K needs fp32 out.
#include <algorithm>
#include <cstdio>
#include <string>
#include "xtc_internal.h"

namespace xtc {

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static bool pow2_in(int v, int lo, int hi) { return v >= lo && v <= hi && (v & (v - 1)) == 0; }

#define ILLEGAL(...) do { char _b[320]; snprintf(_b, sizeof _b, __VA_ARGS__); why = _b; return XTC_E_ILLEGAL_SCHEDULE; } while (0)
#define INVALID(...) do { char _b[320]; snprintf(_b, sizeof _b, __VA_ARGS__); why = _b; return XTC_E_INVALID_ARG; } while (0)

void gemm_view(const xtc_op_desc& d, int64_t& M, int64_t& N, int64_t& K, int64_t& P, int64_t& Q) {
    if (d.kind == XTC_OP_CONV2D) {
        P = (d.h + 2 * d.pad_h - d.r) / d.stride_h + 1;
        Q = (d.w + 2 * d.pad_w - d.s) / d.stride_w + 1;
        M = d.batch * P * Q;
        N = d.f;
        K = d.r * d.s * d.c;
    } else {
        P = Q = 0;
        M = d.m; N = d.n; K = d.k;
    }
}

static int dtype_size(int dt) { return dt == XTC_BF16 ? 2 : 4; }

xtc_status check_desc(const xtc_op_desc& d, std::string& why) {
    if (d.kind != XTC_OP_MATMUL && d.kind != XTC_OP_CONV2D) INVALID("unknown op kind %d", d.kind);
    if (d.in_dtype < XTC_F32 || d.in_dtype > XTC_TF32) INVALID("unknown in_dtype %d", d.in_dtype);
    if (d.out_dtype != XTC_F32 && d.out_dtype != XTC_BF16) INVALID("out_dtype must be F32 or BF16");
    if (d.consumer & ~(XTC_CONSUMER_RELU | XTC_CONSUMER_BIAS | XTC_CONSUMER_ACCUMULATE))
        INVALID("unknown consumer bits 0x%x", d.consumer);
    if (d.kind == XTC_OP_MATMUL) {
        if (d.m <= 0 || d.n <= 0 || d.k <= 0) INVALID("matmul extents must be > 0 (m=%lld n=%lld k=%lld)",
                                                      (long long)d.m, (long long)d.n, (long long)d.k);
        if ((d.lda && d.lda < d.k) || (d.ldb && d.ldb < d.n) || (d.ldc && d.ldc < d.n))
            INVALID("leading dimension smaller than the row extent");
    } else {
        if (d.batch <= 0 || d.h <= 0 || d.w <= 0 || d.c <= 0 || d.f <= 0 || d.r <= 0 || d.s <= 0)
            INVALID("conv2d extents must be > 0");
        if (d.stride_h <= 0 || d.stride_w <= 0 || d.pad_h < 0 || d.pad_w < 0) INVALID("bad stride/pad");
        if (d.h + 2 * d.pad_h < d.r || d.w + 2 * d.pad_w < d.s) INVALID("filter larger than padded input");
    }
    int64_t M, N, K, P, Q;
    gemm_view(d, M, N, K, P, Q);
    if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31)) INVALID("extent >= 2^31");
    return XTC_OK;
}

static xtc_status plan_simt(const xtc_op_desc& d, const xtc_schedule& s, int num_sms, Plan& p, std::string& why) {
    if (d.in_dtype != XTC_F32) ILLEGAL("SIMT engine computes fp32 inputs only (in_dtype must be F32)");
    int TM = s.inner_m, TN = s.inner_n;
    if (!pow2_in(TM, 1, 8) || !pow2_in(TN, 1, 16)) ILLEGAL("SIMT inner_m/inner_n (thread tile) must be 1,2,4 or 8 (inner_n 16 with inner_m <= 2)");
    if (TN == 16 && TM > 2) ILLEGAL("SIMT inner_n 16 (a 16-wide register row) needs inner_m <= 2");
    if (s.tile_m < 1 || s.tile_n < 1 || s.tile_m > 256 || s.tile_n > 256) ILLEGAL("SIMT tile_m/tile_n must be in [1,256]");
    if (s.tile_m % TM || s.tile_n % TN) ILLEGAL("strip-mine: tile_m %% inner_m and tile_n %% inner_n must be 0");
    int threads = (s.tile_m / TM) * (s.tile_n / TN);
    if (threads < 1 || threads > simt_max_threads(TM, TN))
        ILLEGAL("SIMT tile/inner gives %d threads (must be 1..%d for a %dx%d thread tile)", threads,
                simt_max_threads(TM, TN), TM, TN);
    if (s.tile_k < 1 || s.tile_k > 64) ILLEGAL("SIMT tile_k must be in [1,64]");
    int U = s.unroll_k == 0 ? 1 : s.unroll_k;
    if (!pow2_in(U, 1, 8)) ILLEGAL("SIMT unroll_k must be 1,2,4 or 8");
    if (s.tile_k % U) ILLEGAL("unroll: unroll_k (%d) must divide the k-tile trip count %d (S:271)", U, s.tile_k);
    int V = s.vector_n == 0 ? 1 : s.vector_n;
    if (V != 1 && V != 4) ILLEGAL("SIMT vector_n must be 1 or 4");
    if (V == 4 && TN % 4) ILLEGAL("vectorize: vector_n 4 needs inner_n %% 4 == 0");
    int st = s.stages == 0 ? 1 : s.stages;
    if (st != 1 && st != 2) ILLEGAL("SIMT stages must be 1 or 2");
    if (s.swizzle < 0 || s.swizzle > 8) ILLEGAL("SIMT swizzle (SMEM pad) must be in [0,8] floats");
    if (s.buffer_c != 0) ILLEGAL("SIMT engine: buffer_c must be 0 (the register tile is the write buffer)");
    if (s.acc_buffers > 1) ILLEGAL("SIMT engine: acc_buffers must be 0 or 1");
    if (s.cluster_m > 1) ILLEGAL("SIMT engine: cluster_m must be 1");
    if (s.pack_warps > 1) ILLEGAL("SIMT engine: pack_warps must be 0 or 1 (all threads pack)");
    if (s.b_resident) ILLEGAL("SIMT engine: b_resident must be 0");
    if (s.pack_halo) ILLEGAL("SIMT engine: pack_halo must be 0");
    if (s.cluster_n > 1) ILLEGAL("SIMT engine: cluster_n must be 0 or 1");
    if (V == 4 && (s.tile_n + s.swizzle) % 4) ILLEGAL("vectorize: vector_n 4 needs (tile_n + pad) %% 4 == 0 for aligned float4");
    auto r4 = [](int x) { return (x + 3) / 4 * 4; };
    int smem = st * (r4(s.tile_k * (s.tile_m + s.swizzle)) + r4(s.tile_k * (s.tile_n + s.swizzle))) * 4;
    if (smem > kSmemMaxOptin) ILLEGAL("SMEM %d B exceeds the %d B per-CTA limit", smem, kSmemMaxOptin);
    p.block = threads;
    p.smem = smem;
    p.tiles_m = (int)cdiv(p.M, s.tile_m);
    p.tiles_n = (int)cdiv(p.N, s.tile_n);
    int64_t ksplit = cdiv(p.K, p.split_k);
    p.k_per_split = cdiv(ksplit, s.tile_k) * s.tile_k;
    if ((p.split_k - 1) * p.k_per_split >= p.K) ILLEGAL("split: split_k %d leaves an empty K segment (K=%lld, tile_k=%d)",
                                                      p.split_k, (long long)p.K, s.tile_k);
    p.num_tiles = (int64_t)p.tiles_m * p.tiles_n * p.split_k;
    if (p.num_tiles >= (1ll << 31)) ILLEGAL("too many tiles");
    p.grid_x = s.persistent ? (int)std::min<int64_t>(p.num_tiles, (int64_t)num_sms * std::max(1, 2048 / threads))
                            : (int)p.num_tiles;
    return XTC_OK;
}

// pack at the output-tile level for stride-1 conv2d (pack_halo = 1).  A tile is tile_m
// "virtual rows" = (tile_m / Wp) output rows x Wp pixel slots, Wp = the power of two
// >= max(8, Q + S - 1) dividing 128; slots q >= Q and rows p >= P are computed on
// don't-care data and never stored.  The patch holds tile rows + R - 1 input rows of Wp
// pixels starting at (p0 - pad_h, -pad_w) for every 128-byte channel plane; TMA
// zero-fills everything outside the image (the zero padding).  Tap (r, s) of virtual row
// v reads patch row v + r*Wp + s, so each UMMA's A operand is the patch advanced by
// (r*Wp + s) 128-byte rows (profiles/r01_umma_row_shift_microtest.txt).
static xtc_status plan_tc_halo(const xtc_op_desc& d, const xtc_schedule& s, int num_sms, Plan& p, std::string& why) {
    const int es = dtype_size(d.in_dtype), os = dtype_size(d.out_dtype);
    if (d.kind != XTC_OP_CONV2D) ILLEGAL("pack_halo applies to conv2d only");
    if (s.pack_halo != 1 && s.pack_halo != 2) ILLEGAL("pack_halo must be 0, 1 or 2");
    // pack_halo = 2 (compact rows): output row p's slots sit at the padded row width Wc = Q + S - 1
    // (not the power of two above it) and a tile is 128 x tile_m/128 CONSECUTIVE virtual rows of one
    // image's P x Wc grid, so a tile starts mid-row: its patch starts at the padded input row of its
    // first virtual row and every UMMA A view is advanced by the tile's offset into that row.  Fewer
    // don't-care slots (L56: 58 of 64) and fewer tiles (L56 N=32: 832 instead of 896, 6 per SM
    // instead of 7).  One CTA per tile (cluster_m 1), no s-fold, no split, direct stores.
    const bool compact = s.pack_halo == 2;
    if (d.stride_h != 1 || d.stride_w != 1) ILLEGAL("pack_halo needs stride 1 (taps must be row shifts of one patch)");
    // cluster_m = 2: two CTAs on adjacent M tiles (same N tile) each fetch half of every filter
    // stage and TMA-multicast it to both (the filter stream per SM is halved)
    const int hcl = s.cluster_m == 0 ? 1 : s.cluster_m;
    if (hcl != 1 && hcl != 2) ILLEGAL("pack_halo: cluster_m must be 1 or 2 (filter multicast pair)");
    // split: K segments (runs of filter taps / channel planes) as their own CTAs; fp32 partials
    // written by direct stores, summed in ascending segment order by the reduction kernel
    if (p.split_k > 1 && p.atomic) ILLEGAL("pack_halo: split_k needs an ordered reduction (split_k_mode 0 or 2)");
    if (p.split_k > 1 && s.buffer_c) ILLEGAL("pack_halo: split_k writes fp32 partials with direct stores (buffer_c 0)");
    if (s.pack_warps > 1) ILLEGAL("pack_halo: pack_warps must be 0 or 1 (warp 0 packs patches, warp 3 the B ring)");
    if (s.tile_m != 128 && s.tile_m != 256) ILLEGAL("pack_halo: tile_m must be 128 or 256 (1 or 2 UMMA M-tiles per patch)");
    if (s.inner_m != 0 && s.inner_m != 128 && s.inner_m != 256) ILLEGAL("pack_halo: inner_m (UMMA M) must be 128 or 256");
    // inner_m = 256: the UMMA atom spans a CTA pair (cta_group::2).  Each CTA packs the patch of
    // its own 128-row M tile and half of the filter's N columns; the leader issues M = 256
    // UMMAs whose A rows come from both patches and B columns from both filter halves (per
    // SM: the operand reads of the B half and the filter TMA writes are halved)
    const bool pair = s.inner_m == 256;
    if (pair) {
        if (hcl != 2 || s.tile_m != 256) ILLEGAL("pack_halo: inner_m 256 (CTA pair) needs cluster_m 2 and tile_m 256");
        if (p.split_k > 1) ILLEGAL("pack_halo: the CTA pair (inner_m 256) needs split_k 1");
        // tile_n = one 128-byte atom (bf16: 64 filter columns): each CTA holds a 32-column, 64-byte half of
        // every filter k-block in the UMMA's 64-byte-swizzle MN-major layout (TMA SWIZZLE_64B), so the pair
        // halves the filter operand reads per SM at F = 64 too (L56)
        const bool half64 = s.tile_n == p.atom_n && d.in_dtype == XTC_BF16;
        if (s.tile_n % (2 * p.atom_n) && !half64)
            ILLEGAL("pack_halo: the CTA pair needs tile_n %% %d == 0 (a 128-byte filter block per CTA), or tile_n %d "
                    "with bf16 (64-byte filter halves)", 2 * p.atom_n, p.atom_n);
        if (!half64 && d.f % p.atom_n) ILLEGAL("pack_halo: the CTA pair needs F %% %d == 0 (3-D filter TMA)", p.atom_n);
        p.halo_b64 = half64;
    }
    // inner_n = S * tile_n: the s-fold.  The S taps (r, 0..S-1) of a filter row are the N blocks of
    // ONE UMMA on the patch view of row r (N = S * tile_n): accumulator block s of virtual row v
    // holds sum_c x[v + r*Wp + s][c] w[r][s][c][:] minus the s shift, which the epilogue applies by
    // adding block s of row v + s.  A is read once per filter row instead of once per tap.
    int sfold = 1;
    if (s.inner_n != 0 && s.inner_n != s.tile_n) {
        if (s.inner_n != d.s * s.tile_n || d.s < 2)
            ILLEGAL("pack_halo: inner_n (UMMA N) must be tile_n, or S x tile_n (s-fold, S >= 2)");
        if (s.inner_n > 256) ILLEGAL("pack_halo s-fold: UMMA N = S x tile_n = %d exceeds 256", s.inner_n);
        if (pair || hcl != 1 || s.tile_m != 128)
            ILLEGAL("pack_halo s-fold: one CTA per 128-row tile (cluster_m 1, tile_m 128, inner_m 128)");
        if (p.split_k > 1 || p.stream_k) ILLEGAL("pack_halo s-fold: split_k must be 1 (the fold sums whole filter rows)");
        if (s.b_resident != 1) ILLEGAL("pack_halo s-fold: b_resident must be 1 (taps of a row are one strided B operand)");
        if (s.tile_n != p.atom_n) ILLEGAL("pack_halo s-fold: tile_n must be %d (one 128-byte filter block per tap)", p.atom_n);
        if (d.in_dtype != XTC_BF16) ILLEGAL("pack_halo s-fold: bf16 inputs (kind::f16)");
        if (d.c % s.tile_k) ILLEGAL("pack_halo s-fold: tile_k must divide C (whole k-blocks per tap)");
        sfold = (int)d.s;
    }
    if (s.tile_n < p.atom_n || s.tile_n > 256 || s.tile_n % p.atom_n)
        ILLEGAL("tcgen05 tile_n must be a multiple of %d in [%d,256]", p.atom_n, p.atom_n);
    if (s.tile_k < p.atom_k || s.tile_k > 256 || s.tile_k % p.atom_k)
        ILLEGAL("tcgen05 tile_k must be a multiple of %d in [%d,256] (128-byte swizzle atom)", p.atom_k, p.atom_k);
    if (s.unroll_k > 1) ILLEGAL("tcgen05 unroll_k must be 0 or 1");
    if (s.vector_n > 1) ILLEGAL("tcgen05 vector_n must be 0");
    if (s.stages < 2 || s.stages > 8) ILLEGAL("tcgen05 stages must be in [2,8]");
    // producer g % pack_warps fills slot g % stages after waiting for the slot's previous round
    // (k-block g - stages) to be consumed; its own previous wait only guarantees k-block
    // g - pack_warps - stages, so with pack_warps > stages the slot may still be two rounds behind
    // and the mbarrier parity wait aliases (race found by the schedule-invariance sweep)
    if (s.pack_warps > s.stages) ILLEGAL("pack: pack_warps %d > stages %d (ring slot parity would alias)", s.pack_warps, s.stages);
    if (s.swizzle != 0 && s.swizzle != 128) ILLEGAL("tcgen05 swizzle must be 128 (0 = default 128)");
    if (d.c % p.atom_k) ILLEGAL("tcgen05 conv2d needs C %% %d == 0", p.atom_k);
    if ((d.f * es) % 16 || (d.f * os) % 16) ILLEGAL("TMA needs 16-byte row pitch for the filter and the output");
    if (p.K % s.tile_k) ILLEGAL("tcgen05 conv2d needs R*S*C %% tile_k == 0");
    int64_t P, Q, M_, N_, K_;
    gemm_view(d, M_, N_, K_, P, Q);
    int wp = 8;
    while (wp < Q + d.s - 1) wp *= 2;
    if (compact) {
        wp = (int)(Q + d.s - 1);
        // the CTA pair reads both CTAs' A views through the leader's descriptor, so both tiles must start at the
        // same slot offset: the pair takes tile j of images 2i and 2i + 1 (an even batch)
        if (hcl != 1 && !pair) ILLEGAL("pack_halo 2 (compact rows): cluster_m 2 only as the CTA pair (inner_m 256)");
        if (pair && d.batch % 2) ILLEGAL("pack_halo 2 (compact rows) with the CTA pair needs an even batch (images 2i, 2i+1)");
        if (sfold > 1) ILLEGAL("pack_halo 2 (compact rows): no s-fold (inner_n must be tile_n)");
        if (p.split_k > 1 || p.stream_k) ILLEGAL("pack_halo 2 (compact rows): split_k must be 1");
        // a warp's 32 rows start mid-row and wrap into the next output row; the TMA store box of
        // whole-row slots cannot express that (a negative start slot faults), so direct stores
        if (s.buffer_c) ILLEGAL("pack_halo 2 (compact rows): the epilogue stores directly (buffer_c 0)");
    }
    if (wp > 128) ILLEGAL("pack_halo: Q + S - 1 = %lld pixel slots exceed one 128-row UMMA tile", (long long)(Q + d.s - 1));
    const int msub = pair ? 1 : s.tile_m / 128;            // the pair: one 128-row UMMA tile per CTA
    const int rt = compact ? 0 : 128 / wp;                 // output rows per UMMA M-tile (pow2 rows)
    // patch rows: pow2 rows: the tile's rows + R - 1; compact: the rows spanned by the largest patch
    // index any virtual row of the tile reads, (Wc - 1) + 128*msub - 1 + (R-1)*Wc + S - 1, + 1
    const int64_t pr = compact ? ((int64_t)wp - 1 + 128 * msub - 1 + (d.r - 1) * wp + d.s - 1) / wp + 1
                               : (int64_t)msub * rt + d.r - 1;
    if (pr > 256) ILLEGAL("pack_halo: %lld patch rows exceed the 256-row TMA box", (long long)pr);
    const int accb = s.acc_buffers == 0 ? 1 : s.acc_buffers;
    if (accb < 1 || accb > 2) ILLEGAL("acc_buffers must be 1 or 2");
    int alloc = 32;
    while (alloc < accb * msub * s.tile_n * sfold) alloc *= 2;
    if (alloc > 512) ILLEGAL("bufferize: %d TMEM columns (acc_buffers x tile_m/128 x tile_n) exceed 512", alloc);
    p.tmem_cols = alloc;
    const int64_t planes = d.c / p.atom_k;
    // each channel plane starts 1024-byte aligned (the 128-byte swizzle atom; compact rows give
    // pr * Wc * 128 bytes that are not a multiple of 1024)
    const int64_t patch = planes * (((int64_t)pr * wp * 128 + 1023) / 1024 * 1024);
    const int64_t b_stage = (int64_t)s.tile_k * (pair ? s.tile_n / 2 : s.tile_n) * es;   // per CTA
    p.tiles_n = (int)cdiv(N_, s.tile_n);
    p.kb_total = (int)cdiv(K_, s.tile_k);
    int64_t b_bytes;
    if (s.b_resident) {
        if (s.b_resident != 1) ILLEGAL("b_resident must be 0 or 1");
        if (p.tiles_n != 1) ILLEGAL("pack: b_resident needs a single N tile (N <= tile_n)");
        if (p.kb_total > kHaloMaxResidentKb)
            ILLEGAL("pack_halo: b_resident supports at most %d k-blocks (one barrier each)", kHaloMaxResidentKb);
        b_bytes = p.kb_total * b_stage;
    } else {
        b_bytes = s.stages * b_stage;
    }
    // s-fold: per epilogue warp and chunk parity, rows 0..s-1 of accumulator blocks s = 1..S-1 for the
    // warp above (the rows v + s of its last lanes), 32 fp32 each
    const int64_t xbytes = sfold > 1 ? 4LL * 2 * (sfold * (sfold - 1) / 2) * 128 : 0;
    const int64_t fixed = b_bytes + (s.buffer_c ? kTcEpiSmem : 0) + kSmemReserve + kTileTableBytes + xbytes;
    // three patch buffers when they fit (A/B on B200 after the epilogue de-spill, tools/halo_nbuf_ab.py:
    // L56 N=32 22.06 -> 21.65 us, L14 N=32 19.44 -> 19.26 us), else two, else one
    int nbuf = 3;
    if (const char* e = getenv("XTC_HALO_NBUF")) nbuf = std::max(1, std::min(kHaloMaxPatchBufs, atoi(e)));   // diagnostics
    while (nbuf > 1 && fixed + nbuf * patch > kSmemMaxOptin) --nbuf;
    if (fixed + nbuf * patch > kSmemMaxOptin)
        ILLEGAL("pack_halo: patch %lld B + B operand %lld B + epilogue exceed %d B SMEM", (long long)patch,
                (long long)b_bytes, kSmemMaxOptin);
    if (s.buffer_c && d.out_dtype == XTC_BF16 && s.tile_n % 64) ILLEGAL("bufferize: bf16 TMA-store staging needs tile_n %% 64 == 0");
    p.smem = (int)(fixed + nbuf * patch);
    p.halo = true;
    p.halo_wp = wp;
    p.halo_rt = rt;
    p.halo_msub = msub;
    p.halo_pr = (int)pr;
    p.halo_planes = (int)planes;
    p.halo_nbuf = nbuf;
    p.halo_patch_bytes = patch;
    p.halo_tpi = compact ? (int)cdiv(P * wp, 128LL * msub) : (int)cdiv(P, (int64_t)rt * msub);
    p.halo_compact = compact;
    p.tiles_m = (int)(d.batch * p.halo_tpi);
    if (pair) {
        if (p.tiles_m % 2) ILLEGAL("pack_halo: the CTA pair needs an even number of M tiles (%d)", p.tiles_m);
        p.tiles_m /= 2;                                 // the tile loop runs over M-tile pairs
    } else if (hcl == 2) {
        if (s.b_resident) ILLEGAL("pack_halo: cluster_m 2 multicasts the filter ring; b_resident must be 0");
        if ((s.tile_n / p.atom_n) % 2) ILLEGAL("pack_halo: cluster_m 2 needs an even number of 128-byte filter blocks (tile_n)");
        if (p.tiles_m % 2) ILLEGAL("pack_halo: cluster_m 2 needs an even number of M tiles (%d)", p.tiles_m);
        if (d.f % p.atom_n) ILLEGAL("pack_halo: cluster_m 2 needs F %% %d == 0 (3-D filter TMA)", p.atom_n);
        p.tiles_m /= 2;                                 // the tile loop runs over M-tile pairs
    }
    p.halo_cl = hcl;
    p.kb_per_split = (int)cdiv(p.kb_total, p.split_k);
    if ((int64_t)(p.split_k - 1) * p.kb_per_split >= p.kb_total)
        ILLEGAL("split: split_k %d leaves an empty K segment (%d k-blocks of %d)", p.split_k, p.kb_total, s.tile_k);
    p.k_per_split = (int64_t)p.kb_per_split * s.tile_k;
    p.num_tiles = (int64_t)p.tiles_m * p.tiles_n * p.split_k;
    if (p.num_tiles >= (1ll << 31)) ILLEGAL("too many tiles");
    p.halo_pair = pair;
    p.halo_sfold = sfold;
    p.cta_group = pair ? 2 : 1;                         // UMMA M = 128 * cta_group (abi.cu idesc)
    p.block = kTcThreads;
    p.cluster = hcl;
    if (p.stream_k) {
        if (hcl != 1) ILLEGAL("pack_halo: stream-K needs cluster_m 1");
        p.sk_iters = p.num_tiles * (int64_t)p.kb_total;
        p.grid_x = (int)std::min<int64_t>(p.sk_iters, num_sms);
        p.sk_slot = 128LL * msub * s.tile_n;
        p.workspace_bytes = (int64_t)p.grid_x * p.sk_slot * 4;
        return XTC_OK;
    }
    if (p.split_cluster) {
        // the split_k segments of a tile = the CTAs of one cluster, reduced in the kernel
        if (hcl != 1) ILLEGAL("pack_halo: split_k_mode 2 needs cluster_m 1 (the cluster holds the K segments)");
        if (s.b_resident) ILLEGAL("pack_halo: split_k_mode 2 needs b_resident 0");
        p.num_tiles = (int64_t)p.tiles_m * p.tiles_n;
        p.cluster = p.split_k;
        const int64_t ctas = p.num_tiles * p.split_k;
        const int64_t cap = (int64_t)(num_sms / p.split_k) * p.split_k;
        if (s.persistent && cap < p.split_k) ILLEGAL("parallelize: %d SMs hold no cluster of %d CTAs", num_sms, p.split_k);
        p.grid_x = s.persistent ? (int)std::min<int64_t>(ctas, cap) : (int)ctas;
        return XTC_OK;
    }
    const int64_t ctas = p.num_tiles * hcl;
    p.grid_x = s.persistent ? (int)std::min<int64_t>(ctas, num_sms - num_sms % hcl) : (int)ctas;
    return XTC_OK;
}

// Warp-MMA engine (conv_mma.cu): mma.sync m16n8k16 tiles over an im2col gather, any channel count
static xtc_status plan_mma(const xtc_op_desc& d, const xtc_schedule& s, int num_sms, Plan& p, std::string& why) {
    if (d.in_dtype != XTC_BF16) ILLEGAL("MMA engine computes bf16 inputs (mma.sync m16n8k16 bf16 -> fp32)");
    if (s.tile_m != 64 && s.tile_m != 128 && !(s.pack_halo && (s.tile_m == 256 || s.tile_m == 512)))
        ILLEGAL("MMA engine: tile_m must be 64 or 128 (16-row warp tiles; 256 / 512 with pack_halo)");
    if (s.tile_n != 16 && s.tile_n != 32 && s.tile_n != 64) ILLEGAL("MMA engine: tile_n must be 16, 32 or 64");
    if (s.tile_k != 16 && s.tile_k != 32 && s.tile_k != 64) ILLEGAL("MMA engine: tile_k must be 16, 32 or 64");
    if (s.inner_m || s.inner_n) ILLEGAL("MMA engine: inner_m / inner_n must be 0 (the warp tile is 16 x tile_n)");
    if (s.unroll_k > 1 || s.vector_n > 1 || s.stages > 1 || s.swizzle) ILLEGAL("MMA engine: unroll_k, vector_n, stages, swizzle must be 0/1");
    if (p.split_k != 1) ILLEGAL("MMA engine: split_k must be 1");
    if (s.buffer_c || s.acc_buffers > 1) ILLEGAL("MMA engine: buffer_c 0, acc_buffers 0/1 (register accumulators)");
    if (s.cluster_m > 1 || s.cluster_n > 1 || s.pack_warps > 1 || s.b_resident)
        ILLEGAL("MMA engine: cluster_m, cluster_n, pack_warps, b_resident must be 0/1");
    if (s.pack_halo) {
        // pack above the (r, s, c) loops: the tile's input patch staged once in SMEM
        if (d.kind != XTC_OP_CONV2D) ILLEGAL("MMA engine: pack_halo is a conv2d placement");
        if (s.tile_k != 16) ILLEGAL("MMA engine pack_halo: tile_k must be 16 (the whole K is resident; 16 = the step)");
        if (d.c > 16) ILLEGAL("MMA engine pack_halo: C must be <= 16 (channels padded to 4/8/16 in the patch)");
        int64_t M_, N_, K_, P, Q;
        gemm_view(d, M_, N_, K_, P, Q);
        if (Q > 512) ILLEGAL("MMA engine pack_halo: Q must be <= 512 (one output row per CTA at most 16 warps)");
        MmaPatch g;
        // pack_halo 1: the TMA patch layout where it applies; 2: always the thread-filled padded layout
        if (s.pack_halo > 2) ILLEGAL("MMA engine: pack_halo must be 0, 1 (TMA patch where legal) or 2 (thread-filled)");
        const bool allow_tma = s.pack_halo == 1;
        if (!mma_patch_geom((int)d.h, (int)d.w, (int)d.c, (int)P, (int)Q, (int)d.r, (int)d.s, (int)d.stride_w,
                            (int)d.stride_h, (int)d.pad_w, s.tile_m, s.tile_n, dtype_size(d.out_dtype), allow_tma, g))
            ILLEGAL("MMA engine pack_halo: tile_m %d gives %d pixels per CTA (> 512)", s.tile_m, (int)(Q * (s.tile_m / Q)));
        if (g.smem > kSmemMaxOptin)
            ILLEGAL("MMA engine pack_halo: SMEM %d B (patch %d + filter %d + staging %d) > %d", g.smem, g.smem_patch,
                    g.smem_b, g.smem_out, kSmemMaxOptin);
        p.mma_patch = true;
        p.mp = g;
        p.block = g.warps * 32;
        p.smem = g.smem;
        p.tiles_m = (int)(d.batch * cdiv(P, g.tp));
        p.tiles_n = (int)cdiv(p.N, s.tile_n);
        p.kb_total = g.kp / 16;
        p.kb_per_split = p.kb_total;
        p.k_per_split = p.K;
        p.num_tiles = (int64_t)p.tiles_m * p.tiles_n;
        if (p.num_tiles >= (1ll << 31)) ILLEGAL("too many tiles");
        const int per_sm = std::max(1, std::min(2048 / p.block, kSmemMaxOptin / std::max(1, g.smem + 1024)));
        p.grid_x = s.persistent ? (int)std::min<int64_t>(p.num_tiles, (int64_t)num_sms * per_sm) : (int)p.num_tiles;
        return XTC_OK;
    }
    p.block = 256;
    p.smem = 0;
    p.tiles_m = (int)cdiv(p.M, s.tile_m);
    p.tiles_n = (int)cdiv(p.N, s.tile_n);
    p.kb_total = (int)cdiv(p.K, s.tile_k);
    p.kb_per_split = p.kb_total;
    p.k_per_split = p.K;
    p.num_tiles = (int64_t)p.tiles_m * p.tiles_n;
    if (p.num_tiles >= (1ll << 31)) ILLEGAL("too many tiles");
    p.grid_x = s.persistent ? (int)std::min<int64_t>(p.num_tiles, (int64_t)num_sms * 8) : (int)p.num_tiles;
    return XTC_OK;
}

static xtc_status plan_tc(const xtc_op_desc& d, const xtc_schedule& s, int num_sms, Plan& p, std::string& why) {
    // F32 inputs on the tensor cores: the 3xTF32 split, fp32-accurate:
    // a = hi + lo with hi = a truncated to tf32 (what kind::tf32 reads) and lo = a - hi
    // (exact in fp32); C = hi*lo + lo*hi + hi*hi.  Matmul, 1-CTA, single TMA producer.
    p.split3 = d.in_dtype == XTC_F32;
    if (p.split3) {
        if (d.kind != XTC_OP_MATMUL) ILLEGAL("tcgen05 fp32 (3xTF32 split) is defined for matmul only");
        if (s.pack_halo) ILLEGAL("tcgen05 fp32 (3xTF32 split): pack_halo must be 0");
        if (s.cluster_m > 1) ILLEGAL("tcgen05 fp32 (3xTF32 split): cluster_m must be 1");
        if (s.pack_warps > 1) ILLEGAL("tcgen05 fp32 (3xTF32 split): pack_warps must be 0 or 1 (warps 2-3 split)");
        if (s.b_resident) ILLEGAL("tcgen05 fp32 (3xTF32 split): b_resident must be 0");
    } else if (d.in_dtype != XTC_BF16 && d.in_dtype != XTC_TF32) {
        ILLEGAL("tcgen05 engine needs BF16, TF32 or F32 (3xTF32 split) inputs");
    }
    if (s.pack_halo) {
        if (s.cluster_n > 1) ILLEGAL("pack_halo: cluster_n must be 0 or 1 (cluster_m multicasts the filter)");
        p.atom_k = p.atom_n = 128 / dtype_size(d.in_dtype);
        return plan_tc_halo(d, s, num_sms, p, why);
    }
    int es = dtype_size(d.in_dtype);
    p.atom_k = 128 / es;          // elements per 128-byte swizzle row
    p.atom_n = 128 / es;
    int cg = s.cluster_m == 0 ? 1 : s.cluster_m;
    if (cg != 1 && cg != 2) ILLEGAL("tcgen05 cluster_m must be 1 (cta_group::1) or 2 (cta_group::2 CTA pair)");
    p.cta_group = cg;
    // M-subtiles: tile_m = 128 * cta_group * ms; ms = 2 stacks two UMMA row tiles per CTA that share
    // every B stage (matmul; B leaves L2 once per 256 rows per CTA instead of per 128)
    const int ms = s.tile_m == 256 * cg ? 2 : 1;
    if (s.tile_m != 128 * cg * ms)
        ILLEGAL("tcgen05 tile_m must be %d or %d for cluster_m=%d (128-row UMMA subtiles per CTA)", 128 * cg, 256 * cg, cg);
    if (s.inner_m != 0 && s.inner_m != 128 * cg) ILLEGAL("tcgen05 inner_m (UMMA M) must be %d", 128 * cg);
    if (ms == 2) {
        if (d.kind != XTC_OP_MATMUL) ILLEGAL("tcgen05 tile_m %d (two M-subtiles per CTA) applies to matmul only", s.tile_m);
        if (p.split3) ILLEGAL("tcgen05 two M-subtiles: not with the 3xTF32 split");
        if (s.b_resident) ILLEGAL("tcgen05 two M-subtiles: b_resident must be 0");
        if (s.cluster_n > 1) ILLEGAL("tcgen05 two M-subtiles: cluster_n must be 0 or 1");
    }
    p.msub = ms;
    if (s.inner_n != 0 && s.inner_n != s.tile_n) ILLEGAL("tcgen05 inner_n (UMMA N) must equal tile_n");
    int bn_cta = s.tile_n / cg;
    if (s.tile_n < p.atom_n * cg || s.tile_n > 256 || bn_cta % p.atom_n)
        ILLEGAL("tcgen05 tile_n must be a multiple of %d in [%d,256] (B swizzle atom x cta_group)", p.atom_n * cg, p.atom_n * cg);
    if (s.tile_k < p.atom_k || s.tile_k > 256 || s.tile_k % p.atom_k)
        ILLEGAL("tcgen05 tile_k must be a multiple of %d in [%d,256] (128-byte swizzle atom)", p.atom_k, p.atom_k);
    if (s.unroll_k > 1) ILLEGAL("tcgen05 unroll_k must be 0 or 1 (the k-steps of a stage are always fully unrolled)");
    if (s.pack_warps < 0 || s.pack_warps > 3) ILLEGAL("pack: pack_warps (TMA-issuing warps) must be in [0,3]");
    if (s.vector_n > 1) ILLEGAL("tcgen05 vector_n must be 0 (the UMMA atom is the vector unit)");
    if (s.stages < 2 || s.stages > 8) ILLEGAL("tcgen05 stages must be in [2,8]");
    // producer g % pack_warps fills slot g % stages after waiting for the slot's previous round
    // (k-block g - stages) to be consumed; its own previous wait only guarantees k-block
    // g - pack_warps - stages, so with pack_warps > stages the slot may still be two rounds behind
    // and the mbarrier parity wait aliases (race found by the schedule-invariance sweep)
    if (s.pack_warps > s.stages) ILLEGAL("pack: pack_warps %d > stages %d (ring slot parity would alias)", s.pack_warps, s.stages);
    if (s.swizzle != 0 && s.swizzle != 128) ILLEGAL("tcgen05 swizzle must be 128 (0 = default 128)");
    int accb = s.acc_buffers == 0 ? 1 : s.acc_buffers;
    if (accb < 1 || accb > 2) ILLEGAL("acc_buffers must be 1 or 2");
    int cols = accb * s.tile_n * ms;
    int alloc = 32;
    while (alloc < cols) alloc *= 2;
    if (alloc > 512) ILLEGAL("bufferize: %d TMEM columns (acc_buffers x tile_n, pow2) exceed 512", alloc);
    p.tmem_cols = alloc;
    int a_stage = 128 * ms * s.tile_k * es;
    int b_stage = s.tile_k * bn_cta * es;
    int smem = 0;
    if (s.b_resident) {
        // pack B once per CTA (outermost loop level): all k-blocks of B stay in SMEM
        if (s.b_resident != 1) ILLEGAL("b_resident must be 0 or 1");
        if (cdiv(p.N, s.tile_n) != 1) ILLEGAL("pack: b_resident needs a single N tile (N <= tile_n)");
        if (p.split_k != 1) ILLEGAL("pack: b_resident needs split_k 1");
        const int64_t kbt = cdiv(p.K, s.tile_k);
        const int64_t b_all = kbt * b_stage;
        const int64_t tot = b_all + (int64_t)s.stages * a_stage + (s.buffer_c ? kTcEpiSmem : 0) + kSmemReserve;
        if (tot > kSmemMaxOptin)
            ILLEGAL("pack: resident B (%lld B) + %d A stages + epilogue = %lld B SMEM exceeds %d B", (long long)b_all,
                    s.stages, (long long)tot, kSmemMaxOptin);
        smem = (int)tot;
    } else {
        // 3xTF32: every stage also holds the lo parts of its A and B tiles
        const int per_stage = (a_stage + b_stage) * (p.split3 ? 2 : 1);
        smem = s.stages * per_stage + (s.buffer_c ? kTcEpiSmem : 0) + kSmemReserve;
        // bufferize, overlapped: with two M-subtiles, bf16 output and 256-column tiles, the epilogue drains
        // TMEM into a 64 KB SMEM tile + registers and releases it before its (slow) TMA stores, so the
        // next tile's MMAs overlap the stores -- when the 64 KB fit
        if (ms == 2 && s.buffer_c && d.out_dtype == XTC_BF16 && p.split_k == 1 && s.tile_n == 256 &&
            !(d.consumer & XTC_CONSUMER_ACCUMULATE) && (d.consumer == 0 || s.fuse) &&
            accb == 1 && s.stages * per_stage + 2 * kTcEpiSmem + kSmemReserve <= kSmemMaxOptin &&
            getenv("XTC_NO_OVERLAP_EPILOGUE") == nullptr) {
            p.ovl = true;
            smem = s.stages * per_stage + 2 * kTcEpiSmem + kSmemReserve;
        }
        if (smem > kSmemMaxOptin) ILLEGAL("pack: %d stages x %d B + epilogue = %d B SMEM exceeds %d B",
                                          s.stages, per_stage, smem, kSmemMaxOptin);
    }
    p.smem = smem;
    // TMA pitch / alignment rules (cuda.h cuTensorMapEncodeTiled: strides % 16 B)
    int os = dtype_size(d.out_dtype);
    if (d.kind == XTC_OP_MATMUL) {
        int64_t lda = d.lda ? d.lda : d.k, ldb = d.ldb ? d.ldb : d.n;
        if ((lda * es) % 16 || (ldb * es) % 16) ILLEGAL("TMA needs 16-byte row pitch for A and B (lda, ldb)");
    } else {
        if (d.c % p.atom_k) ILLEGAL("tcgen05 conv2d needs C %% %d == 0 (one 128-byte channel block per im2col load)", p.atom_k);
        if ((d.f * es) % 16) ILLEGAL("TMA needs 16-byte row pitch for the RSCF filter");
        if (p.K % s.tile_k) ILLEGAL("tcgen05 conv2d needs R*S*C %% tile_k == 0");
        if (d.stride_h > 8 || d.stride_w > 8) ILLEGAL("im2col TMA traversal stride must be <= 8");
        if (d.pad_h > 127 || d.pad_w > 127 || d.r > 128 || d.s > 128) ILLEGAL("im2col corner offsets out of [-128,127]");
    }
    p.tiles_m = (int)cdiv(p.M, s.tile_m);
    p.tiles_n = (int)cdiv(p.N, s.tile_n);
    p.kb_total = (int)cdiv(p.K, s.tile_k);
    p.kb_per_split = (int)cdiv(p.kb_total, p.split_k);
    if ((int64_t)(p.split_k - 1) * p.kb_per_split >= p.kb_total)
        ILLEGAL("split: split_k %d leaves an empty K segment (%d k-blocks of %d)", p.split_k, p.kb_total, s.tile_k);
    p.k_per_split = (int64_t)p.kb_per_split * s.tile_k;
    p.num_tiles = (int64_t)p.tiles_m * p.tiles_n * p.split_k;
    if (p.num_tiles >= (1ll << 31)) ILLEGAL("too many tiles");
    if (s.buffer_c) {
        int64_t ldc = (d.kind == XTC_OP_MATMUL && d.ldc) ? d.ldc : p.n_total;
        if (p.split_k == 1 && (ldc * os) % 16) ILLEGAL("bufferize: TMA store needs a 16-byte output row pitch");
    }
    if (s.buffer_c && d.out_dtype == XTC_BF16 && p.split_k == 1 && s.tile_n % 64)
        ILLEGAL("bufferize: bf16 TMA-store staging needs tile_n %% 64 == 0");
    if (p.atomic && s.buffer_c) ILLEGAL("atomic split-K uses direct red.global stores: buffer_c must be 0");
    p.block = kTcThreads;
    p.cluster = cg;
    if (p.split_cluster) {
        // one cluster of split_k CTAs per output tile; persistent: whole clusters on at most num_sms SMs
        if (cg != 1 || ms != 1) ILLEGAL("split: split_k_mode 2 needs cluster_m 1 and tile_m 128 (one UMMA tile per CTA)");
        if (s.cluster_n > 1) ILLEGAL("split: split_k_mode 2 needs cluster_n 0/1 (the cluster holds the K segments)");
        if (s.b_resident) ILLEGAL("split: split_k_mode 2 needs b_resident 0");
        p.num_tiles = (int64_t)p.tiles_m * p.tiles_n;
        p.cluster = p.split_k;
        const int64_t ctas = p.num_tiles * p.split_k;
        const int64_t cap = (int64_t)(num_sms / p.split_k) * p.split_k;
        if (s.persistent && cap < p.split_k) ILLEGAL("parallelize: %d SMs hold no cluster of %d CTAs", num_sms, p.split_k);
        p.grid_x = s.persistent ? (int)std::min<int64_t>(ctas, cap) : (int)ctas;
        return XTC_OK;
    }
    if (p.stream_k) {
        if (cg != 1 || ms != 1) ILLEGAL("split: stream-K needs cluster_m 1 and tile_m 128 (one UMMA tile per CTA)");
        if (s.cluster_n > 1) ILLEGAL("split: stream-K needs cluster_n 0/1");
        p.sk_iters = p.num_tiles * (int64_t)p.kb_total;
        p.grid_x = (int)std::min<int64_t>(p.sk_iters, num_sms);
        p.sk_slot = 128LL * s.tile_n;
        p.workspace_bytes = (int64_t)p.grid_x * p.sk_slot * 4;
        return XTC_OK;
    }
    // cluster_n: cn CTAs on adjacent N tiles of one M tile share every A stage by TMA multicast
    // (each loads 128/cn of its rows); a "tile" of the tile map is then a cluster tile
    const int cn = s.cluster_n == 0 ? 1 : s.cluster_n;
    if (cn != 1) {
        if (cn != 2 && cn != 4) ILLEGAL("parallelize: cluster_n must be 1, 2 or 4");
        if (d.kind != XTC_OP_MATMUL) ILLEGAL("parallelize: cluster_n (A multicast) applies to matmul only");
        if (cg != 1) ILLEGAL("parallelize: cluster_n needs cluster_m 1");
        if (p.split3) ILLEGAL("parallelize: cluster_n needs bf16/tf32 inputs (not the 3xTF32 split)");
        if (s.b_resident) ILLEGAL("parallelize: cluster_n needs b_resident 0");
        if (p.tiles_n % cn) ILLEGAL("parallelize: cluster_n %d must divide the %d N tiles", cn, p.tiles_n);
        p.cluster_n = cn;
        p.cluster = cn;
        p.num_tiles = (int64_t)p.tiles_m * (p.tiles_n / cn) * p.split_k;
        const int64_t ctas = p.num_tiles * cn;
        p.grid_x = s.persistent ? (int)std::min<int64_t>(ctas, num_sms - num_sms % cn) : (int)ctas;
        return XTC_OK;
    }
    // one CTA (pair) per tile, or a persistent grid of at most one CTA per SM
    const int64_t ctas = p.num_tiles * cg;
    p.grid_x = s.persistent ? (int)std::min<int64_t>(ctas, num_sms - num_sms % cg) : (int)ctas;
    return XTC_OK;
}

xtc_status make_plan(const xtc_op_desc& d, const xtc_schedule& s, int num_sms, Plan& p, std::string& why) {
    xtc_status st = check_desc(d, why);
    if (st != XTC_OK) return st;
    if (num_sms <= 0) num_sms = kNumSmsB200;
    p = Plan();
    p.sch = s;
    p.engine = s.engine;
    int64_t M, N, K, P, Q;
    gemm_view(d, M, N, K, P, Q);
    p.M = M; p.N = N; p.K = K; p.n_total = N;
    if (s.order != XTC_ORDER_MN && s.order != XTC_ORDER_NM) ILLEGAL("interchange: order must be 0 (MN) or 1 (NM)");
    if (s.raster_group < 0 || s.raster_group > 64) ILLEGAL("raster_group must be in [0,64]");
    if (s.persistent != 0 && s.persistent != 1) ILLEGAL("persistent must be 0 or 1");
    // parallelize over a number of cores: the persistent grid spreads over at most
    // grid_sms SMs of the device (0 = all of them)
    if (s.grid_sms < 0 || s.grid_sms > 4096) ILLEGAL("parallelize: grid_sms must be in [0,4096]");
    if (s.grid_sms && !s.persistent) ILLEGAL("parallelize: grid_sms needs persistent 1 (one CTA per tile otherwise)");
    if (s.grid_sms) num_sms = std::min(num_sms, (int)s.grid_sms);
    p.split_k = s.split_k == 0 ? 1 : s.split_k;
    if (p.split_k < 1 || p.split_k > 64) ILLEGAL("split_k must be in [1,64]");
    if (s.split_k_mode < XTC_SPLITK_ORDERED || s.split_k_mode > XTC_SPLITK_STREAM) ILLEGAL("unknown split_k_mode");
    // stream-K: the split points of the flattened (tile, k-block) loop come from the persistent grid
    p.stream_k = s.split_k_mode == XTC_SPLITK_STREAM;
    if (p.stream_k) {
        if (s.engine != XTC_ENGINE_TCGEN05) ILLEGAL("split: split_k_mode 3 (stream-K) needs the tcgen05 engine");
        if (p.split_k != 1) ILLEGAL("split: stream-K derives the split points from the grid; split_k must be 0/1");
        if (!s.persistent) ILLEGAL("split: stream-K needs persistent 1 (a fixed grid of co-resident CTAs)");
    }
    p.atomic = (p.split_k > 1 && s.split_k_mode == XTC_SPLITK_ATOMIC);
    // the K segments of a tile as the CTAs of one cluster, reduced inside the kernel (splitk_cluster.cuh)
    p.split_cluster = (p.split_k > 1 && s.split_k_mode == XTC_SPLITK_CLUSTER);
    if (p.split_cluster) {
        if (s.engine != XTC_ENGINE_TCGEN05) ILLEGAL("split: split_k_mode 2 (cluster reduction) needs the tcgen05 engine");
        if (p.split_k > kSplitClusterMaxCtas) ILLEGAL("split: split_k_mode 2 puts the %d K segments in one cluster (<= %d CTAs)",
                                                     p.split_k, kSplitClusterMaxCtas);
    }
    if (p.atomic && d.out_dtype != XTC_F32) ILLEGAL("atomic split-K needs fp32 output");
    if (s.split_n_at) {
        if (s.split_n_at < 0 || s.split_n_at >= N) ILLEGAL("split: split_n_at %d must be in (0, N=%lld)", s.split_n_at, (long long)N);
        if (d.kind != XTC_OP_MATMUL) ILLEGAL("split_n_at is defined for matmul only");
        p.has_tail = true;
        p.tail_n0 = s.split_n_at;
        p.tail_n = N - s.split_n_at;
        p.N = s.split_n_at;
        // remainder root: SIMT 16x16 tiles, 1x1 inner (the paper's scalar remainder loop)
        p.tail_grid_x = (int)cdiv(p.tail_n, 16);
        p.tail_grid_y = (int)cdiv(M, 16);
        if (d.in_dtype != XTC_F32 && d.in_dtype != XTC_BF16 && d.in_dtype != XTC_TF32) ILLEGAL("bad dtype");
    }
    // fuse: the consumer runs in the producer's epilogue, in the split-K
    // reduction (which produces the complete sums), or as its own elementwise pass
    if (s.fuse != 0 && s.fuse != 1) ILLEGAL("fuse must be 0 or 1");
    if (d.consumer) {
        if (s.fuse && p.atomic && (d.consumer & XTC_CONSUMER_RELU))
            ILLEGAL("fuse: relu cannot be fused with atomic split-K (partial sums)");
        if (!s.fuse && (d.consumer & XTC_CONSUMER_ACCUMULATE))
            ILLEGAL("fuse: accumulate must be fused (an unfused C += A*B would need a temporary for A*B)");
        // atomic split-K: the first K segment adds the bias, accumulate = C is not cleared
        p.cons_epi = (s.fuse && (p.split_k == 1 || p.atomic)) ? d.consumer : 0;
        p.cons_reduce = (s.fuse && p.split_k > 1 && !p.atomic) ? d.consumer : 0;
        p.cons_pass = s.fuse ? 0 : d.consumer;
        p.cons_tail = s.fuse ? d.consumer : 0;
    }
    if (s.engine == XTC_ENGINE_SIMT) st = plan_simt(d, s, num_sms, p, why);
    else if (s.engine == XTC_ENGINE_TCGEN05) st = plan_tc(d, s, num_sms, p, why);
    else if (s.engine == XTC_ENGINE_MMA) {
        if (p.has_tail) ILLEGAL("MMA engine: split_n_at must be 0");
        if (p.atomic) ILLEGAL("MMA engine: split_k must be 1");
        st = plan_mma(d, s, num_sms, p, why);
    }
    else ILLEGAL("unknown engine %d", s.engine);
    if (st != XTC_OK) return st;
    if (p.grid_x < std::max(1, p.cluster))
        ILLEGAL("parallelize: grid_sms %d leaves no room for one cluster of %d CTAs", s.grid_sms, p.cluster);
    if (p.split_k > 1 && !p.atomic) {
        p.ws_ld = cdiv(p.N, 4) * 4;
        p.workspace_bytes = (int64_t)p.split_k * p.M * p.ws_ld * 4;
    }
    // (stream-K: per-CTA partial slots, sized by the planner above)
    return XTC_OK;
}

}  // namespace xtc
