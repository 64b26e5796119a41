// xtc_internal.h -- types shared by the planner (host) and the sm_100a kernels.
// Not part of the public ABI (include/xtc.h is).
#pragma once
#include <stdint.h>
#include <functional>
#include <string>
#include <vector>
#include "../../include/xtc.h"
#include <cuda_runtime.h>

#ifdef __CUDACC__
#define XTC_HD __host__ __device__ __forceinline__
#else
#define XTC_HD inline
#endif

namespace xtc {

constexpr int kNumSmsB200 = 148;
constexpr int kSmemMaxOptin = 232448;       // sm_100: (228 - 1) KB per CTA (opt-in)
constexpr int kSmemReserve = 2048;          // barriers + alignment slack in the tcgen05 kernel
constexpr int kTcThreads = 256;             // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warp3 idle, warps4-7 epilogue
constexpr int kTcEpiStageBytes = 4096;      // one warp's 32 rows x 128 B output staging chunk
constexpr int kTcEpiBuffers = 2;            // double-buffered per warp
constexpr int kTcEpiSmem = 4 * kTcEpiStageBytes * kTcEpiBuffers;
constexpr int kHaloMaxPatchBufs = 4;        // conv_halo: patch buffers (at most; the planner fits what SMEM allows)
constexpr int kHaloMaxResidentKb = 32;      // conv_halo: resident-filter k-blocks (one mbarrier each)
constexpr int kSplitClusterMaxCtas = 16;    // split_k_mode 2: K segments per cluster (> 8: non-portable size)
constexpr int kSkMaxCtas = 4096;            // split_k_mode 3: stream-K grid limit (publish flags per op)

// cudaFuncSetAttribute is a driver round trip: set the dynamic-SMEM opt-in once
// per kernel variant and device, not on every launch (sweeps launch thousands).
cudaError_t ensure_smem_attr_impl(const void* kernel, int smem);   // keyed by (kernel, device)

template <typename F>
inline cudaError_t ensure_smem_attr(F* kernel, int smem) {
    return ensure_smem_attr_impl(reinterpret_cast<const void*>(kernel), smem);
}
// cluster sizes 9..16 need cudaFuncAttributeNonPortableClusterSizeAllowed (set once per kernel)
cudaError_t ensure_nonportable_cluster_impl(const void* kernel);
template <typename F>
inline cudaError_t ensure_nonportable_cluster(F* kernel) {
    return ensure_nonportable_cluster_impl(reinterpret_cast<const void*>(kernel));
}

// SIMT register budget: the TM x TN accumulator tile plus operands must fit
// without spills, so large thread tiles cap the CTA size (65536 regs / SM).
XTC_HD constexpr int simt_max_threads(int tm, int tn) {
    return tm * tn >= 32 ? 256 : (tm * tn >= 16 ? 512 : 1024);
}
// Register-tiled variants ask for two resident CTAs per SM (<= 128 regs/thread): one CTA leaves 2 warps
// per scheduler, too few to hide LDS latency -- except the 8x8 tile, whose 64 accumulators + 16 fragments
// spilled to the stack at 128 registers (136 bytes, 3x slower); it gets the whole register file.
XTC_HD constexpr int simt_min_blocks(int tm, int tn) { return tm * tn >= 64 ? 1 : (tm * tn >= 32 ? 2 : 1); }

// Tile-order mapping: the schedule's interchange + grouped raster.
// Linear tile id -> (split segment ks, tile row mb, tile col nb).
// order MN: the M-tile loop is outer, the N-tile loop inner; raster_group G
// strip-mines the outer loop by G and moves the inner loop inside the strip.
struct TileMap {
    int32_t tiles_m, tiles_n, split_k, order, group;
};

// 32-bit unsigned arithmetic: the planner caps the tile count below 2^31, and 64-bit
// integer division is a long software sequence on the GPU (every role calls this per tile).
XTC_HD void tile_coords(const TileMap& t, int64_t id64, int& mb, int& nb, int& ks) {
    const uint32_t id = (uint32_t)id64;
    const uint32_t per = (uint32_t)t.tiles_m * (uint32_t)t.tiles_n;
    const uint32_t k = id / per;
    const uint32_t r = id - k * per;
    const uint32_t outer_n = (t.order == XTC_ORDER_MN) ? t.tiles_m : t.tiles_n;   // extent of outer loop
    const uint32_t inner_n = (t.order == XTC_ORDER_MN) ? t.tiles_n : t.tiles_m;
    const uint32_t G = t.group < 1 ? 1u : (uint32_t)t.group;
    const uint32_t strip = G * inner_n;
    const uint32_t g = r / strip;
    const uint32_t w = r - g * strip;
    uint32_t rows = outer_n - g * G;
    if (rows > G) rows = G;
    const uint32_t inner = w / rows;
    const uint32_t outer = g * G + (w - inner * rows);
    ks = (int)k;
    if (t.order == XTC_ORDER_MN) { mb = (int)outer; nb = (int)inner; } else { nb = (int)outer; mb = (int)inner; }
}

// Warp-MMA engine with the pack at the tile level (engine 2, pack_halo = 1; conv_mma.cu): a CTA tile
// is tp whole output rows of one image (px = tp*Q pixels, 32 per warp); its input patch of pr input
// rows is staged in SMEM once, K is ordered (r, then a contiguous run of kpr = ksr*16 elements of
// patch row r), so every 16-deep MMA step of a pixel is one contiguous 32-byte run of its patch row
// and the A fragments are plain 32-bit LDS at (pixel base + offset).  Two patch layouts:
//  * tma (sw*C even, W*C % 16 == 0): the raw NHWC row, loaded by ONE 4-D TMA {16, chunks, pr, 1}
//    over the input viewed as {16-element chunk, W*C/16 chunks, H, N}, double-buffered; the row
//    starts at element x0 = 16*floor(-pw*C/16) (out-of-bounds chunks / rows are TMA zero fill =
//    the zero padding, reading 3); pixel q's run starts at element q*sw*C - pw*C - x0 - delta,
//    delta in {0,1} making every start even (4-byte aligned pairs); filter tap t = kl - delta.
//  * padded (otherwise, C <= 16): pixel slots of cp = 4/8/16 channels filled by the threads
//    (zeros past C and outside the image), taps s padded to sp; tap t = kl, s = t / cp.
// Padded K positions carry zero filter weights.
struct MmaPatch {
    int32_t tma, tp, cp, sp, ksr, kpr, kp, pr, px, warps, b_pitch;
    int32_t wpatch;          // padded: pixel slots per patch row
    int32_t chunks, x0;      // tma: 16-element chunks per patch row, first element of the row
    int32_t rowpitch;        // bytes per patch row in SMEM
    int32_t pix_stride;      // elements between the runs of adjacent output pixels (sw*cp or sw*C)
    int32_t off0;            // element offset of pixel 0's run in its patch row
    int32_t bcp, delta;      // filter packing: tap t = kl - delta, s = t / bcp, c = t % bcp (c < C valid)
    int32_t smem_patch;      // bytes per patch buffer (x nbuf)
    int32_t nbuf, smem_b, smem_out, smem;
};
XTC_HD bool mma_patch_geom(int H, int W, int C, int P, int Q, int R, int S, int sw, int sh, int pw, int tile_m,
                           int tile_n, int out_size, bool allow_tma, MmaPatch& g) {
    (void)H;
    if (Q <= 0 || P <= 0 || C > 16) return false;
    g.tp = tile_m / Q < 1 ? 1 : tile_m / Q;
    if (g.tp > P) g.tp = P;
    g.px = g.tp * Q;
    g.warps = (g.px + 31) / 32;
    g.pr = (g.tp - 1) * sh + R;
    g.tma = allow_tma && (sw * C) % 2 == 0 && (W * C) % 16 == 0;
    if (g.tma) {
        g.cp = C;
        g.x0 = -(((pw * C) + 15) / 16) * 16;                     // 16 * floor(-pw*C / 16)
        g.delta = (-pw * C - g.x0) & 1;
        g.kpr = (S * C + g.delta + 15) / 16 * 16;
        g.off0 = -pw * C - g.x0 - g.delta;
        g.pix_stride = sw * C;
        const int last = (Q - 1) * g.pix_stride + g.off0 + g.kpr - 1;   // last element read, from x0
        g.chunks = last / 16 + 1;
        if (g.chunks > 256 || g.pr > 256) g.tma = 0;
    }
    if (g.tma) {
        g.sp = 0; g.wpatch = 0;
        g.rowpitch = g.chunks * 32;
        g.bcp = C;
        g.nbuf = 2;
        g.smem_patch = (g.pr * g.rowpitch + 127) / 128 * 128;
    } else {
        g.cp = C <= 4 ? 4 : (C <= 8 ? 8 : 16);
        const int spq = 16 / g.cp;                                 // taps per 16-deep step
        g.sp = (S + spq - 1) / spq * spq;
        g.kpr = g.sp * g.cp;
        g.wpatch = (Q - 1) * sw + g.sp;
        g.rowpitch = g.wpatch * g.cp * 2;
        g.pix_stride = sw * g.cp;
        g.off0 = 0; g.x0 = 0; g.chunks = 0;
        g.bcp = g.cp; g.delta = 0;
        g.nbuf = 1;
        g.smem_patch = (g.pr * g.rowpitch + 127) / 128 * 128;
    }
    g.ksr = g.kpr / 16;
    g.kp = R * g.kpr;
    g.b_pitch = g.kp + 8;                                         // elements; = 8 mod 16 -> conflict-free B fragments
    g.smem_b = (tile_n * g.b_pitch * 2 + 127) / 128 * 128;
    g.smem_out = g.warps * 32 * tile_n * out_size;
    g.smem = g.nbuf * g.smem_patch + g.smem_b + g.smem_out + 16 + 4 * g.kp;  // + 2 mbarriers + the k table
    return g.warps <= 16;
}
// ------------------------------------------------------------------ plans --
struct Plan {
    xtc_schedule sch{};
    int engine = 0;
    // GEMM view of the main root
    int64_t M = 0, N = 0, K = 0;        // N = columns of the main root (split_n_at or full N)
    int64_t n_total = 0;
    int32_t tiles_m = 0, tiles_n = 0, split_k = 1;
    int64_t num_tiles = 0;              // tiles_m * tiles_n * split_k
    int64_t k_per_split = 0;            // SIMT: K elements per segment (multiple of tile_k)
    int32_t kb_total = 0, kb_per_split = 0;   // tcgen05: k-blocks of tile_k
    int32_t grid_x = 1, grid_y = 1, grid_z = 1, block = 1, cluster = 1;
    int32_t smem = 0, tmem_cols = 0;
    int32_t cta_group = 1;
    bool split3 = false;                // tcgen05 with F32 inputs: 3xTF32 split (hi*lo + lo*hi + hi*hi)
    int32_t atom_k = 0, atom_n = 0;     // tcgen05: elements per 128-byte swizzle row
    int64_t ws_ld = 0;                  // split-K workspace row pitch (floats)
    int64_t workspace_bytes = 0;
    bool atomic = false;
    // split_n_at remainder root (SIMT, fixed 16x16x16 1x1 tile)
    // consumer (XTC_CONSUMER_* bits) placement: fused in the epilogue, fused in the split-K
    // reduction, in the split_n_at remainder root, or a separate pass (fuse = 0)
    int32_t cons_epi = 0, cons_reduce = 0, cons_pass = 0, cons_tail = 0;
    bool has_tail = false;
    int64_t tail_n0 = 0, tail_n = 0;
    int32_t tail_grid_x = 0, tail_grid_y = 0;
    // pack_halo conv (planner.cpp plan_tc_halo): Wp pixel slots per output row, rt output
    // rows per 128-row UMMA tile, msub UMMA tiles per CTA tile, pr patch rows, planes
    // 128-byte channel planes, nbuf patch buffers, tpi tiles per image
    bool halo = false;
    int32_t halo_wp = 0, halo_rt = 0, halo_msub = 0, halo_pr = 0, halo_planes = 0, halo_nbuf = 0, halo_tpi = 0;
    int32_t halo_cl = 1;                // CTAs per cluster sharing the filter stream (TMA multicast, or a pair)
    bool halo_pair = false;             // inner_m 256: cta_group::2 UMMAs (M = 256) over a CTA pair
    int32_t halo_sfold = 1;             // inner_n = S * tile_n: the filter row's S taps folded into the UMMA N
    bool halo_compact = false;          // pack_halo 2: rows at Wc = Q + S - 1 slots, tiles of consecutive rows
    bool halo_b64 = false;              // CTA pair with tile_n = 64 (bf16): 64-byte-swizzle filter halves per CTA
    bool ovl = false;                   // overlapped epilogue (see TcParams::ovl); 64 KB epilogue SMEM
    int32_t msub = 1;                   // tcgen05 matmul: 128-row M-subtiles per CTA (tile_m = 128*cta_group*msub)
    bool stream_k = false;              // split_k_mode 3: stream-K over the persistent grid (stream_k.cuh)
    int64_t sk_iters = 0, sk_slot = 0;  // num_tiles x kb_total iterations; partial slot floats per CTA
    bool split_cluster = false;         // split_k_mode 2: the split_k K segments of a tile = one cluster's CTAs,
                                        // reduced in-kernel; num_tiles then counts output tiles
    int32_t cluster_n = 1;              // tcgen05 matmul: CTAs on adjacent N tiles sharing A by multicast;
                                        // tiles (num_tiles) then count cluster tiles of cluster_n N tiles
    int64_t halo_patch_bytes = 0;
    bool mma_patch = false;             // engine 2 with pack_halo: the patch-staged warp-MMA conv
    MmaPatch mp{};
};

// Host-only: legality + plan derivation.  Returns XTC_OK or an error with reason.
xtc_status make_plan(const xtc_op_desc& d, const xtc_schedule& s, int num_sms, Plan& p, std::string& why);
xtc_status check_desc(const xtc_op_desc& d, std::string& why);
void gemm_view(const xtc_op_desc& d, int64_t& M, int64_t& N, int64_t& K, int64_t& P, int64_t& Q);

// ------------------------------------------------------- kernel parameters --
struct ConvGeom {
    int32_t is_conv;
    int32_t H, W, C, P, Q, R, S, sh, sw, ph, pw;
};

struct SimtParams {
    const void* A; const void* B; void* C; float* Wk;
    int64_t M, N, K, lda, ldb, ldc, ws_ld;
    int32_t tile_m, tile_n, tile_k, pad, stages;
    int64_t k_per_split;
    TileMap tm;
    int64_t num_tiles;
    int32_t out_bf16, split_out, atomic;
    int32_t fast;        // aligned matmul: 16-byte vectorised pack + float4 A fragments
    int32_t cons;        // fused consumer bits (XTC_CONSUMER_*) applied in the epilogue
    const float* bias;   // XTC_CONSUMER_BIAS: one fp32 value per output column
    ConvGeom cg;
};

struct TcParams {
    int64_t M, N, K;
    int32_t tile_n, tile_k, stages;
    int32_t kb_total, kb_per_split;
    TileMap tm;
    int64_t num_tiles;
    int32_t acc_buffers, buffer_c, atomic, out_bf16, split_out;
    int32_t pack_warps;      // 1..3 TMA-issuing warps (warps 0, 2, 3)
    int32_t b_resident;      // all of B packed once per CTA (kb_total x b_stage_bytes before the A ring)
    int32_t cons;            // fused consumer bits (XTC_CONSUMER_*) applied in the epilogue
    const float* bias;       // XTC_CONSUMER_BIAS: one fp32 value per output column
    int32_t a3d, b3d;        // one 3-D TMA per stage for all 128-B atoms of A / B (tmA / tmB are 3-D maps)
    int32_t debug_late_alloc;  // diagnostics (A/B): XTC_DEBUG_LATE_ALLOC=1 allocates TMEM before the
                               // prologue barrier, i.e. the producers wait for the allocation
    int32_t debug_skip_mma;  // diagnostics only: XTC_DEBUG_SKIP_MMA, or XTC_DEBUG_SKIP=mask.  conv_halo (output
                             // invalid unless noted): 1 no MMAs, 2 no patch TMA, 4 no output stores, 8 no TMEM
                             // drain, 16 plain arrives, 64 no epilogue, 128 sleeping waits, 256 no tap shifts,
                             // 512 every UMMA twice, 1024 (+64) free-run MMA warp (no patch loads, no per-tile
                             // waits or commits), 2048 (+1024) per-tile commits, 4096 no per-tile tcgen05
                             // fence; valid output: 8192 no early producer start, 65536 full bulk wait at exit,
                             // 0x20000 last tile drained by warps 4..7 only.
                             // tc_gemm: any bit but 65536 = no MMAs; 65536 as above.
    int64_t ldc, ws_ld;
    void* C; float* Wk;
    uint32_t idesc;
    uint32_t tmem_cols;
    uint32_t a_stage_bytes, b_stage_bytes;
    uint32_t lo_off;         // 3xTF32: byte offset from a hi stage (A or B ring) to its lo copy
    ConvGeom cg;
    // pack_halo conv only (see Plan)
    int32_t wp, rt, msub, planes, nbuf, tpi, cl, pair;
    int32_t b64;             // pack_halo CTA pair, tile_n 64: each CTA's filter half is 32 columns x 64 bytes
                             // (TMA SWIZZLE_64B, UMMA MN-major SW64 descriptor: 8-row groups 512 bytes apart)
    int32_t compact;         // pack_halo 2: wp = Q + S - 1 and a tile = 128*msub consecutive virtual rows
                             // of an image (starts mid-row at TileInfo::off)
    int32_t sfold;           // pack_halo s-fold: the S taps of a filter row are the N blocks of one UMMA
                             // (N = S * tile_n); the epilogue sums block s of row v + s (1 = off)
    int32_t cn;              // cluster_n: CTAs of a cluster on adjacent N tiles, A stages multicast (1 = none)
    int32_t ms;              // M-subtiles per CTA (tile_m = 128 * cta_group * ms; matmul: 1 or 2)
    int32_t ovl;             // overlapped epilogue (two M-subtiles, bf16, tile_n 256): subtile 1 drained to a
                             // 64 KB SMEM tile, subtile 0 to registers, TMEM released before the stores
    uint32_t patch_bytes, plane_bytes;
    uint32_t patch_tx;       // bytes the patch TMAs deliver (planes x rows x Wp x 128; planes start 1024-aligned)
    // Diagnostics (XTC_TRACE): %globaltimer stamps for CTAs < kTraceCtas, laid out
    // [cta][kTraceSlots]: slot 0 kernel entry, 1 setup done; producer issue of k-block i at
    // 8+i, MMA full-wait done at 8+kTraceK+i, epilogue tile j start/end at 8+2kTraceK+2j(+1).
    uint64_t* trace;
    // xtc_run_gather (fused all-gather): n_gather CUtensorMaps in device memory, one per
    // destination ([dest_rows][N] each); output tile rows land at gather_row0 + row
    const void* gather;
    int32_t n_gather, gather_row0;
    // split_k_mode XTC_SPLITK_CLUSTER: the ksc K segments of a tile are the CTAs of one cluster
    // (1 = off); cons_red = the consumer bits applied by that in-kernel reduction
    int32_t ksc, cons_red;
    // xtc_run_multicast: the staged output tiles are read back from SMEM and written with 16-byte
    // stores to mc ([rows][mc_ld] elements, tile rows at gather_row0 + row); mc_mode 1 = st.global,
    // 2 = multimem.st (NVLS multicast address), 0 = off
    void* mc;
    int64_t mc_ld;
    int32_t mc_mode;
    // split_k_mode XTC_SPLITK_STREAM (stream_k.cuh): stream-K over sk_iters = num_tiles x kb_total
    // iterations; CTA g's partial slot is Wk + g * sk_slot floats, its flags sk_flags[4g .. 4g+3]
    // (one per epilogue warp) hold the epoch of the launch that last published it
    int32_t sk;
    int64_t sk_iters, sk_slot;
    uint32_t* sk_flags;
    uint32_t sk_epoch;
};
// conv_halo: the first kTileTable tiles of a CTA's walk, decoded once into SMEM (after the barriers)
struct TileInfo {
    int32_t t, nimg, p0, n0, ks, kb0, kb1, off;   // off: pack_halo 2, the tile's first slot in patch row 0
};
constexpr int kTileTable = 64;
constexpr int kTileTableBytes = kTileTable * (int)sizeof(TileInfo) + 16;
constexpr int kTraceCtas = 160;          // >= #SMs: the whole persistent grid
constexpr int kTraceK = 96;
constexpr int kTraceTiles = 16;
constexpr int kTracePhase = 8 + 2 * kTraceK + 2 * kTraceTiles;   // conv_halo epilogue phase cycle totals (warp 4):
                                                                   // +0 tfull wait, +1 tile decode, +2 TMEM ld+wait,
                                                                   // +3 staging-buffer wait, +4 stage+store, +5 tiles;
                                                                   // MMA warp: +6 wait cycles, +7 issue cycles
constexpr int kTraceSlots = kTracePhase + 8;

// Validation of the consumer (harness.cu compare_kernel): bits, bias, and the snapshot of
// the output taken before the validated run (XTC_CONSUMER_ACCUMULATE; same layout as C).
struct CmpConsumer {
    int32_t cons;
    const float* bias;
    const void* c_old;
};

// counters.cpp: named hardware counters through the CUPTI range profiler (dlopen'ed).
// split_counter_names strips the "gpu." prefix; collect_counters wraps one range around
// run_once() (replayed once per counter pass, each replay preceded by prepare() outside the range) and returns false with `why` when CUPTI,
// the device or a metric name is unavailable.
std::vector<std::string> split_counter_names(const char* list);
bool collect_counters(int device, const std::vector<std::string>& names, const std::function<bool()>& prepare,
                      const std::function<bool()>& run_once, std::vector<double>& values, std::string& why);

}  // namespace xtc
