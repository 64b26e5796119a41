// conv_mma.cu -- KB3s: implicit-GEMM conv2d (and matmul) for operands TMA and tcgen05 cannot
// address: a channel count that is not a multiple of the 128-byte swizzle atom, e.g. the
// paper's stem conv [112,112,16] x [7,7,3] step 2 (DESIGN reading 4: C = 3, a 6-byte
// pixel).  Engine XTC_ENGINE_MMA: warp-level tensor-core tiles (mma.sync.m16n8k16 bf16 ->
// fp32), the instruction tier that needs no TMA-addressable layout.
//
// The contraction is the paper's Fig.2 loop nest over the implicit-GEMM view M = N*P*Q,
// N = F, K = R*S*C (c fastest), with
//   strip_mine -> CTA tile tile_m x tile_n x tile_k (k padded to the 16-deep MMA step; the
//                 pad reads zeros), warp tile 16 x tile_n (tile_m / 16 warps)
//   pack       -> A gathered through the im2col index map (zero padding = the bounds test,
//                 reading 3) and B transposed, both into SMEM, once per k-chunk
//   bufferize  -> fp32 accumulators in registers; the consumer and the single rounding in
//                 the epilogue (fuse)
//   parallelize-> one CTA per tile or a persistent grid
// For the stem, K = 147 -> 160 and N = 16: a 128 x 16 x 160 tile is 0.66 MFLOP, too small for
// tcgen05 (a 128 x 16 UMMA is issue- and SMEM-port-bound), and the op is bound by its gather.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string.h>
#include <cuda.h>
#include "consumer.cuh"
#include "ptx.cuh"
#include "xtc_internal.h"

namespace xtc {

struct MmaParams {
    const uint16_t* A;           // conv: x NHWC; matmul: A [M][lda]
    const uint16_t* B;           // conv: w RSCF = [K][F]; matmul: B [K][ldb]
    void* C;                     // [M][ldc]
    int64_t M, N, K, lda, ldb, ldc;
    int32_t tile_m, tile_n, tile_k;
    TileMap tm;
    int64_t num_tiles;
    int32_t out_bf16, cons;
    const float* bias;
    ConvGeom cg;
    MmaPatch pg;                 // pack_halo: the patch-staged conv (conv_mma_patch_kernel)
    int32_t batch;
};

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ uint32_t lds32(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}

// NT = tile_n / 8 n8-blocks per warp; BK = k-chunk (multiple of 16)
template <int NT, int BK>
__global__ void __launch_bounds__(256) conv_mma_kernel(const MmaParams p) {
    constexpr int LDS = BK + 8;                     // bf16 row pitch in SMEM (breaks bank aliasing)
    __shared__ __align__(16) uint16_t As[128 * LDS];
    __shared__ __align__(16) uint16_t Bs[NT * 8 * LDS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int BM = p.tile_m;                        // 64 or 128: BM / 16 warps compute
    const bool is_conv = p.cg.is_conv != 0;
    const int C = p.cg.C, S = p.cg.S;
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, ks;
        tile_coords(p.tm, t, mb, nb, ks);
        const int64_t m0 = (int64_t)mb * BM, n0 = (int64_t)nb * (NT * 8);
        // each thread gathers for one A row (tid % BM) a strided set of k (tid / BM + j * (256 / BM))
        const int arow = tid % BM, akoff = tid / BM, astep = 256 / BM;
        const int64_t m = m0 + arow;
        int img = 0, h0 = 0, w0 = 0;
        if (is_conv && m < p.M) {
            const int pq = p.cg.P * p.cg.Q;
            img = (int)(m / pq);
            const int rem = (int)(m - (int64_t)img * pq);
            const int pp = rem / p.cg.Q, qq = rem - pp * p.cg.Q;
            h0 = pp * p.cg.sh - p.cg.ph;
            w0 = qq * p.cg.sw - p.cg.pw;
        }
        float acc[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        for (int64_t k0 = 0; k0 < p.K; k0 += BK) {
            __syncthreads();                            // the previous chunk's fragments are read
            // ---- pack A: im2col gather (zero outside the image, past K and past M) ----
            for (int kk = akoff; kk < BK; kk += astep) {
                const int64_t k = k0 + kk;
                uint16_t v = 0;
                if (m < p.M && k < p.K) {
                    if (is_conv) {
                        const int rs = (int)(k / C), c = (int)(k - (int64_t)rs * C);
                        const int r = rs / S, s = rs - r * S;
                        const int h = h0 + r, w = w0 + s;
                        if (h >= 0 && h < p.cg.H && w >= 0 && w < p.cg.W)
                            v = __ldg(p.A + (((int64_t)img * p.cg.H + h) * p.cg.W + w) * C + c);
                    } else {
                        v = __ldg(p.A + m * p.lda + k);
                    }
                }
                As[arow * LDS + kk] = v;
            }
            // ---- pack B transposed: Bs[n][k] (k contiguous per column: the mma's col-major B) ----
            for (int i = tid; i < NT * 8 * BK; i += 256) {
                const int nn = i / BK, kk = i - nn * BK;
                const int64_t k = k0 + kk, n = n0 + nn;
                Bs[nn * LDS + kk] = (k < p.K && n < p.N) ? __ldg(p.B + k * p.ldb + n) : (uint16_t)0;
            }
            __syncthreads();
            if (warp * 16 < BM) {
#pragma unroll
                for (int kk = 0; kk < BK; kk += 16) {
                    // fragments of m16n8k16 (row.col): a0/a1 rows g / g+8 at k 2t.., a2/a3 at k 2t+8..
                    const int g = lane >> 2, tq = lane & 3;
                    const uint16_t* ar = As + (warp * 16 + g) * LDS + kk + 2 * tq;
                    uint32_t a[4];
                    a[0] = *reinterpret_cast<const uint32_t*>(ar);
                    a[1] = *reinterpret_cast<const uint32_t*>(ar + 8 * LDS);
                    a[2] = *reinterpret_cast<const uint32_t*>(ar + 8);
                    a[3] = *reinterpret_cast<const uint32_t*>(ar + 8 * LDS + 8);
#pragma unroll
                    for (int j = 0; j < NT; ++j) {
                        const uint16_t* br = Bs + (j * 8 + g) * LDS + kk + 2 * tq;
                        uint32_t b[2];
                        b[0] = *reinterpret_cast<const uint32_t*>(br);
                        b[1] = *reinterpret_cast<const uint32_t*>(br + 8);
                        mma_bf16_16816(acc[j], a, b);
                    }
                }
            }
        }
        // ---- epilogue: d0,d1 at (row g, cols 2t, 2t+1), d2,d3 at row g + 8 ----
        if (warp * 16 < BM) {
            const int g = lane >> 2, tq = lane & 3;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int64_t row = m0 + warp * 16 + g + (e >> 1) * 8;
                    const int64_t col = n0 + j * 8 + 2 * tq + (e & 1);
                    if (row >= p.M || col >= p.N) continue;
                    const int64_t off = row * p.ldc + col;
                    float v = acc[j][e];
                    if (p.cons) v = consume1(v, p.cons, p.bias, p.C, p.out_bf16 != 0, off, col);
                    if (p.out_bf16) reinterpret_cast<__nv_bfloat16*>(p.C)[off] = __float2bfloat16_rn(v);
                    else reinterpret_cast<float*>(p.C)[off] = v;
                }
        }
    }
}


// ---- pack at the tile level (pack_halo = 1/2, conv only): the patch-staged kernel ----
// A CTA tile = pg.tp whole output rows (p0 .. p0+tp) of image `img` x tile_n filters.  Its input
// patch (pg.pr input rows) is staged in SMEM once per tile -- by one 4-D TMA per tile into a double
// buffer (TMA: the raw NHWC rows, prefetched one tile ahead, zero fill = the padding), or by the
// threads into pixel slots of CP channels (PAD) -- and the filter slice transposed (Bs[n][k], k =
// (r, run element kl), tap t = kl - delta; padded positions carry zero weights).  Every 16-deep
// step (r, j) of pixel i then reads A from patch row (i / Q) * sh + r at element
// (i % Q) * pix_stride + off0 + 16 j: a contiguous 32-byte run, so the m16n8k16 A fragments are
// four 32-bit LDS per 16 pixels.  Each warp owns 32 pixels (two m16 blocks) and all tile_n
// filters; the epilogue applies the consumer, rounds once, stages the warp's 32 x tile_n block in
// SMEM and writes it with 16-byte stores.
// MODE: 0 = TMA raw rows; 4 / 8 / 16 = thread-filled slots of that many channels.
template <int NT, int MODE>
__global__ void __launch_bounds__(512) conv_mma_patch_kernel(const __grid_constant__ CUtensorMap tmX, const MmaParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr bool TMA = MODE == 0;
    constexpr int CP = TMA ? 4 : MODE;                 // (unused in TMA mode)
    const MmaPatch g = p.pg;
    uint8_t* const Bs = smem + g.nbuf * g.smem_patch;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int nthr = blockDim.x;
    const int os = p.out_bf16 ? 2 : 4;
    constexpr int tn = NT * 8;
    uint8_t* const Os = Bs + g.smem_b + warp * 32 * tn * os;
    uint64_t* const full = reinterpret_cast<uint64_t*>(Bs + g.smem_b + g.smem_out);
    const int H = p.cg.H, W = p.cg.W, C = p.cg.C, P = p.cg.P, Q = p.cg.Q, S = p.cg.S;
    const int tiles_p = (P + g.tp - 1) / g.tp;
    const uint32_t patch_tx = (uint32_t)(g.pr * g.rowpitch);
#define XTC_TILE_POS(t, img, p0, nb)                                   \
    do {                                                               \
        int mb_, ks_;                                                  \
        tile_coords(p.tm, (t), mb_, nb, ks_);                          \
        img = mb_ / tiles_p;                                           \
        p0 = (mb_ - img * tiles_p) * g.tp;                             \
    } while (0)
#define XTC_ISSUE_PATCH(t, buf)                                                                          \
    do {                                                                                                 \
        int img_, p0_, nb_;                                                                              \
        XTC_TILE_POS((t), img_, p0_, nb_);                                                               \
        ptx::mbar_arrive_expect_tx(&full[(buf)], patch_tx);                                              \
        ptx::tma_load_4d(&tmX, smem + (buf) * g.smem_patch, &full[(buf)], 0, g.x0 / 16,                  \
                         p0_ * p.cg.sh - p.cg.ph, img_);                                                 \
    } while (0)
    // k -> row (r*S + s)*C + c of the RSCF filter, -1 for the zero-weight padding of K
    int* const koff = reinterpret_cast<int*>(Bs + g.smem_b + g.smem_out + 16);
    for (int kk = tid; kk < g.kp; kk += nthr) {
        const int r = kk / g.kpr, tap = kk - r * g.kpr - g.delta;
        const int s = tap / g.bcp, c = tap - s * g.bcp;
        koff[kk] = (tap >= 0 && s < S && c < C) ? (r * S + s) * C + c : -1;
    }
    if (TMA && tid == 0) {
        ptx::prefetch_tmap(&tmX);
        ptx::mbar_init(&full[0], 1);
        ptx::mbar_init(&full[1], 1);
        ptx::fence_mbarrier_init();
    }
    __syncthreads();
    if (TMA && tid == 0 && (int64_t)blockIdx.x < p.num_tiles) XTC_ISSUE_PATCH((int64_t)blockIdx.x, 0);
    // tile-invariant operand offsets (bytes within a patch buffer / the filter slice) of this lane
    uint32_t a_off[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            int i = warp * 32 + b * 16 + hh * 8 + gq;
            if (i >= g.px) i = g.px - 1;             // rows past the tile compute a copy, never stored
            const int pp = i / Q, qq = i - pp * Q;
            a_off[b][hh] = (uint32_t)(pp * p.cg.sh * g.rowpitch + (qq * g.pix_stride + g.off0) * 2 + 4 * tq);
        }
    const uint32_t b_lane = ptx::smem_u32(Bs) + (gq * g.b_pitch + 2 * tq) * 2;
    int cur_nb = -1;
    int it = 0;
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        int img, p0, nb;
        XTC_TILE_POS(t, img, p0, nb);
        const int n0 = nb * tn;
        const int buf = TMA ? (it & 1) : 0;
        uint8_t* const patch = smem + buf * g.smem_patch;
        // the next tile's patch into the other buffer: its last reader (tile it-1) passed the
        // __syncthreads at the end of the previous iteration
        if (TMA && tid == 0 && t + gridDim.x < p.num_tiles) XTC_ISSUE_PATCH(t + gridDim.x, buf ^ 1);
        if (!TMA) {
            // ---- thread-filled patch: one CP-channel pixel slot per thread-iteration ----
            const int h_base = p0 * p.cg.sh - p.cg.ph;
            const int slots = g.pr * g.wpatch;
            for (int sl = tid; sl < slots; sl += nthr) {
                const int rr = sl / g.wpatch, ww = sl - rr * g.wpatch;
                const int h = h_base + rr, w = ww - p.cg.pw;
                uint16_t v[CP];
#pragma unroll
                for (int c = 0; c < CP; ++c) v[c] = 0;
                if (h >= 0 && h < H && w >= 0 && w < W) {
                    const uint16_t* src = p.A + (((int64_t)img * H + h) * W + w) * C;
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < C) v[c] = __ldg(src + c);
                }
                uint32_t* dst = reinterpret_cast<uint32_t*>(patch + (size_t)sl * CP * 2);
#pragma unroll
                for (int c = 0; c < CP; c += 2) dst[c / 2] = (uint32_t)v[c] | ((uint32_t)v[c + 1] << 16);
            }
        }
        const bool refill = nb != cur_nb;
        if (refill) {
            // ---- the filter slice transposed: Bs[n][k] (once per CTA when tiles_n == 1), through
            // the k -> filter-row table built once per CTA ----
            // 16 loads in flight per thread per batch (one L2 round trip for the stem's 3.6 K entries)
            const int total = tn * g.kp;
            for (int base = 0; base < total; base += 16 * nthr) {
                uint16_t v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int i = base + u * nthr + tid;
                    v[u] = 0;
                    if (i < total) {
                        const int ko = koff[i / tn];
                        const int64_t n = n0 + i % tn;
                        if (ko >= 0 && n < p.N) v[u] = __ldg(p.B + (int64_t)ko * p.ldb + n);
                    }
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int i = base + u * nthr + tid;
                    if (i < total) reinterpret_cast<uint16_t*>(Bs)[(i % tn) * g.b_pitch + i / tn] = v[u];
                }
            }
            cur_nb = nb;
        }
        if (!TMA || refill) __syncthreads();          // thread-filled patch / (re)filled filter visible
        if (TMA) ptx::mbar_wait(&full[buf], (uint32_t)((it >> 1) & 1));
        // ---- contraction: 2 m16 blocks x NT n8 blocks per warp ----
        float acc[2][NT][4];
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[b][j][0] = acc[b][j][1] = acc[b][j][2] = acc[b][j][3] = 0.f;
        // one flat loop over the R * ksr 16-deep steps; the fragments of step ks+1 are loaded before
        // the MMAs of step ks issue (register double buffer), so LDS latency overlaps the MMA chain
        const uint32_t pbase = ptx::smem_u32(patch);
        const int nks = p.cg.R * g.ksr;
        const uint32_t row_jump = (uint32_t)(g.rowpitch - g.ksr * 32 + 32);
        uint32_t ar = pbase, br = b_lane;
        int jj = 0;
        uint32_t fa[2][4], fb[NT][2];
        auto load_frags = [&](uint32_t (&xa)[2][4], uint32_t (&xb)[NT][2], uint32_t a_at, uint32_t b_at) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                xb[nt][0] = lds32(b_at + nt * 16 * g.b_pitch);
                xb[nt][1] = lds32(b_at + nt * 16 * g.b_pitch + 16);
            }
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                xa[b][0] = lds32(a_at + a_off[b][0]);
                xa[b][1] = lds32(a_at + a_off[b][1]);
                xa[b][2] = lds32(a_at + a_off[b][0] + 16);
                xa[b][3] = lds32(a_at + a_off[b][1] + 16);
            }
        };
        load_frags(fa, fb, ar, br);
#pragma unroll 1
        for (int ks = 0; ks < nks; ++ks) {
            // address of step ks+1 (the last iteration re-reads step ks: harmless)
            if (ks + 1 < nks) {
                ++jj;
                const bool wrap = jj == g.ksr;
                jj = wrap ? 0 : jj;
                ar += wrap ? row_jump : 32u;
                br += 32u;
            }
            uint32_t na[2][4], nbf[NT][2];
            load_frags(na, nbf, ar, br);
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) mma_bf16_16816(acc[b][nt], fa[b], fb[nt]);
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int q = 0; q < 4; ++q) fa[b][q] = na[b][q];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) { fb[nt][0] = nbf[nt][0]; fb[nt][1] = nbf[nt][1]; }
        }
        // ---- epilogue: consumer + one rounding, staged per warp, 16-byte stores ----
        const int rows_valid = min(g.tp, P - p0) * Q;             // pixels of this tile that exist
        const int64_t m_tile = ((int64_t)img * P + p0) * Q;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int il = b * 16 + hh * 8 + gq;          // row within the warp's 32
                    const int i = warp * 32 + il;
                    const int cl = nt * 8 + 2 * tq;
                    float v0 = acc[b][nt][hh * 2], v1 = acc[b][nt][hh * 2 + 1];
                    if (p.cons && i < rows_valid) {
                        const int64_t off = (m_tile + i) * p.ldc + n0 + cl;
                        if (n0 + cl < p.N) v0 = consume1(v0, p.cons, p.bias, p.C, p.out_bf16 != 0, off, n0 + cl);
                        if (n0 + cl + 1 < p.N) v1 = consume1(v1, p.cons, p.bias, p.C, p.out_bf16 != 0, off + 1, n0 + cl + 1);
                    }
                    if (p.out_bf16) {
                        const uint32_t w = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v0)) |
                                           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v1)) << 16);
                        *reinterpret_cast<uint32_t*>(Os + (il * tn + cl) * 2) = w;
                    } else {
                        *reinterpret_cast<float2*>(Os + (il * tn + cl) * 4) = make_float2(v0, v1);
                    }
                }
        __syncwarp();
        const int wrows = max(0, min(32, rows_valid - warp * 32));
        const int64_t m_w = m_tile + warp * 32;
        const int row_b = tn * os;                                 // staged bytes per row
        const bool vec = (n0 + tn <= p.N) && ((p.ldc * os) % 16 == 0) && ((n0 * os) % 16 == 0) &&
                         ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0);
        uint8_t* const Cb = static_cast<uint8_t*>(p.C);
        if (vec) {
            const int lv = __ffs(row_b / 16) - 1;                  // log2 of the 16-byte vectors per row
            for (int e = lane; e < (wrows << lv); e += 32) {
                const int rr = e >> lv, vv = e - (rr << lv);
                const uint4 w = *reinterpret_cast<const uint4*>(Os + rr * row_b + vv * 16);
                *reinterpret_cast<uint4*>(Cb + ((m_w + rr) * p.ldc + n0) * os + vv * 16) = w;
            }
        } else {
            for (int e = lane; e < wrows * tn; e += 32) {
                const int rr = e / tn, cc = e - rr * tn;
                if (n0 + cc >= p.N) continue;
                uint8_t* dst = Cb + ((m_w + rr) * p.ldc + n0 + cc) * os;
                if (os == 2) *reinterpret_cast<uint16_t*>(dst) = *reinterpret_cast<const uint16_t*>(Os + (rr * tn + cc) * 2);
                else *reinterpret_cast<float*>(dst) = *reinterpret_cast<const float*>(Os + (rr * tn + cc) * 4);
            }
        }
        __syncthreads();          // patch buffer, filter and staging free for the next tile
    }
}

#undef XTC_TILE_POS
#undef XTC_ISSUE_PATCH

template <int NT>
static cudaError_t launch_patch_nt(const CUtensorMap* tmX, const MmaParams& p, int grid, int block, int smem,
                                   cudaStream_t st) {
    auto k = p.pg.tma ? conv_mma_patch_kernel<NT, 0>
                      : (p.pg.cp == 4 ? conv_mma_patch_kernel<NT, 4>
                                      : (p.pg.cp == 8 ? conv_mma_patch_kernel<NT, 8> : conv_mma_patch_kernel<NT, 16>));
    cudaError_t e = ensure_smem_attr(k, smem);
    if (e != cudaSuccess) return e;
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof dummy);
    k<<<grid, block, smem, st>>>(tmX ? *tmX : dummy, p);
    return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_mma_nt(int tile_k, const MmaParams& p, int grid, cudaStream_t st) {
    switch (tile_k) {
        case 16: conv_mma_kernel<NT, 16><<<grid, 256, 0, st>>>(p); break;
        case 64: conv_mma_kernel<NT, 64><<<grid, 256, 0, st>>>(p); break;
        default: conv_mma_kernel<NT, 32><<<grid, 256, 0, st>>>(p); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_conv_mma(const void* A, const void* B, void* C, const Plan& pl, const xtc_op_desc& d,
                            const float* bias, int cons, const CUtensorMap* tmX, cudaStream_t st) {
    MmaParams p;
    memset(&p, 0, sizeof p);
    p.A = static_cast<const uint16_t*>(A);
    p.B = static_cast<const uint16_t*>(B);
    p.C = C;
    p.M = pl.M; p.N = pl.N; p.K = pl.K;
    const bool conv = d.kind == XTC_OP_CONV2D;
    p.lda = conv ? 0 : (d.lda ? d.lda : d.k);
    p.ldb = conv ? d.f : (d.ldb ? d.ldb : d.n);
    p.ldc = conv ? d.f : (d.ldc ? d.ldc : d.n);
    p.tile_m = pl.sch.tile_m; p.tile_n = pl.sch.tile_n; p.tile_k = pl.sch.tile_k;
    p.tm = TileMap{pl.tiles_m, pl.tiles_n, 1, pl.sch.order, pl.sch.raster_group};
    p.num_tiles = pl.num_tiles;
    p.out_bf16 = d.out_dtype == XTC_BF16;
    p.cons = cons;
    p.bias = bias;
    if (conv) {
        int64_t M_, N_, K_, P, Q;
        gemm_view(d, M_, N_, K_, P, Q);
        p.cg.is_conv = 1;
        p.cg.H = (int)d.h; p.cg.W = (int)d.w; p.cg.C = (int)d.c; p.cg.P = (int)P; p.cg.Q = (int)Q;
        p.cg.R = (int)d.r; p.cg.S = (int)d.s; p.cg.sh = (int)d.stride_h; p.cg.sw = (int)d.stride_w;
        p.cg.ph = (int)d.pad_h; p.cg.pw = (int)d.pad_w;
    }
    if (pl.mma_patch) {
        p.pg = pl.mp;
        p.batch = (int)d.batch;
        switch (pl.sch.tile_n) {
            case 16: return launch_patch_nt<2>(tmX, p, pl.grid_x, pl.block, pl.smem, st);
            case 32: return launch_patch_nt<4>(tmX, p, pl.grid_x, pl.block, pl.smem, st);
            default: return launch_patch_nt<8>(tmX, p, pl.grid_x, pl.block, pl.smem, st);
        }
    }
    switch (pl.sch.tile_n) {
        case 16: return launch_mma_nt<2>(p.tile_k, p, pl.grid_x, st);
        case 32: return launch_mma_nt<4>(p.tile_k, p, pl.grid_x, st);
        default: return launch_mma_nt<8>(p.tile_k, p, pl.grid_x, st);
    }
}

}  // namespace xtc
