// gemm_simt.cuh -- KB1/KB4: schedule-parametrised fp32 GEMM / implicit-GEMM conv2d
// on the CUDA cores (FFMA), the fp32 path (tolerance 1e-5).
//
// This is the GPU form of the paper's Fig.3 register-tiled kernel:
// each thread keeps a TM x TN register tile of C ("bufferize" in registers) and
// performs VBROADCAST(A) x VLOAD(B) -> VFMADD outer products over k, with the
// CUDA thread in place of the 8-wide SIMD vector.  Knobs:
//   strip_mine : CTA tile tile_m x tile_n x tile_k; thread tile TM x TN (templates)
//   interchange: tile order MN / NM + grouped raster (TileMap)
//   unroll     : U k-steps of the SMEM tile unrolled (template, divides tile_k)
//   vectorize  : VEC=4 -> thread's TN columns contiguous, float4 SMEM reads;
//                VEC=1 -> columns strided by the thread count (conflict-free scalar reads)
//   parallelize: one CTA per tile, or persistent grid-stride over tiles
//   split      : K segments (split_k) -> fp32 workspace or atomics
//   pack       : A and B k-tiles copied to SMEM (A transposed to k-major), padded by
//                `pad` floats per row against bank conflicts; stages=2
//                double-buffers the pack with cp.async (zero-fill for out-of-range)
// Per output the k sum runs in ascending order with fmaf, so for split_k = 1 the
// result is bit-identical for every (tile, thread-tile, order, unroll, vector) choice.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "xtc_internal.h"

namespace xtc {

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// A[m][k] of the GEMM view: the matrix itself, or the implicit im2col of x.
__device__ __forceinline__ const float* a_elem(const SimtParams& p, int64_t m, int64_t k, bool& valid) {
    const float* A = static_cast<const float*>(p.A);
    if (!p.cg.is_conv) return A + m * p.lda + k;
    const ConvGeom& g = p.cg;
    const int64_t pq = (int64_t)g.P * g.Q;
    const int64_t n = m / pq;
    const int64_t rem = m - n * pq;
    const int pp = (int)(rem / g.Q), qq = (int)(rem - (int64_t)pp * g.Q);
    const int rs = (int)(k / g.C), c = (int)(k - (int64_t)rs * g.C);
    const int r = rs / g.S, s = rs - r * g.S;
    const int h = pp * g.sh + r - g.ph, w = qq * g.sw + s - g.pw;
    if (h < 0 || h >= g.H || w < 0 || w >= g.W) { valid = false; return A; }
    return A + ((n * g.H + h) * g.W + w) * g.C + c;
}

template <int TM, int TN, int U, int VEC>
__global__ void __launch_bounds__(simt_max_threads(TM, TN), simt_min_blocks(TM, TN)) simt_gemm_kernel(const SimtParams p) {
    extern __shared__ __align__(16) float sm[];
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int BM = p.tile_m, BN = p.tile_n, BK = p.tile_k;
    const int lda_s = BM + p.pad, ldb_s = BN + p.pad;
    const int a_sz = ((BK * lda_s + 3) / 4) * 4, b_sz = ((BK * ldb_s + 3) / 4) * 4;
    const int tx_n = BN / TN;
    const int tx = tid % tx_n, ty = tid / tx_n;
    const float* Bg = static_cast<const float*>(p.B);

    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, ks;
        tile_coords(p.tm, t, mb, nb, ks);
        const int64_t m0 = (int64_t)mb * BM, n0 = (int64_t)nb * BN;
        const int64_t k_begin = (int64_t)ks * p.k_per_split;
        const int64_t k_end = min(p.K, k_begin + p.k_per_split);
        const int nk = (int)((k_end - k_begin + BK - 1) / BK);

        float acc[TM][TN];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

        auto load_tile = [&](int kt, float* As, float* Bs, bool async) {
            const int64_t k0 = k_begin + (int64_t)kt * BK;
            for (int e = tid; e < BM * BK; e += nthr) {
                const int i = e / BK, kk = e - i * BK;
                const int64_t m = m0 + i, k = k0 + kk;
                bool valid = (m < p.M) && (k < k_end);
                const float* src = valid ? a_elem(p, m, k, valid) : static_cast<const float*>(p.A);
                if (async) cp_async4(&As[kk * lda_s + i], src, valid);
                else As[kk * lda_s + i] = valid ? *src : 0.f;
            }
            for (int e = tid; e < BK * BN; e += nthr) {
                const int kk = e / BN, j = e - kk * BN;
                const int64_t k = k0 + kk, n = n0 + j;
                const bool valid = (k < k_end) && (n < p.N);
                const float* src = valid ? Bg + k * p.ldb + n : Bg;
                if (async) cp_async4(&Bs[kk * ldb_s + j], src, valid);
                else Bs[kk * ldb_s + j] = valid ? *src : 0.f;
            }
        };

        auto compute = [&](const float* As, const float* Bs) {
            for (int kk = 0; kk < BK; kk += U) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    float a[TM], b[TN];
                    const float* ar = As + (kk + u) * lda_s + ty * TM;
                    if constexpr (TM % 4 == 0) {
                        if (p.fast) {                       // lda_s % 4 == 0: 16-byte A fragment reads
#pragma unroll
                            for (int i = 0; i < TM / 4; ++i) {
                                const float4 v4 = *reinterpret_cast<const float4*>(ar + 4 * i);
                                a[4 * i] = v4.x; a[4 * i + 1] = v4.y; a[4 * i + 2] = v4.z; a[4 * i + 3] = v4.w;
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < TM; ++i) a[i] = ar[i];
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < TM; ++i) a[i] = ar[i];
                    }
                    const float* br = Bs + (kk + u) * ldb_s;
                    if constexpr (VEC == 4) {
#pragma unroll
                        for (int j = 0; j < TN / 4; ++j) {
                            const float4 v4 = *reinterpret_cast<const float4*>(br + tx * TN + 4 * j);
                            b[4 * j] = v4.x; b[4 * j + 1] = v4.y; b[4 * j + 2] = v4.z; b[4 * j + 3] = v4.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < TN; ++j) b[j] = br[tx + j * tx_n];
                    }
#pragma unroll
                    for (int i = 0; i < TM; ++i)
#pragma unroll
                        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
                }
            }
        };

        if (p.fast) {
            // Vectorised pack (aligned matmul): B k-rows by 16-byte cp.async (partial vectors
            // zero-filled via src-size), A by 16-byte register loads along K transposed into
            // As[k][m]; the next k-tile is fetched while the current one is computed.
            const float* Ag = static_cast<const float*>(p.A);
            const int vra = BK / 4, vrb = BN / 4;
            float4 ra[4];
            auto load_a_regs = [&](int kt) {
                const int64_t k0 = k_begin + (int64_t)kt * BK;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int v = tid + r * nthr;
                    ra[r] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (v < BM * vra) {
                        const int i = v / vra, kq = v - i * vra;
                        const int64_t m = m0 + i, k = k0 + 4 * kq;
                        if (m < p.M) {
                            const float* src = Ag + m * p.lda + k;
                            if (k + 3 < k_end) ra[r] = *reinterpret_cast<const float4*>(src);
                            else {
                                if (k < k_end) ra[r].x = src[0];
                                if (k + 1 < k_end) ra[r].y = src[1];
                                if (k + 2 < k_end) ra[r].z = src[2];
                            }
                        }
                    }
                }
            };
            auto store_a_regs = [&](float* As) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int v = tid + r * nthr;
                    if (v < BM * vra) {
                        const int i = v / vra, kq = v - i * vra;
                        float* d = As + (4 * kq) * lda_s + i;
                        d[0] = ra[r].x; d[lda_s] = ra[r].y; d[2 * lda_s] = ra[r].z; d[3 * lda_s] = ra[r].w;
                    }
                }
            };
            auto load_b_async = [&](int kt, float* Bs) {
                const int64_t k0 = k_begin + (int64_t)kt * BK;
                for (int v = tid; v < BK * vrb; v += nthr) {
                    const int kk = v / vrb, jq = v - kk * vrb;
                    const int64_t k = k0 + kk, n = n0 + 4 * jq;
                    int bytes = 0;
                    if (k < k_end && n < p.N) bytes = (int)(p.N - n >= 4 ? 16 : 4 * (p.N - n));
                    const float* src = bytes ? Bg + k * p.ldb + n : Bg;
                    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(Bs + kk * ldb_s + 4 * jq));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
                }
            };
            if (nk > 0) {
                load_b_async(0, sm + a_sz);
                cp_async_commit();
                load_a_regs(0);
                store_a_regs(sm);
                cp_async_wait<0>();
                __syncthreads();
            }
            for (int kt = 0; kt < nk; ++kt) {
                const int cur = (p.stages == 2) ? (kt & 1) : 0;
                float* As = sm + cur * (a_sz + b_sz);
                const bool more = kt + 1 < nk;
                if (p.stages == 2 && more) {
                    float* An = sm + (cur ^ 1) * (a_sz + b_sz);
                    load_b_async(kt + 1, An + a_sz);
                    cp_async_commit();
                    load_a_regs(kt + 1);
                    compute(As, As + a_sz);
                    store_a_regs(An);
                    cp_async_wait<0>();
                } else {
                    compute(As, As + a_sz);
                    if (more) {                           // single buffer: refill after everyone is done
                        __syncthreads();
                        load_b_async(kt + 1, As + a_sz);
                        cp_async_commit();
                        load_a_regs(kt + 1);
                        store_a_regs(As);
                        cp_async_wait<0>();
                    }
                }
                __syncthreads();
            }
        } else {
        if (p.stages == 2 && nk > 0) { load_tile(0, sm, sm + a_sz, true); cp_async_commit(); }
        for (int kt = 0; kt < nk; ++kt) {
            float* As;
            float* Bs;
            if (p.stages == 2) {
                const int cur = kt & 1;
                As = sm + cur * (a_sz + b_sz);
                Bs = As + a_sz;
                if (kt + 1 < nk) {
                    float* An = sm + (cur ^ 1) * (a_sz + b_sz);
                    load_tile(kt + 1, An, An + a_sz, true);
                    cp_async_commit();
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
            } else {
                As = sm;
                Bs = sm + a_sz;
                load_tile(kt, As, Bs, false);
            }
            __syncthreads();
            compute(As, Bs);
            __syncthreads();
        }
        }

#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t row = m0 + ty * TM + i;
            if (row >= p.M) continue;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int64_t col = n0 + (VEC == 4 ? tx * TN + j : tx + j * tx_n);
                if (col >= p.N) continue;
                float v = acc[i][j];
                if (p.cons) {                                  // fused consumer
                    const int64_t o = row * p.ldc + col;
                    if ((p.cons & XTC_CONSUMER_ACCUMULATE) && !p.atomic)   // atomics add onto C anyway
                        v += p.out_bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p.C)[o])
                                        : static_cast<const float*>(p.C)[o];
                    if ((p.cons & XTC_CONSUMER_BIAS) && (!p.atomic || ks == 0)) v += __ldg(p.bias + col);
                    if (p.cons & XTC_CONSUMER_RELU) v = fmaxf(v, 0.f);
                }
                if (p.split_out) p.Wk[((int64_t)ks * p.M + row) * p.ws_ld + col] = v;
                else if (p.atomic) atomicAdd(static_cast<float*>(p.C) + row * p.ldc + col, v);
                else if (p.out_bf16) static_cast<__nv_bfloat16*>(p.C)[row * p.ldc + col] = __float2bfloat16_rn(v);
                else static_cast<float*>(p.C)[row * p.ldc + col] = v;
            }
        }
    }
}

template <int TM, int TN, int U, int VEC>
static cudaError_t launch_simt_t(const SimtParams& p, int grid, int block, int smem, cudaStream_t st) {
    auto k = simt_gemm_kernel<TM, TN, U, VEC>;
    if (smem > 48 * 1024) {
        cudaError_t e = ensure_smem_attr(k, smem);
        if (e != cudaSuccess) return e;
    }
    k<<<grid, block, smem, st>>>(p);
    return cudaGetLastError();
}

template <int TM, int TN, int U>
static cudaError_t launch_simt_v(int vec, const SimtParams& p, int grid, int block, int smem, cudaStream_t st) {
    if constexpr (TN % 4 == 0) {
        if (vec == 4) return launch_simt_t<TM, TN, U, 4>(p, grid, block, smem, st);
    }
    return launch_simt_t<TM, TN, U, 1>(p, grid, block, smem, st);
}

template <int TM, int TN>
static cudaError_t launch_simt_u(int u, int vec, const SimtParams& p, int grid, int block, int smem, cudaStream_t st) {
    switch (u) {
        case 1: return launch_simt_v<TM, TN, 1>(vec, p, grid, block, smem, st);
        case 2: return launch_simt_v<TM, TN, 2>(vec, p, grid, block, smem, st);
        case 4: return launch_simt_v<TM, TN, 4>(vec, p, grid, block, smem, st);
        default: return launch_simt_v<TM, TN, 8>(vec, p, grid, block, smem, st);
    }
}

template <int TM>
cudaError_t launch_simt_n(int tn, int u, int vec, const SimtParams& p, int grid, int block, int smem, cudaStream_t st) {
    // a 16-wide register row (e.g. the paper's J1 = 16 vector tile, Fig.4) for thin thread tiles only
    if constexpr (TM <= 2) {
        if (tn == 16) return launch_simt_u<TM, 16>(u, vec, p, grid, block, smem, st);
    }
    switch (tn) {
        case 1: return launch_simt_u<TM, 1>(u, vec, p, grid, block, smem, st);
        case 2: return launch_simt_u<TM, 2>(u, vec, p, grid, block, smem, st);
        case 4: return launch_simt_u<TM, 4>(u, vec, p, grid, block, smem, st);
        default: return launch_simt_u<TM, 8>(u, vec, p, grid, block, smem, st);
    }
}

// explicit instantiations live in gemm_simt_tm{1,2,4,8}.cu (one thread-tile height per
// translation unit, so nvcc compiles the ~60 kernel variants in parallel)
#define XTC_SIMT_TM(TM)                                                                                   \
    template cudaError_t launch_simt_n<TM>(int, int, int, const SimtParams&, int, int, int, cudaStream_t);
#define XTC_SIMT_TM_EXTERN(TM) extern XTC_SIMT_TM(TM)

}  // namespace xtc
