// harness.cu -- on-chip validation and measurement kernels (a8, a9), plus the
// split-K reduction (a5), the split_n_at remainder root and the seeded filler.
//
//   KB5 splitk_reduce : C = sum_{s=0}^{S-1} W[s] in ascending s (deterministic)
//   KB6 ref_gemm/conv : R and D = sum |a||b| in fp64, one output per thread
//                       ("validates that the optimized operator produces results
//                       consistent with the reference implementation")
//   KB7 compare       : max |C-R|/D (+argmax), #bit mismatches vs round_out(R), #NaN/Inf
//   KB8 l2_flush      : overwrite a scratch buffer >= 2 x L2 between timed reps
//   KB9 fill          : counter-based generator, same definition as
//                       seeded_inputs/__init__.py, implemented independently here
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "xtc_internal.h"

namespace xtc {

// ------------------------------------------------------------------ fill --
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_kernel(void* dst, int64_t count, int bf16, uint64_t seed, int mode, int64_t first) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ull + (uint64_t)(first + i));
        float v;
        if (mode == 1) v = (float)((int)((h >> 32) % 5ull) - 2);
        else v = (float)((double)(h >> 40) * (1.0 / 8388608.0) - 1.0);
        if (bf16) static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
        else static_cast<float*>(dst)[i] = v;
    }
}

cudaError_t launch_fill(void* dst, int64_t count, int bf16, uint64_t seed, int mode, int64_t first, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    fill_kernel<<<(int)blocks, 256, 0, st>>>(dst, count, bf16, seed, mode, first);
    return cudaGetLastError();
}

// ---------------------------------------------------------- input loads --
__device__ __forceinline__ double ld_in(const void* p, int64_t i, int bf16) {
    if (bf16) return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
    return (double)static_cast<const float*>(p)[i];
}

// ------------------------------------------------------- fp64 reference --
// 32x32 output tile per 256-thread block, 4 outputs per thread, k staged in SMEM.
__global__ void __launch_bounds__(256) ref_gemm_f64_kernel(const void* A, const void* B, int bf16, int64_t M, int64_t N,
                                                           int64_t K, int64_t lda, int64_t ldb, double* R, double* D) {
    __shared__ double As[32][33];
    __shared__ double Bs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // ty 0..7
    const int64_t m0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
    double s[4] = {0, 0, 0, 0}, d[4] = {0, 0, 0, 0};
    for (int64_t k0 = 0; k0 < K; k0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            const int64_t m = m0 + r, k = k0 + tx;
            As[r][tx] = (m < M && k < K) ? ld_in(A, m * lda + k, bf16) : 0.0;
            const int64_t kb = k0 + r, n = n0 + tx;
            Bs[r][tx] = (kb < K && n < N) ? ld_in(B, kb * ldb + n, bf16) : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk) {
            const double b = Bs[kk][tx];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double a = As[ty + 8 * i][kk];
                s[i] = fma(a, b, s[i]);
                d[i] = fma(fabs(a), fabs(b), d[i]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = m0 + ty + 8 * i, n = n0 + tx;
        if (m < M && n < N) { R[m * N + n] = s[i]; D[m * N + n] = d[i]; }
    }
}

__global__ void ref_conv_f64_kernel(const void* x, const void* w, int bf16, ConvGeom g, int64_t Nb, int64_t F,
                                    double* R, double* D) {
    const int64_t total = Nb * g.P * g.Q * F;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = o % F;
        const int64_t pix = o / F;
        const int q = (int)(pix % g.Q);
        const int p = (int)((pix / g.Q) % g.P);
        const int64_t n = pix / ((int64_t)g.P * g.Q);
        double s = 0, d = 0;
        for (int r = 0; r < g.R; ++r) {
            const int h = p * g.sh + r - g.ph;
            if (h < 0 || h >= g.H) continue;
            for (int sx = 0; sx < g.S; ++sx) {
                const int ww = q * g.sw + sx - g.pw;
                if (ww < 0 || ww >= g.W) continue;
                const int64_t xb = ((n * g.H + h) * g.W + ww) * g.C;
                const int64_t wb = ((int64_t)(r * g.S + sx) * g.C) * F + f;
                for (int c = 0; c < g.C; ++c) {
                    const double a = ld_in(x, xb + c, bf16), b = ld_in(w, wb + (int64_t)c * F, bf16);
                    s = fma(a, b, s);
                    d = fma(fabs(a), fabs(b), d);
                }
            }
        }
        R[o] = s;
        D[o] = d;
    }
}

cudaError_t launch_ref_gemm(const void* A, const void* B, int bf16, int64_t M, int64_t N, int64_t K, int64_t lda,
                            int64_t ldb, double* R, double* D, cudaStream_t st) {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
    ref_gemm_f64_kernel<<<grid, 256, 0, st>>>(A, B, bf16, M, N, K, lda, ldb, R, D);
    return cudaGetLastError();
}

cudaError_t launch_ref_conv(const void* x, const void* w, int bf16, const ConvGeom& g, int64_t Nb, int64_t F,
                            double* R, double* D, cudaStream_t st) {
    ref_conv_f64_kernel<<<148 * 16, 256, 0, st>>>(x, w, bf16, g, Nb, F, R, D);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- compare --
struct CmpOut {
    unsigned long long n_mismatch, n_nan;
};

__global__ void compare_kernel(const void* C, int out_bf16, CmpConsumer cc, int64_t M, int64_t N, int64_t ldc,
                               const double* R, const double* D, double* blk_err, int64_t* blk_idx, CmpOut* out) {
    double best = -1.0;
    int64_t best_i = -1;
    unsigned long long mism = 0, nan = 0;
    const int64_t total = M * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / N, n = i - m * N;
        // the reference of the consumer op: relu(C_old + R + bias); the normaliser gains |C_old| + |bias|
        // (relu is 1-Lipschitz: |relu a - relu b| <= |a - b|)
        double r = R[i], d = D[i];
        if (cc.cons & XTC_CONSUMER_ACCUMULATE) {
            const int64_t o = m * ldc + n;
            const double old = out_bf16 ? (double)__bfloat162float(static_cast<const __nv_bfloat16*>(cc.c_old)[o])
                                        : (double)static_cast<const float*>(cc.c_old)[o];
            r += old;
            d += fabs(old);
        }
        if (cc.cons & XTC_CONSUMER_BIAS) {
            r += (double)cc.bias[n];
            d += fabs((double)cc.bias[n]);
        }
        if (cc.cons & XTC_CONSUMER_RELU) r = fmax(r, 0.0);
        double c;
        bool bits_ok;
        if (out_bf16) {
            const __nv_bfloat16 cv = static_cast<const __nv_bfloat16*>(C)[m * ldc + n];
            c = (double)__bfloat162float(cv);
            const __nv_bfloat16 rr = __float2bfloat16_rn(__double2float_rn(r));
            bits_ok = __bfloat16_as_ushort(cv) == __bfloat16_as_ushort(rr);
        } else {
            const float cv = static_cast<const float*>(C)[m * ldc + n];
            c = (double)cv;
            bits_ok = __float_as_uint(cv) == __float_as_uint(__double2float_rn(r));
        }
        double e;
        if (isnan(c) || isinf(c)) { ++nan; e = INFINITY; }
        else e = (d > 0) ? fabs(c - r) / d : (c == r ? 0.0 : INFINITY);
        if (!bits_ok) ++mism;
        if (e > best) { best = e; best_i = i; }
    }
    // block reduce (max with index; counts by atomics)
    __shared__ double se[256];
    __shared__ int64_t si[256];
    se[threadIdx.x] = best;
    si[threadIdx.x] = best_i;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double o = se[threadIdx.x + w];
            const int64_t oi = si[threadIdx.x + w];
            if (o > se[threadIdx.x] || (o == se[threadIdx.x] && oi >= 0 && (si[threadIdx.x] < 0 || oi < si[threadIdx.x]))) {
                se[threadIdx.x] = o;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { blk_err[blockIdx.x] = se[0]; blk_idx[blockIdx.x] = si[0]; }
    if (mism) atomicAdd(&out->n_mismatch, mism);
    if (nan) atomicAdd(&out->n_nan, nan);
}

cudaError_t launch_compare(const void* C, int out_bf16, const CmpConsumer& cc, int64_t M, int64_t N, int64_t ldc,
                           const double* R, const double* D, double* blk_err, int64_t* blk_idx, void* counts, int blocks,
                           cudaStream_t st) {
    compare_kernel<<<blocks, 256, 0, st>>>(C, out_bf16, cc, M, N, ldc, R, D, blk_err, blk_idx,
                                           static_cast<CmpOut*>(counts));
    return cudaGetLastError();
}

// Device-side end of the compare (used by the asynchronous sweep): one block reduces
// the per-block (max err, index) partials and the counters into `slot`
// {max_err, (double)index, (double)n_mismatch, (double)n_nan}, then clears the counters.
__global__ void compare_finalize_kernel(const double* blk_err, const int64_t* blk_idx, int blocks, CmpOut* counts,
                                        double* slot) {
    __shared__ double se[256];
    __shared__ int64_t si[256];
    double best = -1.0;
    int64_t bi = -1;
    for (int i = threadIdx.x; i < blocks; i += blockDim.x) {
        const double e = blk_err[i];
        const int64_t x = blk_idx[i];
        if (x >= 0 && (e > best || (e == best && (bi < 0 || x < bi)))) { best = e; bi = x; }
    }
    se[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double o = se[threadIdx.x + w];
            const int64_t oi = si[threadIdx.x + w];
            if (oi >= 0 && (o > se[threadIdx.x] || (o == se[threadIdx.x] && (si[threadIdx.x] < 0 || oi < si[threadIdx.x])))) {
                se[threadIdx.x] = o;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        slot[0] = se[0] < 0 ? 0.0 : se[0];
        slot[1] = (double)si[0];
        slot[2] = (double)counts->n_mismatch;
        slot[3] = (double)counts->n_nan;
        counts->n_mismatch = 0;
        counts->n_nan = 0;
    }
}

cudaError_t launch_compare_finalize(const double* blk_err, const int64_t* blk_idx, int blocks, void* counts,
                                    double* slot, cudaStream_t st) {
    compare_finalize_kernel<<<1, 256, 0, st>>>(blk_err, blk_idx, blocks, static_cast<CmpOut*>(counts), slot);
    return cudaGetLastError();
}

// The consumer (include/xtc.h xtc_consumer) on one complete sum v of output (m, col):
// relu(C_old + v + bias[col]).  The caller reads C_old from C before overwriting it.
__device__ __forceinline__ float consume(float v, int cons, const float* bias, const void* C, int out_bf16,
                                         int64_t off, int64_t col) {
    if (cons & XTC_CONSUMER_ACCUMULATE)
        v += out_bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(C)[off]) : static_cast<const float*>(C)[off];
    if (cons & XTC_CONSUMER_BIAS) v += bias[col];
    if (cons & XTC_CONSUMER_RELU) v = fmaxf(v, 0.f);
    return v;
}

// --------------------------------------------- unfused consumer (fuse = 0) --
// bias / relu as their own elementwise pass over the output (the paper's separate graph
// ops); one read + one write of C.  (Accumulate is never unfused: C would be gone.)
__global__ void consumer_pass_kernel(void* C, int out_bf16, int64_t M, int64_t N, int64_t ldc, int cons,
                                     const float* bias) {
    const int64_t total = M * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / N, n = i - m * N, o = m * ldc + n;
        if (out_bf16) {
            __nv_bfloat16* p = static_cast<__nv_bfloat16*>(C) + o;
            *p = __float2bfloat16_rn(consume(__bfloat162float(*p), cons, bias, C, out_bf16, o, n));
        } else {
            float* p = static_cast<float*>(C) + o;
            *p = consume(*p, cons, bias, C, out_bf16, o, n);
        }
    }
}

cudaError_t launch_consumer_pass(void* C, int out_bf16, int64_t M, int64_t N, int64_t ldc, int cons,
                                 const float* bias, cudaStream_t st) {
    int64_t blocks = (M * N + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    consumer_pass_kernel<<<(int)blocks, 256, 0, st>>>(C, out_bf16, M, N, ldc, cons & ~XTC_CONSUMER_ACCUMULATE, bias);
    return cudaGetLastError();
}

// --------------------------------------------------------------- L2 flush --
// Streams through a buffer >= 2 x L2 with loads, leaving L2 full of CLEAN lines
// of that buffer: the next kernel finds none of its data cached and pays no
// write-back of dirty flush lines (a store-based flush would bill the next
// kernel for evicting ~L2-size of dirty data).  The store is never taken; it
// only keeps the loads alive.
__global__ void flush_kernel(const uint4* __restrict__ buf, int64_t n16, uint32_t salt, uint32_t* sink) {
    uint32_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == salt + 0x9E3779B9u) sink[0] = acc;
}

// Device-side delay: keeps the stream busy while the host enqueues the timed
// reps, so per-rep CUDA events bracket GPU execution, not host submission.
__global__ void delay_kernel(uint64_t ns) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint64_t t = t0;
    while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}

// ------------------------------------------------- fault injection (tests) --
// kind 1: C[row][col] += 1 (a wrong value); 2: C[row][col] = NaN (an output the
// schedule "forgot" to write); 3: a 32x32 block at (row, col) zeroed (a dropped tile).
__global__ void fault_kernel(void* C, int out_bf16, int64_t M, int64_t N, int64_t ldc, int kind, int64_t row,
                             int64_t col) {
    const int64_t r = row + (kind == 3 ? threadIdx.x / 32 : 0);
    const int64_t c = col + (kind == 3 ? threadIdx.x % 32 : 0);
    if (kind != 3 && threadIdx.x) return;
    if (r >= M || c >= N) return;
    const int64_t i = r * ldc + c;
    if (out_bf16) {
        __nv_bfloat16* p = static_cast<__nv_bfloat16*>(C) + i;
        const float v = __bfloat162float(*p);
        *p = __float2bfloat16_rn(kind == 1 ? v + 1.0f : kind == 2 ? __int_as_float(0x7fc00000) : 0.0f);
    } else {
        float* p = static_cast<float*>(C) + i;
        *p = kind == 1 ? *p + 1.0f : kind == 2 ? __int_as_float(0x7fc00000) : 0.0f;
    }
}

cudaError_t launch_fault(void* C, int out_bf16, int64_t M, int64_t N, int64_t ldc, int kind, int64_t row, int64_t col,
                         cudaStream_t st) {
    fault_kernel<<<1, 1024, 0, st>>>(C, out_bf16, M, N, ldc, kind, row, col);
    return cudaGetLastError();
}

cudaError_t launch_delay(uint64_t ns, cudaStream_t st) {
    delay_kernel<<<1, 32, 0, st>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_flush(void* buf, int64_t bytes, uint32_t salt, cudaStream_t st) {
    if (const char* c = getenv("XTC_CARVEOUT")) {     // diagnostics (A/B): same carveout as the GEMM kernels
        static bool done = false;
        if (!done) { cudaFuncSetAttribute(flush_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(c)); done = true; }
    }
    // the last 16 bytes of the buffer serve as the (never written) sink
    flush_kernel<<<148 * 8, 512, 0, st>>>(static_cast<const uint4*>(buf), bytes / 16 - 1, salt,
                                          reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + bytes - 16));
    return cudaGetLastError();
}

// ----------------------------------------------------------- split-K reduce --
__global__ void splitk_reduce_kernel(const float* __restrict__ W, int S, int64_t M, int64_t N, int64_t ws_ld,
                                     void* C, int64_t ldc, int out_bf16, int cons, const float* bias) {
    const int64_t groups_per_row = (N + 3) / 4;
    const int64_t total = M * groups_per_row;
    const int64_t plane = M * ws_ld;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = g / groups_per_row;
        const int64_t n = (g - m * groups_per_row) * 4;
        const float4* src = reinterpret_cast<const float4*>(W + m * ws_ld + n);
        float4 acc = src[0];
        for (int s = 1; s < S; ++s) {                 // ascending s: deterministic order
            const float4 v = *reinterpret_cast<const float4*>(W + s * plane + m * ws_ld + n);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        float a[4] = {acc.x, acc.y, acc.z, acc.w};
        const int cnt = (int)((N - n) < 4 ? (N - n) : 4);
        if (cons)                                      // fused consumer on the complete sums
            for (int j = 0; j < cnt; ++j) a[j] = consume(a[j], cons, bias, C, out_bf16, m * ldc + n + j, n + j);
        for (int j = 0; j < cnt; ++j) {
            if (out_bf16) static_cast<__nv_bfloat16*>(C)[m * ldc + n + j] = __float2bfloat16_rn(a[j]);
            else static_cast<float*>(C)[m * ldc + n + j] = a[j];
        }
    }
}

cudaError_t launch_splitk_reduce(const float* W, int S, int64_t M, int64_t N, int64_t ws_ld, void* C, int64_t ldc,
                                 int out_bf16, int cons, const float* bias, cudaStream_t st) {
    int64_t total = M * ((N + 3) / 4);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    splitk_reduce_kernel<<<(int)blocks, 256, 0, st>>>(W, S, M, N, ws_ld, C, ldc, out_bf16, cons, bias);
    return cudaGetLastError();
}

// ---------------------------------------------- split_n_at remainder root --
// The paper's scalar remainder loop (Fig.3 lines 33-35): one output
// per thread, ascending k, fp32 FMA.
__global__ void tail_gemm_kernel(const void* A, const void* B, int bf16_in, void* C, int out_bf16, int cons,
                                 const float* bias,
                                 int64_t M, int64_t n0, int64_t ntail, int64_t K, int64_t lda, int64_t ldb,
                                 int64_t ldc) {
    const int64_t j = (int64_t)blockIdx.x * 16 + (threadIdx.x & 15);
    const int64_t i = (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
    if (i >= M || j >= ntail) return;
    const int64_t col = n0 + j;
    float s = 0.f;
    for (int64_t k = 0; k < K; ++k) {
        float a, b;
        if (bf16_in) {
            a = __bfloat162float(static_cast<const __nv_bfloat16*>(A)[i * lda + k]);
            b = __bfloat162float(static_cast<const __nv_bfloat16*>(B)[k * ldb + col]);
        } else {
            a = static_cast<const float*>(A)[i * lda + k];
            b = static_cast<const float*>(B)[k * ldb + col];
        }
        s = fmaf(a, b, s);
    }
    if (cons) s = consume(s, cons, bias, C, out_bf16, i * ldc + col, col);
    if (out_bf16) static_cast<__nv_bfloat16*>(C)[i * ldc + col] = __float2bfloat16_rn(s);
    else static_cast<float*>(C)[i * ldc + col] = s;
}

cudaError_t launch_tail_gemm(const void* A, const void* B, int bf16_in, void* C, int out_bf16, int cons,
                             const float* bias, int64_t M, int64_t n0, int64_t ntail, int64_t K, int64_t lda, int64_t ldb,
                             int64_t ldc, int gx, int gy, cudaStream_t st) {
    tail_gemm_kernel<<<dim3(gx, gy), 256, 0, st>>>(A, B, bf16_in, C, out_bf16, cons, bias, M, n0, ntail, K, lda, ldb,
                                                   ldc);
    return cudaGetLastError();
}

}  // namespace xtc
