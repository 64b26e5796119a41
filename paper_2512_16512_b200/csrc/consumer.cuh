// consumer.cuh -- the fused elementwise consumer (fuse) applied in the
// epilogues: v = relu(C_old + v + bias[col]) before the single rounding to the output
// type (include/xtc.h, xtc_consumer).  The unit is the epilogues' chunk: 32 consecutive
// columns of one output row, held by one thread (a TMEM lane / a SIMT register row).
#pragma once
#include <stdint.h>
#include "../../include/xtc.h"

namespace xtc {

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }

// C_old[row][col0 .. col0+ncols) as fp32 (read before the epilogue overwrites it)
__device__ __forceinline__ void load_row32(const void* C, bool bf16, int64_t off, int ncols, float (&o)[32]) {
    if (bf16) {
        const uint16_t* s = reinterpret_cast<const uint16_t*>(C) + off;
        if (ncols == 32 && (reinterpret_cast<uintptr_t>(s) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 w = reinterpret_cast<const uint4*>(s)[j];
                const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    o[8 * j + 2 * e] = bf16_bits_to_f32((uint16_t)(u[e] & 0xFFFFu));
                    o[8 * j + 2 * e + 1] = bf16_bits_to_f32((uint16_t)(u[e] >> 16));
                }
            }
        } else {
            #pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncols) o[j] = bf16_bits_to_f32(s[j]);
        }
    } else {
        const float* s = reinterpret_cast<const float*>(C) + off;
        if (ncols == 32 && (reinterpret_cast<uintptr_t>(s) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 w = reinterpret_cast<const float4*>(s)[j];
                o[4 * j] = w.x; o[4 * j + 1] = w.y; o[4 * j + 2] = w.z; o[4 * j + 3] = w.w;
            }
        } else {
            #pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncols) o[j] = s[j];
        }
    }
}

// One complete sum v of output element `off` (column col): relu(C_old + v + bias[col]), the
// same order as apply_consumer32 (used by the in-kernel split-K reduction).
__device__ __forceinline__ float consume1(float v, int cons, const float* bias, const void* C, bool out_bf16,
                                          int64_t off, int64_t col) {
    if (cons & XTC_CONSUMER_ACCUMULATE)
        v += out_bf16 ? bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(C)[off]) : reinterpret_cast<const float*>(C)[off];
    if (cons & XTC_CONSUMER_BIAS) v += __ldg(bias + col);
    if (cons & XTC_CONSUMER_RELU) v = fmaxf(v, 0.f);
    return v;
}

// v[j] (fp32 bits) for columns col0 + j, j < ncols, of output row `row`.  cons = XTC_CONSUMER_*
// bits; add_old / add_bias let atomic split-K drop the terms that are not its segment's.
__device__ __forceinline__ void apply_consumer32(uint32_t (&v)[32], int cons, const float* bias, const void* C,
                                                 bool out_bf16, int64_t row, int64_t ldc, int64_t col0, int ncols,
                                                 bool add_old = true, bool add_bias = true) {
    if ((cons & XTC_CONSUMER_ACCUMULATE) && add_old) {
        float o[32];
        load_row32(C, out_bf16, row * ldc + col0, ncols, o);
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < ncols) v[j] = __float_as_uint(__uint_as_float(v[j]) + o[j]);
    }
    if ((cons & XTC_CONSUMER_BIAS) && add_bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < ncols) v[j] = __float_as_uint(__uint_as_float(v[j]) + __ldg(bias + col0 + j));
    }
    if (cons & XTC_CONSUMER_RELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(fmaxf(__uint_as_float(v[j]), 0.f));
    }
}

}  // namespace xtc
