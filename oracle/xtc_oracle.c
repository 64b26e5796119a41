/*
 * xtc_oracle.c -- CPU oracle for the XTC B200 hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2512_16512_b200) never links, imports or calls it,
 * and this file shares no code, header or constant with the CUDA path.
 *
 * What it computes is the plain definition of the two operators, in fp64,
 * written as the paper's naive loop nest (Fig.2):
 *
 *     for (I) for (J) for (K)  C[I][J] += A[I][K] * B[K][J];
 *
 * with the readings of DESIGN.md §3:
 *   - C is overwritten (reading 1): the accumulator starts at 0.0.
 *   - row-major A[M][K], B[K][N], C[M][N] (reading 2).
 *   - accumulation in fp64 (BASELINE.json north_star; reading 6).  Products
 *     of two bf16 or two fp32 inputs are exact in fp64.
 *   - conv2d is the paper's padding(zero) -> conv2d graph (P:252, P:1152,
 *     reading 3) in NHWC x RSCF -> NPQF layout (reading 2), written as a
 *     direct loop with an explicit bounds test standing for the zero pad.
 *
 * Both functions also emit D = sum |a|*|b| over the same terms, the
 * normaliser of the tolerance "max |C - O| / D" (reading 7).
 *
 * Compiled with -O2 -fno-fast-math -ffp-contract=off (no FMA contraction, no
 * reassociation: the k loop runs strictly in ascending order) and OpenMP over
 * output rows; the order of the k sum is unaffected by threading.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* PAPER.md Fig.2: I, J, K loop nest, K innermost, ascending. */
void oracle_matmul_f64(int64_t M, int64_t N, int64_t K,
                       const double* A, const double* B,
                       double* C, double* D)
{
    int64_t i;
#pragma omp parallel for schedule(dynamic, 1)
    for (i = 0; i < M; i++) {
        for (int64_t j = 0; j < N; j++) {
            double s = 0.0, d = 0.0;
            for (int64_t k = 0; k < K; k++) {
                double a = A[i * K + k];
                double b = B[k * N + j];
                s += a * b;
                d += fabs(a) * fabs(b);
            }
            C[i * N + j] = s;
            if (D) D[i * N + j] = d;
        }
    }
}

/*
 * conv2d:
 *   y[n,p,q,f] = sum_{r,s,c} xpad[n, p*sh + r, q*sw + s, c] * w[r,s,c,f]
 * where xpad is x zero-padded by (ph, pw) on each side, i.e.
 *   xpad[n, h + ph, w + pw, c] = x[n,h,w,c] inside, 0 outside.
 * Output extent P = floor((H + 2ph - R)/sh) + 1, Q likewise (S:38 + pad).
 * Reduction order: r, s, c lexicographic (c fastest), ascending.
 */
void oracle_conv2d_f64(int64_t Nb, int64_t H, int64_t W, int64_t C, int64_t F,
                       int64_t R, int64_t S, int64_t sh, int64_t sw,
                       int64_t ph, int64_t pw,
                       const double* x, const double* w,
                       double* y, double* D)
{
    int64_t P = (H + 2 * ph - R) / sh + 1;
    int64_t Q = (W + 2 * pw - S) / sw + 1;
    int64_t np_;
#pragma omp parallel for schedule(dynamic, 1)
    for (np_ = 0; np_ < Nb * P; np_++) {
        int64_t n = np_ / P, p = np_ % P;
        for (int64_t q = 0; q < Q; q++) {
            for (int64_t f = 0; f < F; f++) {
                double acc = 0.0, d = 0.0;
                for (int64_t r = 0; r < R; r++) {
                    for (int64_t s = 0; s < S; s++) {
                        int64_t h = p * sh + r - ph;   /* position in unpadded x */
                        int64_t ww = q * sw + s - pw;
                        for (int64_t c = 0; c < C; c++) {
                            double xv = 0.0;           /* the padding op's zero fill */
                            if (h >= 0 && h < H && ww >= 0 && ww < W)
                                xv = x[((n * H + h) * W + ww) * C + c];
                            double wv = w[((r * S + s) * C + c) * F + f];
                            acc += xv * wv;
                            d += fabs(xv) * fabs(wv);
                        }
                    }
                }
                int64_t o = ((n * P + p) * Q + q) * F + f;
                y[o] = acc;
                if (D) D[o] = d;
            }
        }
    }
}

int oracle_num_threads(void)
{
    int t = 1;
#ifdef _OPENMP
#pragma omp parallel
    {
#pragma omp single
        t = omp_get_num_threads();
    }
#endif
    return t;
}
