/*
 * xtc.h -- C-ABI of the B200-native XTC hot path (libxtc.so).
 *
 * The paper's statement of the problem (PAPER.md, arXiv 2512.16512):
 *   - an operator from a fixed set (matmul, conv2d, ...) with a hyper-
 *     rectangular iteration space (§III-A, Fig.2);
 *   - a schedule built from the primitives of Table I:
 *     strip-mine, interchange, unroll, vectorize, parallelize, split,
 *     pack, bufferize (fuse is not on this path);
 *   - a compiled module conforming to "XTC's ABI: a function named after
 *     the graph and taking as parameters the graph's inputs and outputs,
 *     each passed as a contiguous raw pointer" (§IV-A);
 *   - an Executor that "validates that the optimized operator produces
 *     results consistent with the reference implementation" and an
 *     Evaluator that "generates input tensors, executes the compiled code,
 *     and collects performance metrics" (§IV-B).
 *
 * Here the four steps are: xtc_op_create (operator), xtc_schedule_apply
 * (schedule -> sm_100a launch plan), xtc_run (the compiled function) and
 * xtc_measure (Executor + Evaluator on the GPU).
 *
 * Conventions (all entry points):
 *   - Tensors are DEVICE pointers, row-major, contiguous unless a leading
 *     dimension is given.  The caller owns every tensor buffer and every
 *     stream; the library owns the xtc_op handle, its plan, its TMA
 *     descriptors, its split-K workspace and its cached validation
 *     reference.  Streams are passed as `void*` holding a cudaStream_t
 *     (NULL = the legacy default stream).
 *   - Argument order follows the paper's ABI: inputs, then outputs
 *     (P:757-761).  matmul: inputs {A[M][K], B[K][N]}, outputs {C[M][N]}.
 *     conv2d: inputs {x[N][H][W][C], w[R][S][C][F]}, outputs {y[N][P][Q][F]}.
 *   - Every call returns xtc_status; no C++ exception crosses the ABI and
 *     the library never aborts the process.  On any status other than
 *     XTC_OK a human-readable reason is available from xtc_last_error()
 *     (thread-local, valid until the next xtc_* call on the same thread).
 *   - XTC_E_ILLEGAL_SCHEDULE: nothing was launched and the op keeps its
 *     previous schedule.  XTC_E_CUDA: a CUDA error; sticky device errors
 *     leave the context unusable (the process must exit).
 *   - A handle is single-owner: do not drive one handle from two threads
 *     at once.  Distinct handles may be used concurrently.
 */
#ifndef XTC_H
#define XTC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XTC_ABI_VERSION 2

typedef enum {
    XTC_OK = 0,
    XTC_E_INVALID_ARG = 1,       /* malformed descriptor / null pointer / bad size      */
    XTC_E_UNSUPPORTED = 2,       /* well-formed but not implemented (dtype combination) */
    XTC_E_ILLEGAL_SCHEDULE = 3,  /* schedule violates a legality rule   */
    XTC_E_NO_SCHEDULE = 4,       /* xtc_run / xtc_measure before xtc_schedule_apply     */
    XTC_E_CUDA = 5,              /* CUDA runtime/driver error                           */
    XTC_E_VALIDATION_FAILED = 6, /* xtc_measure: cfg->validate == 2 and the check failed */
    XTC_E_OOM = 7                /* device allocation failed                            */
} xtc_status;

typedef enum { XTC_OP_MATMUL = 0, XTC_OP_CONV2D = 1 } xtc_op_kind;

/* Storage / arithmetic types.  XTC_TF32: fp32 storage, tf32 tensor-core math. */
typedef enum { XTC_F32 = 0, XTC_BF16 = 1, XTC_TF32 = 2 } xtc_dtype;

/* Operator descriptor (paper: O.tensor / O.mm / conv2d).
 *   matmul : C[m][n] = sum_k A[m][k] * B[k][n]      (C overwritten, reading 1)
 *            lda/ldb/ldc = row pitch in elements, 0 = packed (k, n, n).
 *   conv2d : y[b][p][q][f] = sum_{r,s,c} xpad[b][p*sh+r][q*sw+s][c] * w[r][s][c][f]
 *            xpad = x zero-padded by (pad_h, pad_w) (reading 3);
 *            p < P = (h + 2 pad_h - r)/stride_h + 1, q < Q likewise.
 *            Implicit GEMM view: M = batch*P*Q, N = f, K = r*s*c (c fastest).
 * in_dtype: F32 (SIMT engine, fp32 FFMA), TF32 or BF16 (tcgen05 engine).
 * out_dtype: F32 or BF16 (RNE).
 * consumer: elementwise consumer ops applied to the result (the paper's graph
 *   matmul -> relu, Fig.9; fuse), a bitmask of
 *     XTC_CONSUMER_RELU       out = max(v, 0)
 *     XTC_CONSUMER_BIAS       v += bias[n]  (bias = inputs[2]: fp32, one value per
 *                             output column n / output channel f, device memory)
 *     XTC_CONSUMER_ACCUMULATE v += C_old    (beta = 1: the output is also an input,
 *                             Fig.2's C[i][j] += ...; reading 1's NEXT flag)
 *   applied as out = round_out(relu(C_old + A*B + bias)), rounded once.  Whether
 *   they run fused into the contraction's epilogue (or split-K reduction) or as
 *   their own pass is the schedule's `fuse` knob (accumulate must be fused). */
typedef enum { XTC_CONSUMER_NONE = 0, XTC_CONSUMER_RELU = 1, XTC_CONSUMER_BIAS = 2,
               XTC_CONSUMER_ACCUMULATE = 4 } xtc_consumer;
typedef struct {
    int32_t kind;       /* xtc_op_kind */
    int32_t in_dtype;   /* xtc_dtype   */
    int32_t out_dtype;  /* xtc_dtype: XTC_F32 or XTC_BF16 */
    int32_t consumer;   /* xtc_consumer */
    int64_t m, n, k, lda, ldb, ldc;                         /* matmul */
    int64_t batch, h, w, c, f, r, s;                        /* conv2d */
    int64_t stride_h, stride_w, pad_h, pad_w;               /* conv2d */
} xtc_op_desc;

/* Engines (the instruction tier a schedule runs on):
 *   SIMT     fp32 FFMA register tiles (fp32 inputs)
 *   TCGEN05  tcgen05.mma, TMA-fed SMEM rings, TMEM accumulators (bf16 / tf32 / fp32 via 3xTF32)
 *   MMA      warp-level tensor-core tiles (mma.sync m16n8k16 bf16 -> fp32) fed by an im2col
 *            gather: conv2d / matmul whose operands TMA cannot address, e.g. the C = 3 stem conv
 *            (P:1084).  tile_m 64|128, tile_n 16|32|64, tile_k 16|32|64, split_k 1, buffer_c 0. */
typedef enum { XTC_ENGINE_SIMT = 0, XTC_ENGINE_TCGEN05 = 1, XTC_ENGINE_MMA = 2 } xtc_engine;
typedef enum { XTC_ORDER_MN = 0, XTC_ORDER_NM = 1 } xtc_order;
/* Reduction of the split K segments:
 *   ORDERED  fp32 partials in a workspace, summed in ascending segment order by a second kernel
 *   ATOMIC   fp32 atomics into C (fp32 output; exact on integer data only, order not fixed)
 *   CLUSTER  tcgen05: the split_k segments of an output tile are the CTAs of one thread-block
 *            cluster (split_k <= 16); after all partials are written each CTA sums 1/split_k of
 *            the tile's rows in ascending segment order inside the same kernel -- bit-identical
 *            to ORDERED, one launch, no second pass over the workspace.  Needs cluster_m 1,
 *            cluster_n 0/1, tile_m 128 (matmul), b_resident 0 (and buffer_c 0 for pack_halo).
 *   STREAM   tcgen05, persistent 1, split_k 0/1 ("stream-K"): the persistent grid of G CTAs splits
 *            the flattened (output tile, k-block) loop into G equal contiguous ranges, so the split
 *            points fall inside tiles wherever the tile count is not a multiple of G; a CTA whose
 *            range ends inside a tile adds, in ascending k order, the fp32 partials that the CTAs
 *            holding the rest of that tile wrote to the workspace (one launch, cooperative: all CTAs
 *            resident).  Matmul: cluster_m 1, tile_m 128, cluster_n 0/1; pack_halo: cluster_m 1. */
typedef enum { XTC_SPLITK_ORDERED = 0, XTC_SPLITK_ATOMIC = 1, XTC_SPLITK_CLUSTER = 2,
               XTC_SPLITK_STREAM = 3 } xtc_splitk_mode;

/* A schedule: Table I primitives as GPU loop-nest knobs.  The
 * mapping, value ranges and legality rules are in DESIGN.md §4 (SURVEY.md
 * §8(a) a2).  Unused knobs must be 0 (or 1 where noted); a knob value 0
 * means "default" only where stated.
 *
 * strip_mine   tile_m, tile_n, tile_k : CTA tile of the (M,N,K) loops; tcgen05: tile_m = 128 x
 *                                                   cluster_m (one UMMA row tile per CTA) or 256 x cluster_m
 *                                                   (matmul: two 128-row UMMA subtiles per CTA sharing every
 *                                                   B stage, two TMEM accumulators)
 *                          inner_m, inner_n       : SIMT thread register tile (TM x TN);
 *                                                   tcgen05: UMMA atom (inner_m = tile_m / cta_group,
 *                                                   inner_n = tile_n); 0 = derive
 * interchange  order                  : XTC_ORDER_MN: M-tile loop outer, N-tile loop inner
 *                          raster_group           : strip-mine the outer tile loop by this many tiles
 *                                                   and move the inner loop inside it (grouped raster)
 * unroll       unroll_k               : SIMT: k-loop unroll inside the SMEM tile (divides tile_k)
 *                                                   tcgen05: k-steps per stage, must be 0/1 (= fully unrolled)
 * vectorize    vector_n               : SIMT: 1 or 4 (float4 SMEM/global access along N); tcgen05: 0
 * parallelize  persistent             : 0 = one CTA per tile, 1 = #SM CTAs loop over tiles
 *                          grid_sms               : persistent only: the number of SMs ("cores") the
 *                                                   persistent grid spreads over, 0 = all of the device's;
 *                                                   e.g. SMs left free for a concurrent collective, or few
 *                                                   SMs so that every CTA strides over many tiles
 *                          cluster_m              : tcgen05: 1, or 2 = CTA pair (cta_group::2, tile_m = 256)
 *                          cluster_n              : tcgen05 matmul (cluster_m 1): 0/1, or 2 / 4 CTAs on adjacent
 *                                                   N tiles of one M tile form a cluster; each TMA-loads
 *                                                   1/cluster_n of the rows of every A stage and multicasts
 *                                                   it to all of them (A leaves L2 once per cluster);
 *                                                   needs tiles_n % cluster_n == 0, b_resident 0
 * split        split_k, split_k_mode  : K split into split_k contiguous segments + reduction
 *                          split_n_at             : 0, or the J split point s: [0,s) main root,
 *                                                   [s,N) remainder root on the SIMT engine (Fig.3/4)
 * pack         stages                 : SMEM ring depth (SIMT 1|2, tcgen05 2..8)
 *                          swizzle                : tcgen05: 128 (TMA/UMMA 128-byte swizzle);
 *                                                   SIMT: SMEM row padding in floats (0..8)
 *                          pack_warps             : tcgen05: warps issuing the TMA copies (1..3; 0 = 1);
 *                                                   warp w owns every pack_warps-th k-block of the ring
 *                          b_resident             : tcgen05: 1 = pack all of B once per CTA at the outermost
 *                                                   loop (needs a single N tile and split_k 1); the ring
 *                                                   then streams A only
 *                          pack_halo              : tcgen05 conv2d, stride 1: 1 = pack the input at the
 *                                                   output-tile level instead of per k-block -- one haloed
 *                                                   NHWC patch (tile rows + R-1 rows, Wp >= Q+S-1 pixel
 *                                                   slots) per tile, every filter tap (r, s) read as a
 *                                                   row-shifted view of it; tile_m = 128 or 256 virtual
 *                                                   rows (128/Wp output rows each), cluster_m 1, split_k 1;
 *                                                   2 = the same with compact rows: Wc = Q+S-1 slots per
 *                                                   row and tiles of consecutive virtual rows that may
 *                                                   start mid-row (one CTA per tile, no s-fold, no split,
 *                                                   buffer_c 0); the warp-MMA engine reads 1 / 2 as its
 *                                                   TMA-staged / thread-filled patch
 * bufferize    buffer_c             : 1 = SMEM-staged output + TMA store, 0 = direct stores
 *                          acc_buffers            : tcgen05 TMEM accumulator buffers (1|2)
 * fuse         fuse                   : 1 = the op's consumer (relu) is applied in the producer's
 *                                                   epilogue (or in the split-K reduction); 0 = it runs as a
 *                                                   separate elementwise pass over the output */
typedef struct {
    int32_t engine;
    int32_t tile_m, tile_n, tile_k;
    int32_t inner_m, inner_n;
    int32_t order, raster_group;
    int32_t unroll_k;
    int32_t vector_n;
    int32_t stages, swizzle;
    int32_t buffer_c, acc_buffers;
    int32_t split_k, split_k_mode;
    int32_t cluster_m;
    int32_t persistent;
    int32_t split_n_at;
    int32_t pack_warps;
    int32_t b_resident;
    int32_t fuse;
    int32_t pack_halo;
    int32_t cluster_n;
    int32_t grid_sms;
} xtc_schedule;

/* What the planner derived for a legal schedule (for reports and tests). */
typedef struct {
    int32_t engine;
    int32_t grid_x, grid_y, grid_z, block_x, cluster_x;
    int32_t smem_bytes;
    int32_t tmem_cols;
    int64_t num_tiles;          /* output tiles x split_k segments           */
    int64_t k_blocks_per_split;
    int64_t workspace_bytes;    /* split-K workspace                          */
    int32_t tail_grid_x, tail_grid_y; /* split_n_at remainder launch (0 if none) */
    int32_t reserved[4];
} xtc_plan_info;

/* Measurement configuration (Evaluator). */
typedef struct {
    int32_t warmup;       /* untimed launches before the timed ones (>= 0)            */
    int32_t repeats;      /* timed launches, each bracketed by its own CUDA events (>=1) */
    int32_t flush_l2;     /* 1: overwrite a 2 x L2-size scratch buffer before every rep  */
    int32_t validate;     /* 0: no; 1: validate, report; 2: validate, fail on mismatch   */
    int32_t exact;        /* 1: inputs are integer-valued -> require bit-exact output    */
    int32_t reuse_reference; /* 1: reuse the cached GPU reference if the input pointers
                                are unchanged (caller promises the data is unchanged)   */
    double tol;           /* max |C - R| / D allowed (<= 0: 1e-5 fp32, 5e-3 bf16/tf32)  */
    double peak_tflops;   /* denominator for frac_peak (0 = not reported)              */
    /* Hardware counters by human-readable name: NULL or a
     * comma-separated list of up to 8 Nsight-Compute metric names, each optionally
     * prefixed "gpu." (e.g. "gpu.dram__bytes_read.sum,gpu.sm__throughput.avg.pct_of_peak_sustained_elapsed").
     * Collected by the CUPTI range profiler in a separate replay pass AFTER the timed
     * reps (one range around one xtc_run), never inside the timed region. */
    const char* counters;
} xtc_measure_cfg;

/* Results of xtc_measure. */
typedef struct {
    int32_t status;        /* xtc_status of the measurement                          */
    int32_t valid;         /* 1 validated and within tolerance, 0 failed, -1 not run */
    double max_norm_err;   /* max_ij |C - R| / D   (D = sum_k |a||b|, fp64 on GPU)     */
    int64_t n_mismatch;    /* #elements whose bits differ from round_out(R)           */
    int64_t n_nan;         /* #NaN/Inf outputs (outputs are pre-filled with NaN)      */
    int64_t err_row, err_col; /* location of max_norm_err (output row-major [M][N])   */
    double t_min_ns, t_med_ns, t_mean_ns, t_max_ns;
    double tflops_med, tflops_min;   /* 2*M*N*K / t (FLOPs of the definition)     */
    double frac_peak;      /* tflops_med / cfg->peak_tflops                          */
    double sm_clock_mhz;   /* NVML SM clock sampled right after the timed window (0 if n/a) */
    int32_t n_reps;
    int32_t n_counters;    /* values in counters[] (in cfg->counters order); -1: CUPTI, the device
                              or a metric name unavailable -- the measurement itself is still
                              XTC_OK and xtc_last_error() says why */
    double counters[8];
} xtc_metrics;

typedef struct xtc_op_s* xtc_op;

/* a1 -- operator instantiation.  Validates the descriptor (shapes > 0, dtype
 * combination supported), binds it to CUDA device `device` and returns a new
 * handle in *out.  Nothing is launched.  Errors: INVALID_ARG, UNSUPPORTED. */
xtc_status xtc_op_create(const xtc_op_desc* desc, int32_t device, xtc_op* out);

/* Releases the handle and everything it owns (workspace, reference cache). */
void xtc_op_destroy(xtc_op op);

/* a2 -- pure host-side legality check + plan derivation for (desc, sch); needs
 * no GPU.  num_sms <= 0 means 148 (B200).  Returns XTC_OK and fills *info (may
 * be NULL), or XTC_E_ILLEGAL_SCHEDULE / XTC_E_INVALID_ARG with the violated
 * rule in xtc_last_error(). */
xtc_status xtc_schedule_check(const xtc_op_desc* desc, const xtc_schedule* sch,
                              int32_t num_sms, xtc_plan_info* info);

/* a2 -- apply a schedule to an op: check legality against the op's device,
 * select the kernel variant, size the grid / SMEM / TMEM, allocate the split-K
 * workspace.  On error the previous schedule stays in effect. */
xtc_status xtc_schedule_apply(xtc_op op, const xtc_schedule* sch);

/* Strategy.default_schedule(opt_level): a heuristic schedule for
 * the descriptor.  opt_level 0 = the plainest legal schedule (SIMT 8x8x8,
 * 1x1 inner); >= 2 = the engine's tuned default. */
xtc_status xtc_schedule_default(const xtc_op_desc* desc, int32_t opt_level, xtc_schedule* out);

/* a3..a7 -- run the scheduled operator once, asynchronously on `stream`.
 * inputs[0..1], outputs[0] as in the conventions above; inputs[2] = the fp32
 * bias (n or f values) when the consumer has XTC_CONSUMER_BIAS (NULL ->
 * XTC_E_INVALID_ARG).  With XTC_CONSUMER_ACCUMULATE, outputs[0] is read too.
 * The TMA descriptors are re-encoded only when a pointer differs from the
 * previous call. */
xtc_status xtc_run(xtc_op op, const void* const* inputs, void* const* outputs, void* stream);

/* a3..a7 + §8(e) -- xtc_run of one M-shard of a matmul whose all-gather is
 * fused into the epilogue (BASELINE config 5, "large matmul
 * ... sharded by M ... NCCL all-gather", where the gather is the exchange step
 * after the per-rank GEMM).  Every output tile staged in SMEM is written by TMA
 * to EACH of the n_dest destinations: dests[d] is a device pointer (local, or
 * a peer GPU's buffer mapped into this device's address space, e.g. CUDA IPC /
 * symmetric memory over NVLink) to a row-major [dest_rows][N] output (row pitch
 * desc.ldc if set, else N); this op's output row i lands at row row_offset + i
 * of every destination.  The caller owns every buffer and must order the
 * destinations' readers after this launch (a cross-device barrier for peers).
 * Requires: tcgen05 engine, matmul, buffer_c = 1, split_k = 1, no split_n_at
 * root, no separate consumer pass, no XTC_CONSUMER_ACCUMULATE, M a multiple of
 * the CTA tile rows (a ragged last tile would overwrite a neighbour's rows),
 * 1 <= n_dest <= 8, row_offset + M <= dest_rows, 16-byte aligned dests.
 * Violations -> XTC_E_INVALID_ARG / XTC_E_UNSUPPORTED, nothing launched. */
xtc_status xtc_run_gather(xtc_op op, const void* const* inputs, void* const* dests, int32_t n_dest,
                          int64_t row_offset, int64_t dest_rows, void* stream);

/* The same fused all-gather through ONE multicast destination (the NVLS form):
 * `dest` is an NVLink-SHARP multicast address (CUDA multicast object bound to every rank's
 * [dest_rows][N] buffer and mapped here, e.g. torch symmetric memory's multicast_ptr); the
 * epilogue reads each staged output tile back from SMEM and writes it with
 * multimem.st.global.v4 (16-byte vectors, whole 512-byte row segments per warp), and the
 * NVSwitch replicates every store to all ranks -- each GPU sends its shard once instead of
 * once per peer.  multimem = 0 writes the same vectors with ordinary st.global.v4 to a plain
 * device pointer (one destination; the single-GPU form of the same write-out path).
 * Row placement, requirements and ordering as xtc_run_gather, plus N (and the row pitch) a
 * multiple of 8 bf16 / 4 fp32 elements.  A multimem address on a device without multicast
 * support faults (the caller checks CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED). */
xtc_status xtc_run_multicast(xtc_op op, const void* const* inputs, void* dest, int64_t row_offset,
                             int64_t dest_rows, int32_t multimem, void* stream);

/* a8 + a9 -- Executor + Evaluator.  Synchronous.  Sequence:
 *   1. if cfg->validate: fill outputs with NaN, run once, compute (or reuse)
 *      the fp64 GPU reference R and D, compare -> max_norm_err, n_mismatch, n_nan;
 *      the reference includes the consumer (C_old + R + bias, relu; with
 *      ACCUMULATE the output is snapshotted instead of NaN-filled, and every
 *      timed run keeps accumulating into it);
 *   2. cfg->warmup untimed runs;
 *   3. cfg->repeats timed runs, each between two CUDA events on `stream`, with
 *      the L2 flush (if requested) outside the event window;
 *   4. min / median / mean / max, TFLOP/s, clock sample.
 * Returns XTC_E_VALIDATION_FAILED only when cfg->validate == 2 and the check
 * failed (metrics are still filled). */
xtc_status xtc_measure(xtc_op op, const void* const* inputs, void* const* outputs,
                       const xtc_measure_cfg* cfg, xtc_metrics* out, void* stream);

/* a10 -- measure a batch of candidate schedules on one op (the sweep's inner
 * loop without the GIL): for each i, apply cands[i] (illegal -> out[i].status =
 * XTC_E_ILLEGAL_SCHEDULE, nothing launched), then xtc_measure.  Returns XTC_OK
 * unless a CUDA error made the context unusable. */
xtc_status xtc_sweep(xtc_op op, const xtc_schedule* cands, int32_t n,
                     const void* const* inputs, void* const* outputs,
                     const xtc_measure_cfg* cfg, xtc_metrics* out, void* stream);

/* Seeded input generator (Evaluator "generates input tensors").
 * Fills count elements of dtype (F32/TF32: float, BF16: bf16) at device pointer
 * dst with element i = value(seed, first + i) of the counter-based generator
 * in DESIGN.md §3 (identical to seeded_inputs/__init__.py).  mode 0 =
 * uniform [-1,1), 1 = integers {-2..2}.  Asynchronous on stream. */
xtc_status xtc_fill(void* dst, int64_t count, int32_t dtype, uint64_t seed, int32_t mode,
                    int64_t first, void* stream);

/* 2*M*N*K (matmul) or 2*N*P*Q*F*R*S*C (conv2d): FLOPs of the definition. */
double xtc_op_flops(const xtc_op_desc* desc);

/* Algorithmic bytes: inputs read once + output written once. */
double xtc_op_min_bytes(const xtc_op_desc* desc);

/* Device-side counters of the last xtc_run/xtc_measure on this op: number of
 * kernels launched by the last xtc_run (main + split-K reduce + tail root). */
int32_t xtc_last_launch_count(xtc_op op);

/* Reason for the last non-OK status on this thread ("" if none). */
const char* xtc_last_error(void);

/* sizeof of the public structs, for binding self-checks:
 * [0]=xtc_op_desc [1]=xtc_schedule [2]=xtc_plan_info [3]=xtc_measure_cfg [4]=xtc_metrics */
void xtc_abi_sizes(int64_t* out5);

#ifdef __cplusplus
}
#endif
#endif /* XTC_H */
