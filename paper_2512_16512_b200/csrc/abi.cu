// abi.cu -- the C-ABI of include/xtc.h: op handles, schedule application,
// TMA descriptor encoding, run, Executor/Evaluator (measure) and sweep.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "xtc_internal.h"

namespace xtc {
cudaError_t launch_tc_gemm(bool tf32, bool conv, int cta_group, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                           const TcParams& p, int grid, int smem, cudaStream_t st);
cudaError_t launch_tc_conv_halo(bool tf32, const CUtensorMap& x, const CUtensorMap& b, const CUtensorMap& y,
                                const TcParams& p, int grid, int smem, cudaStream_t st);
cudaError_t launch_conv_mma(const void* A, const void* B, void* C, const Plan& pl, const xtc_op_desc& d,
                            const float* bias, int cons, const CUtensorMap* tmX, cudaStream_t st);
cudaError_t launch_simt_gemm(int tm, int tn, int u, int vec, const SimtParams& p, int grid, int block, int smem,
                             cudaStream_t st);
cudaError_t launch_fill(void* dst, int64_t count, int bf16, uint64_t seed, int mode, int64_t first, cudaStream_t st);
cudaError_t launch_ref_gemm(const void* A, const void* B, int bf16, int64_t M, int64_t N, int64_t K, int64_t lda,
                            int64_t ldb, double* R, double* D, cudaStream_t st);
cudaError_t launch_ref_conv(const void* x, const void* w, int bf16, const ConvGeom& g, int64_t Nb, int64_t F,
                            double* R, double* D, cudaStream_t st);
cudaError_t launch_compare(const void* C, int out_bf16, const CmpConsumer& cc, int64_t M, int64_t N, int64_t ldc,
                           const double* R, const double* D, double* blk_err, int64_t* blk_idx, void* counts, int blocks,
                           cudaStream_t st);
cudaError_t launch_consumer_pass(void* C, int out_bf16, int64_t M, int64_t N, int64_t ldc, int cons,
                                 const float* bias, cudaStream_t st);
cudaError_t launch_compare_finalize(const double* blk_err, const int64_t* blk_idx, int blocks, void* counts,
                                    double* slot, cudaStream_t st);
cudaError_t launch_flush(void* buf, int64_t bytes, uint32_t salt, cudaStream_t st);
cudaError_t launch_delay(uint64_t ns, cudaStream_t st);
cudaError_t launch_fault(void* C, int out_bf16, int64_t M, int64_t N, int64_t ldc, int kind, int64_t row, int64_t col,
                         cudaStream_t st);
cudaError_t launch_splitk_reduce(const float* W, int S, int64_t M, int64_t N, int64_t ws_ld, void* C, int64_t ldc,
                                 int out_bf16, int cons, const float* bias, cudaStream_t st);
cudaError_t launch_tail_gemm(const void* A, const void* B, int bf16_in, void* C, int out_bf16, int cons,
                             const float* bias, int64_t M, int64_t n0, int64_t ntail, int64_t K, int64_t lda, int64_t ldb,
                             int64_t ldc, int gx, int gy, cudaStream_t st);
}  // namespace xtc

using namespace xtc;

static thread_local std::string g_err;

namespace xtc {
cudaError_t ensure_smem_attr_impl(const void* kernel, int smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> set_bytes;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    int& have = set_bytes[{kernel, dev}];
    if (smem <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) have = smem;
    // diagnostics (A/B): XTC_CARVEOUT=<0..100> sets the preferred L1/SMEM carveout of the kernels
    if (e == cudaSuccess)
        if (const char* c = getenv("XTC_CARVEOUT"))
            e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(c));
    return e;
}
cudaError_t ensure_nonportable_cluster_impl(const void* kernel) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, bool> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    bool& d = done[{kernel, dev}];
    if (d) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) d = true;
    return e;
}
}  // namespace xtc

static xtc_status fail(xtc_status s, const std::string& why) {
    g_err = why;
    return s;
}
static xtc_status cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return XTC_E_CUDA;
}
#define CU_TRY(expr, where)                                  \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_fail(_e, where);  \
    } while (0)

// -------------------------------------------------- driver entry points --
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_encodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled g_encode_tiled = nullptr;
static PFN_encodeIm2col g_encode_im2col = nullptr;

static xtc_status load_driver_fns() {
    if (g_encode_tiled && g_encode_im2col) return XTC_OK;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CU_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode_tiled = reinterpret_cast<PFN_encodeTiled>(fn);
    fn = nullptr;
    CU_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(XTC_E_CUDA, "cuTensorMapEncodeIm2col unavailable");
    g_encode_im2col = reinterpret_cast<PFN_encodeIm2col>(fn);
    return XTC_OK;
}

// ------------------------------------------------------------- NVML clock --
typedef int (*PFN_nvmlInit)(void);
typedef int (*PFN_nvmlHandleByPci)(const char*, void**);
typedef int (*PFN_nvmlClock)(void*, int, unsigned int*);
static PFN_nvmlClock g_nvml_clock = nullptr;
static PFN_nvmlHandleByPci g_nvml_handle = nullptr;
static bool g_nvml_tried = false;

static double sm_clock_mhz(int device) {
    if (!g_nvml_tried) {
        g_nvml_tried = true;
        void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
        if (h) {
            auto init = reinterpret_cast<PFN_nvmlInit>(dlsym(h, "nvmlInit_v2"));
            g_nvml_handle = reinterpret_cast<PFN_nvmlHandleByPci>(dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2"));
            g_nvml_clock = reinterpret_cast<PFN_nvmlClock>(dlsym(h, "nvmlDeviceGetClockInfo"));
            if (!init || init() != 0) g_nvml_clock = nullptr;
        }
    }
    if (!g_nvml_clock || !g_nvml_handle) return 0.0;
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return 0.0;
    void* dev = nullptr;
    if (g_nvml_handle(bus, &dev) != 0) return 0.0;
    unsigned int mhz = 0;
    if (g_nvml_clock(dev, 1 /* NVML_CLOCK_SM */, &mhz) != 0) return 0.0;
    return (double)mhz;
}

// ------------------------------------------------------------- op handle --
struct xtc_op_s {
    xtc_op_desc d{};
    int device = 0;
    int num_sms = kNumSmsB200;
    bool has_plan = false;
    Plan plan;
    // per-op owned resources
    float* ws = nullptr;
    int64_t ws_bytes = 0;
    // TMA descriptors, bound to pointers
    alignas(64) CUtensorMap tmA, tmB, tmC;
    const void* bound[3] = {nullptr, nullptr, nullptr};
    bool maps_valid = false;
    bool a3d = false, b3d = false;   // tmA / tmB encoded as 3-D (one TMA per stage)
    // validation reference cache
    double* R = nullptr;
    double* D = nullptr;
    int64_t ref_elems = 0;
    const void* ref_inputs[2] = {nullptr, nullptr};
    bool ref_valid = false;
    double* blk_err = nullptr;
    int64_t* blk_idx = nullptr;
    void* counts = nullptr;
    // consumer inputs of the current call: the bias (inputs[2]) and, for accumulate-mode
    // validation, a snapshot of the output taken before the validated run
    const float* bias = nullptr;
    void* c_old = nullptr;
    int64_t c_old_bytes = 0;
    // timing
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> evs;
    int32_t last_launches = 0;
    // fault injection for harness tests (XTC_DEBUG_FAULT=kind, XTC_DEBUG_FAULT_AT=row,col):
    // 1 = perturb one output, 2 = leave one output unwritten (NaN), 3 = drop a 32x32 block (zeros)
    int fault = 0;
    int64_t fault_row = 0, fault_col = 0;
    // device trace (XTC_TRACE=path): per-launch %globaltimer stamps of the first CTAs,
    // appended to `path` as one JSON line per tcgen05 launch (synchronises; diagnostics only)
    std::string trace_path;
    uint64_t* trace_dev = nullptr;
    // xtc_run_gather: destination tensor maps (host copy + device copy the kernel reads),
    // bound to (dests, row count); re-encoded and re-uploaded only when these change
    alignas(64) CUtensorMap gmaps[8];
    void* gmaps_dev = nullptr;
    uint32_t* sk_flags = nullptr;   // stream-K publish flags (kSkMaxCtas x 4) and the launch epoch
    uint32_t sk_epoch = 0;
    const void* gbound[8] = {nullptr};
    int32_t n_gbound = 0;
    int64_t g_rows = 0;
};

static int dsize(int dt) { return dt == XTC_BF16 ? 2 : 4; }

static void* g_flush_buf[64] = {nullptr};
static int64_t g_flush_bytes[64] = {0};

static void release_op(xtc_op op) {
    if (!op) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(op->device);
    if (op->ws) cudaFree(op->ws);
    if (op->R) cudaFree(op->R);
    if (op->D) cudaFree(op->D);
    if (op->blk_err) cudaFree(op->blk_err);
    if (op->blk_idx) cudaFree(op->blk_idx);
    if (op->counts) cudaFree(op->counts);
    if (op->c_old) cudaFree(op->c_old);
    if (op->trace_dev) cudaFree(op->trace_dev);
    if (op->gmaps_dev) cudaFree(op->gmaps_dev);
    if (op->sk_flags) cudaFree(op->sk_flags);
    for (auto e : op->evs) cudaEventDestroy(e);
    cudaSetDevice(cur);
    delete op;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

extern "C" {

const char* xtc_last_error(void) { return g_err.c_str(); }

void xtc_abi_sizes(int64_t* out5) {
    if (!out5) return;
    out5[0] = sizeof(xtc_op_desc);
    out5[1] = sizeof(xtc_schedule);
    out5[2] = sizeof(xtc_plan_info);
    out5[3] = sizeof(xtc_measure_cfg);
    out5[4] = sizeof(xtc_metrics);
}

double xtc_op_flops(const xtc_op_desc* d) {
    if (!d) return 0.0;
    int64_t M, N, K, P, Q;
    gemm_view(*d, M, N, K, P, Q);
    return 2.0 * (double)M * (double)N * (double)K;
}

double xtc_op_min_bytes(const xtc_op_desc* d) {
    if (!d) return 0.0;
    const double si = dsize(d->in_dtype), so = dsize(d->out_dtype);
    if (d->kind == XTC_OP_CONV2D) {
        int64_t M, N, K, P, Q;
        gemm_view(*d, M, N, K, P, Q);
        return si * (double)(d->batch * d->h * d->w * d->c) + si * (double)(d->r * d->s * d->c * d->f) +
               so * (double)(d->batch * P * Q * d->f);
    }
    return si * (double)(d->m * d->k + d->k * d->n) + so * (double)(d->m * d->n);
}

xtc_status xtc_op_create(const xtc_op_desc* desc, int32_t device, xtc_op* out) {
    if (!desc || !out) return fail(XTC_E_INVALID_ARG, "null argument");
    *out = nullptr;
    std::string why;
    xtc_status st = check_desc(*desc, why);
    if (st != XTC_OK) return fail(st, why);
    int ndev = 0;
    CU_TRY(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(XTC_E_INVALID_ARG, "device index out of range");
    cudaDeviceProp prop;
    CU_TRY(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(XTC_E_UNSUPPORTED, std::string("libxtc is built for sm_100a (B200); device is ") + prop.name);
    xtc_op op = new xtc_op_s();
    op->d = *desc;
    op->device = device;
    op->num_sms = prop.multiProcessorCount;
    if (const char* tp = getenv("XTC_TRACE")) op->trace_path = tp;
    if (const char* f = getenv("XTC_DEBUG_FAULT")) {
        op->fault = atoi(f);
        if (const char* at = getenv("XTC_DEBUG_FAULT_AT")) {
            long long r = 0, c = 0;
            if (sscanf(at, "%lld,%lld", &r, &c) == 2) { op->fault_row = r; op->fault_col = c; }
        }
    }
    *out = op;
    return XTC_OK;
}

void xtc_op_destroy(xtc_op op) { release_op(op); }

int32_t xtc_last_launch_count(xtc_op op) { return op ? op->last_launches : 0; }

xtc_status xtc_schedule_check(const xtc_op_desc* desc, const xtc_schedule* sch, int32_t num_sms, xtc_plan_info* info) {
    if (!desc || !sch) return fail(XTC_E_INVALID_ARG, "null argument");
    Plan p;
    std::string why;
    xtc_status st = make_plan(*desc, *sch, num_sms, p, why);
    if (st != XTC_OK) return fail(st, why);
    if (info) {
        memset(info, 0, sizeof *info);
        info->engine = p.engine;
        info->grid_x = p.grid_x;
        info->grid_y = p.grid_y;
        info->grid_z = p.grid_z;
        info->block_x = p.block;
        info->cluster_x = p.cluster;
        info->smem_bytes = p.smem;
        info->tmem_cols = p.tmem_cols;
        info->num_tiles = p.num_tiles;
        info->k_blocks_per_split = p.engine == XTC_ENGINE_TCGEN05 ? p.kb_per_split : p.k_per_split / std::max(1, sch->tile_k);
        info->workspace_bytes = p.workspace_bytes;
        info->tail_grid_x = p.tail_grid_x;
        info->tail_grid_y = p.tail_grid_y;
    }
    return XTC_OK;
}

xtc_status xtc_schedule_apply(xtc_op op, const xtc_schedule* sch) {
    if (!op || !sch) return fail(XTC_E_INVALID_ARG, "null argument");
    Plan p;
    std::string why;
    xtc_status st = make_plan(op->d, *sch, op->num_sms, p, why);
    if (st != XTC_OK) return fail(st, why);
    DeviceGuard g(op->device);
    if (p.workspace_bytes > op->ws_bytes) {
        if (op->ws) cudaFree(op->ws);
        op->ws = nullptr;
        op->ws_bytes = 0;
        if (cudaMalloc(&op->ws, p.workspace_bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(XTC_E_OOM, "split-K workspace allocation failed");
        }
        op->ws_bytes = p.workspace_bytes;
    }
    op->plan = p;
    op->has_plan = true;
    op->maps_valid = false;
    return XTC_OK;
}

xtc_status xtc_schedule_default(const xtc_op_desc* d, int32_t opt_level, xtc_schedule* out) {
    if (!d || !out) return fail(XTC_E_INVALID_ARG, "null argument");
    std::string why;
    xtc_status st = check_desc(*d, why);
    if (st != XTC_OK) return fail(st, why);
    xtc_schedule s;
    memset(&s, 0, sizeof s);
    int64_t M, N, K, P, Q;
    gemm_view(*d, M, N, K, P, Q);
    if (d->in_dtype == XTC_F32 || opt_level <= 0) {
        s.engine = XTC_ENGINE_SIMT;
        if (opt_level <= 0 || d->in_dtype != XTC_F32) {
            if (d->in_dtype != XTC_F32) return fail(XTC_E_UNSUPPORTED, "opt_level 0 (SIMT) needs fp32 inputs");
            s.tile_m = s.tile_n = s.tile_k = 8;
            s.inner_m = s.inner_n = 1;
            s.unroll_k = 1;
            s.stages = 1;
        } else {
            s.tile_m = 64; s.tile_n = 64; s.tile_k = 16;
            s.inner_m = 4; s.inner_n = 4;
            s.unroll_k = 4; s.vector_n = 4; s.stages = 2; s.swizzle = 4;
            s.raster_group = 8;
        }
        s.split_k = 1;
        *out = s;
        return XTC_OK;
    }
    // tcgen05 default: 128 x N tile, deepest ring that fits, persistent + double-buffered TMEM
    const int es = dsize(d->in_dtype);
    const int atom = 128 / es;
    s.engine = XTC_ENGINE_TCGEN05;
    s.tile_m = 128;
    s.tile_n = N >= 256 ? 256 : (N >= 128 ? 128 : atom * (int)std::max<int64_t>(1, (N + atom - 1) / atom));
    if (s.tile_n > 256) s.tile_n = 256;
    s.tile_k = atom;
    s.swizzle = 128;
    s.buffer_c = 1;
    s.acc_buffers = s.tile_n <= 256 ? 2 : 1;
    if (2 * s.tile_n > 512) s.acc_buffers = 1;
    s.persistent = 1;
    s.raster_group = 8;
    s.split_k = 1;
    const int stage = 128 * s.tile_k * es + s.tile_k * s.tile_n * es;
    int stages = (kSmemMaxOptin - kTcEpiSmem - kSmemReserve) / stage;
    s.stages = std::max(2, std::min(8, stages));
    // low-parallelism shapes: split K so the grid covers the SMs (a5)
    const int64_t tiles = ((M + 127) / 128) * ((N + s.tile_n - 1) / s.tile_n);
    const int64_t kb = (K + s.tile_k - 1) / s.tile_k;
    int sk = 1;
    while (tiles * sk * 2 <= kNumSmsB200 && kb / (sk * 2) >= 4) sk *= 2;
    s.split_k = sk;
    Plan p;
    if (make_plan(*d, s, kNumSmsB200, p, why) != XTC_OK) {
        s.split_k = 1;
        if (make_plan(*d, s, kNumSmsB200, p, why) != XTC_OK) return fail(XTC_E_ILLEGAL_SCHEDULE, "default: " + why);
    }
    *out = s;
    return XTC_OK;
}

xtc_status xtc_fill(void* dst, int64_t count, int32_t dtype, uint64_t seed, int32_t mode, int64_t first, void* stream) {
    if (!dst && count > 0) return fail(XTC_E_INVALID_ARG, "null dst");
    if (mode != 0 && mode != 1) return fail(XTC_E_INVALID_ARG, "mode must be 0 (uniform) or 1 (int)");
    CU_TRY(launch_fill(dst, count, dtype == XTC_BF16, seed, mode, first, (cudaStream_t)stream), "fill");
    return XTC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------- run --
static xtc_status encode_maps(xtc_op op, const void* A, const void* B, void* C) {
    const Plan& p = op->plan;
    const xtc_op_desc& d = op->d;
    xtc_status st = load_driver_fns();
    if (st != XTC_OK) return st;
    const bool tf32 = d.in_dtype == XTC_TF32 || p.split3;     // fp32 storage (tf32 or the 3xTF32 split)
    const CUtensorMapDataType in_t = tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int es = dsize(d.in_dtype);
    const int atom = 128 / es;
    const int tile_k = p.sch.tile_k, tile_n = p.sch.tile_n;
    CUresult r;
    const bool allow3d = getenv("XTC_NO_3D_TMA") == nullptr;
    // B: [K][N] row-major, N-major UMMA operand.  3-D view {atom, K, N/atom} (strides ldb, 128 B):
    // one box {atom, tile_k, bn_cta/atom} per stage lands as [n-block][k][128 B].  Only when N is a
    // multiple of the atom (else the last block would read into the next row instead of zero-filling).
    {
        const int64_t ldb = (d.kind == XTC_OP_MATMUL && d.ldb) ? d.ldb : p.n_total;
        // tf32 MN-major operands must use 32-byte swizzle atoms (UMMA SWIZZLE_128B_BASE32B)
        const CUtensorMapSwizzle bsw = tf32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
        op->b3d = false;
        if (p.halo && p.halo_b64) {
            // the CTA pair's 64-byte filter halves: box {32 columns, tile_k rows}, 64-byte swizzle
            cuuint64_t dims[2] = {(cuuint64_t)p.N, (cuuint64_t)p.K};
            cuuint64_t strides[1] = {(cuuint64_t)(ldb * es)};
            cuuint32_t box[2] = {(cuuint32_t)(atom / 2), (cuuint32_t)tile_k};
            cuuint32_t estr[2] = {1, 1};
            r = g_encode_tiled(&op->tmB, in_t, 2, const_cast<void*>(B), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(B, 64-byte halves) failed: " + std::to_string((int)r));
        } else if (allow3d && p.N % atom == 0) {
            cuuint64_t dims[3] = {(cuuint64_t)atom, (cuuint64_t)p.K, (cuuint64_t)(p.N / atom)};
            cuuint64_t strides[2] = {(cuuint64_t)(ldb * es), (cuuint64_t)(atom * es)};
            // each CTA of a pair (or of a halo multicast cluster) loads its share of the N blocks
            const int b_share = p.halo ? p.halo_cl : p.cta_group;
            cuuint32_t box[3] = {(cuuint32_t)atom, (cuuint32_t)tile_k, (cuuint32_t)(tile_n / b_share / atom)};
            cuuint32_t estr[3] = {1, 1, 1};
            r = g_encode_tiled(&op->tmB, in_t, 3, const_cast<void*>(B), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, bsw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            op->b3d = (r == CUDA_SUCCESS);
        }
        if (!op->b3d && !(p.halo && p.halo_b64)) {
            cuuint64_t dims[2] = {(cuuint64_t)p.N, (cuuint64_t)p.K};
            cuuint64_t strides[1] = {(cuuint64_t)(ldb * es)};
            cuuint32_t box[2] = {(cuuint32_t)atom, (cuuint32_t)tile_k};
            cuuint32_t estr[2] = {1, 1};
            r = g_encode_tiled(&op->tmB, in_t, 2, const_cast<void*>(B), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, bsw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(B) failed: " + std::to_string((int)r));
        }
    }
    op->a3d = false;
    if (d.kind == XTC_OP_MATMUL) {
        // A: [M][K] K-major.  3-D view {atom, M, K/atom} (strides lda, 128 B): one box
        // {atom, 128, tile_k/atom} per stage lands as [k-atom][row][128 B] (needs K % atom == 0).
        const int64_t lda = d.lda ? d.lda : d.k;
        // cluster_n: each CTA loads a 128/cluster_n-row slice of every A atom (2-D boxes)
        const int a_rows = p.cluster_n > 1 ? 128 / p.cluster_n : 128 * p.msub;
        if (allow3d && p.K % atom == 0 && p.cluster_n <= 1) {
            cuuint64_t dims[3] = {(cuuint64_t)atom, (cuuint64_t)p.M, (cuuint64_t)(p.K / atom)};
            cuuint64_t strides[2] = {(cuuint64_t)(lda * es), (cuuint64_t)(atom * es)};
            cuuint32_t box[3] = {(cuuint32_t)atom, (cuuint32_t)a_rows, (cuuint32_t)(tile_k / atom)};
            cuuint32_t estr[3] = {1, 1, 1};
            r = g_encode_tiled(&op->tmA, in_t, 3, const_cast<void*>(A), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            op->a3d = (r == CUDA_SUCCESS);
        }
        if (!op->a3d) {
            cuuint64_t dims[2] = {(cuuint64_t)p.K, (cuuint64_t)p.M};
            cuuint64_t strides[1] = {(cuuint64_t)(lda * es)};
            cuuint32_t box[2] = {(cuuint32_t)atom, (cuuint32_t)a_rows};
            cuuint32_t estr[2] = {1, 1};
            r = g_encode_tiled(&op->tmA, in_t, 2, const_cast<void*>(A), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(A) failed: " + std::to_string((int)r));
        }
    } else if (p.halo) {
        // x: NHWC, tiled 4-D {C, W, H, N}; box {atom channels, Wp slots, patch rows, 1} = one
        // channel plane of the haloed patch, [row][slot][128 B] in SMEM
        cuuint64_t dims[4] = {(cuuint64_t)d.c, (cuuint64_t)d.w, (cuuint64_t)d.h, (cuuint64_t)d.batch};
        cuuint64_t strides[3] = {(cuuint64_t)(d.c * es), (cuuint64_t)(d.w * d.c * es), (cuuint64_t)(d.h * d.w * d.c * es)};
        cuuint32_t box[4] = {(cuuint32_t)atom, (cuuint32_t)p.halo_wp, (cuuint32_t)p.halo_pr, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        r = g_encode_tiled(&op->tmA, in_t, 4, const_cast<void*>(A), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(x patch) failed: " + std::to_string((int)r));
    } else {
        // x: NHWC, im2col: one pixel = `atom` channels (128 B), 128 pixels per column
        cuuint64_t dims[4] = {(cuuint64_t)d.c, (cuuint64_t)d.w, (cuuint64_t)d.h, (cuuint64_t)d.batch};
        cuuint64_t strides[3] = {(cuuint64_t)(d.c * es), (cuuint64_t)(d.w * d.c * es), (cuuint64_t)(d.h * d.w * d.c * es)};
        int lower[2] = {(int)-d.pad_w, (int)-d.pad_h};                                   // {W, H}
        int upper[2] = {(int)(d.pad_w - (d.s - 1)), (int)(d.pad_h - (d.r - 1))};
        cuuint32_t estr[4] = {1, (cuuint32_t)d.stride_w, (cuuint32_t)d.stride_h, 1};
        r = g_encode_im2col(&op->tmA, in_t, 4, const_cast<void*>(A), dims, strides, lower, upper, (cuuint32_t)atom, 128,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeIm2col(x) failed: " + std::to_string((int)r));
    }
    // C (or the split-K workspace): 3-D {N, M, S} so stores clip per segment; box {128 B, 32 rows, 1}
    if (p.sch.buffer_c && p.halo) {
        // y: NPQF as 4-D {F, Q, P, N}; one epilogue warp's 32 virtual rows = box {128 B, min(Wp,32)
        // slots, max(1,32/Wp) rows, 1}; slots q >= Q and rows p >= P are clipped
        int64_t M_, N_, K_, P, Q;
        gemm_view(d, M_, N_, K_, P, Q);
        const int os = dsize(d.out_dtype);
        const CUtensorMapDataType out_t = os == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t dims[4] = {(cuuint64_t)d.f, (cuuint64_t)Q, (cuuint64_t)P, (cuuint64_t)d.batch};
        cuuint64_t strides[3] = {(cuuint64_t)(d.f * os), (cuuint64_t)(Q * d.f * os), (cuuint64_t)(P * Q * d.f * os)};
        const int wq = p.halo_wp < 32 ? p.halo_wp : 32;
        cuuint32_t box[4] = {(cuuint32_t)(128 / os), (cuuint32_t)wq, (cuuint32_t)(32 / wq), 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        r = g_encode_tiled(&op->tmC, out_t, 4, C, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(y) failed: " + std::to_string((int)r));
    } else if (p.sch.buffer_c) {
        const bool to_ws = p.split_k > 1;
        const int os = to_ws ? 4 : dsize(d.out_dtype);
        const CUtensorMapDataType out_t = os == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        const int64_t ld = to_ws ? p.ws_ld : ((d.kind == XTC_OP_MATMUL && d.ldc) ? d.ldc : p.n_total);
        void* base = to_ws ? (void*)op->ws : C;
        cuuint64_t dims[3] = {(cuuint64_t)p.N, (cuuint64_t)p.M, (cuuint64_t)(to_ws ? p.split_k : 1)};
        cuuint64_t strides[2] = {(cuuint64_t)(ld * os), (cuuint64_t)(ld * os * p.M)};
        cuuint32_t box[3] = {(cuuint32_t)(128 / os), 32, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        r = g_encode_tiled(&op->tmC, out_t, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(C) failed: " + std::to_string((int)r));
    } else {
        memset(&op->tmC, 0, sizeof op->tmC);
    }
    (void)tile_n;
    op->bound[0] = A;
    op->bound[1] = B;
    op->bound[2] = C;
    op->maps_valid = true;
    return XTC_OK;
}

static ConvGeom conv_geom(const xtc_op_desc& d) {
    ConvGeom g;
    memset(&g, 0, sizeof g);
    if (d.kind != XTC_OP_CONV2D) return g;
    int64_t M, N, K, P, Q;
    gemm_view(d, M, N, K, P, Q);
    g.is_conv = 1;
    g.H = (int)d.h; g.W = (int)d.w; g.C = (int)d.c; g.P = (int)P; g.Q = (int)Q;
    g.R = (int)d.r; g.S = (int)d.s; g.sh = (int)d.stride_h; g.sw = (int)d.stride_w;
    g.ph = (int)d.pad_h; g.pw = (int)d.pad_w;
    return g;
}

struct GatherArgs {            // xtc_run_gather: device tensor maps of the destinations
    const void* maps;
    int32_t n, row0;
    void* mc = nullptr;        // xtc_run_multicast: the destination and its store mode (1 plain, 2 multimem)
    int64_t mc_ld = 0;
    int32_t mc_mode = 0;
};

static xtc_status run_impl(xtc_op op, const void* A, const void* B, void* C, cudaStream_t st,
                           const GatherArgs* ga = nullptr) {
    const Plan& p = op->plan;
    const xtc_op_desc& d = op->d;
    const int64_t ldc = (d.kind == XTC_OP_MATMUL && d.ldc) ? d.ldc : p.n_total;
    const bool out_bf16 = d.out_dtype == XTC_BF16;
    const bool split_out = p.split_k > 1 && !p.atomic;
    const bool split_cluster = p.split_cluster;      // the reduction runs inside the contraction kernel
    int launches = 0;
    if (p.atomic && !(d.consumer & XTC_CONSUMER_ACCUMULATE)) {
        // atomic split-K accumulates into C: clear the main root's columns first (unless the
        // consumer is C += A*B, which is exactly what the atomics do)
        const int64_t rows = p.M;
        CU_TRY(cudaMemset2DAsync(C, ldc * 4, 0, p.N * 4, rows, st), "memset C (atomic split-K)");
    }
    // cluster_n: the tile map walks cluster tiles (cluster_n adjacent N tiles of one M tile)
    // split cluster: the tile map walks output tiles, the K segment is the CTA's cluster rank
    TileMap tm{p.tiles_m, p.tiles_n / (p.cluster_n > 1 ? p.cluster_n : 1), split_cluster ? 1 : p.split_k, p.sch.order,
               p.sch.raster_group};
    if (p.engine == XTC_ENGINE_MMA) {
        const CUtensorMap* tmX = nullptr;
        if (p.mma_patch && p.mp.tma) {
            // the patch map: x viewed as {16-element chunk, W*C/16 chunks, H, N}; one box
            // {16, chunks, pr, 1} per tile lands as the tile's [row][chunk][32 B] patch
            if (!op->maps_valid || op->bound[0] != A) {
                xtc_status s0 = load_driver_fns();
                if (s0 != XTC_OK) return s0;
                if (reinterpret_cast<uintptr_t>(A) & 15) return fail(XTC_E_INVALID_ARG, "MMA patch (TMA): x must be 16-byte aligned");
                const cuuint64_t wc = (cuuint64_t)(d.w * d.c);
                cuuint64_t dims[4] = {16, wc / 16, (cuuint64_t)d.h, (cuuint64_t)d.batch};
                cuuint64_t strides[3] = {32, wc * 2, (cuuint64_t)d.h * wc * 2};
                cuuint32_t box[4] = {16, (cuuint32_t)p.mp.chunks, (cuuint32_t)p.mp.pr, 1};
                cuuint32_t estr[4] = {1, 1, 1, 1};
                CUresult r = g_encode_tiled(&op->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(A), dims,
                                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(MMA patch) failed: " + std::to_string((int)r));
                op->bound[0] = A; op->bound[1] = B; op->bound[2] = C;
                op->maps_valid = true;
            }
            tmX = &op->tmA;
        }
        CU_TRY(launch_conv_mma(A, B, C, p, d, op->bias, p.cons_epi, tmX, st), "conv_mma launch");
        ++launches;
    } else if (p.engine == XTC_ENGINE_SIMT) {
        SimtParams sp;
        memset(&sp, 0, sizeof sp);
        sp.A = A; sp.B = B; sp.C = C; sp.Wk = op->ws;
        sp.M = p.M; sp.N = p.N; sp.K = p.K;
        sp.lda = (d.kind == XTC_OP_MATMUL && d.lda) ? d.lda : p.K;
        sp.ldb = (d.kind == XTC_OP_MATMUL && d.ldb) ? d.ldb : p.n_total;
        sp.ldc = ldc;
        sp.ws_ld = p.ws_ld;
        sp.tile_m = p.sch.tile_m; sp.tile_n = p.sch.tile_n; sp.tile_k = p.sch.tile_k;
        sp.pad = p.sch.swizzle;
        sp.stages = p.sch.stages == 0 ? 1 : p.sch.stages;
        sp.k_per_split = p.k_per_split;
        sp.tm = tm;
        sp.num_tiles = p.num_tiles;
        sp.out_bf16 = out_bf16; sp.split_out = split_out; sp.atomic = p.atomic;
        sp.cg = conv_geom(d);
        {
            const int BM = sp.tile_m, BN = sp.tile_n, BK = sp.tile_k, pad = sp.pad;
            const bool aligned = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
            sp.fast = (d.kind == XTC_OP_MATMUL) && aligned && sp.lda % 4 == 0 && sp.ldb % 4 == 0 && BK % 4 == 0 &&
                      BN % 4 == 0 && pad % 4 == 0 && (BM + pad) % 4 == 0 && BM * (BK / 4) <= 4 * p.block;
        }
        sp.cons = p.cons_epi;
        sp.bias = op->bias;
        const int u = p.sch.unroll_k == 0 ? 1 : p.sch.unroll_k;
        const int vec = p.sch.vector_n == 0 ? 1 : p.sch.vector_n;
        CU_TRY(launch_simt_gemm(p.sch.inner_m, p.sch.inner_n, u, vec, sp, p.grid_x, p.block, p.smem, st), "simt_gemm launch");
        ++launches;
    } else {
        if (!op->maps_valid || op->bound[0] != A || op->bound[1] != B || op->bound[2] != C) {
            xtc_status s2 = encode_maps(op, A, B, C);
            if (s2 != XTC_OK) return s2;
        }
        TcParams tp;
        memset(&tp, 0, sizeof tp);
        tp.M = p.M; tp.N = p.N; tp.K = p.K;
        tp.tile_n = p.sch.tile_n; tp.tile_k = p.sch.tile_k; tp.stages = p.sch.stages;
        tp.kb_total = p.kb_total; tp.kb_per_split = p.kb_per_split;
        tp.tm = tm;
        tp.num_tiles = p.num_tiles;
        tp.acc_buffers = p.sch.acc_buffers == 0 ? 1 : p.sch.acc_buffers;
        tp.pack_warps = p.sch.pack_warps == 0 ? 1 : p.sch.pack_warps;
        tp.b_resident = p.sch.b_resident;
        tp.cons = p.cons_epi;
        tp.bias = op->bias;
        tp.a3d = op->a3d;
        tp.debug_skip_mma = getenv("XTC_DEBUG_SKIP_MMA") != nullptr;   // diagnostics: output invalid
        if (const char* sk = getenv("XTC_DEBUG_SKIP")) tp.debug_skip_mma = atoi(sk);   // bitmask, see TcParams
        tp.debug_late_alloc = getenv("XTC_DEBUG_LATE_ALLOC") != nullptr && atoi(getenv("XTC_DEBUG_LATE_ALLOC")) != 0;
        tp.b3d = op->b3d;
        tp.buffer_c = p.sch.buffer_c;
        tp.atomic = p.atomic;
        tp.out_bf16 = out_bf16;
        tp.split_out = split_out;
        tp.ldc = ldc;
        tp.ws_ld = p.ws_ld;
        tp.C = C;
        tp.Wk = op->ws;
        const bool tf32 = d.in_dtype == XTC_TF32 || p.split3;     // 3xTF32: kind::tf32 on fp32 storage
        const uint32_t fmt = tf32 ? 2u : 1u;
        tp.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) |
                   ((uint32_t)(p.sch.tile_n >> 3) << 17) | ((uint32_t)((128 * p.cta_group) >> 4) << 24);
        tp.tmem_cols = (uint32_t)p.tmem_cols;
        const int es = dsize(d.in_dtype);
        tp.a_stage_bytes = (uint32_t)(128 * p.msub * p.sch.tile_k * es);
        tp.ms = p.msub;
        tp.ovl = p.ovl ? 1 : 0;
        tp.b_stage_bytes = (uint32_t)(p.sch.tile_k * (p.sch.tile_n / p.cta_group) * es);
        tp.lo_off = p.split3 ? (uint32_t)(p.sch.stages * (tp.a_stage_bytes + tp.b_stage_bytes)) : 0u;
        tp.cg = conv_geom(d);
        tp.cn = p.cluster_n > 1 ? p.cluster_n : 1;
        tp.ksc = split_cluster ? p.split_k : 1;
        if (p.stream_k) {
            if (!op->sk_flags) {            // per-CTA publish flags, zeroed once; epochs only grow
                CU_TRY(cudaMalloc(&op->sk_flags, kSkMaxCtas * 4 * sizeof(uint32_t)), "stream-K flags alloc");
                CU_TRY(cudaMemset(op->sk_flags, 0, kSkMaxCtas * 4 * sizeof(uint32_t)), "stream-K flags clear");
                CU_TRY(cudaDeviceSynchronize(), "stream-K flags clear");
            }
            if (p.grid_x > kSkMaxCtas) return fail(XTC_E_UNSUPPORTED, "stream-K grid exceeds the flag array");
            if (++op->sk_epoch == 0) ++op->sk_epoch;
            tp.sk = 1;
            tp.sk_iters = p.sk_iters;
            tp.sk_slot = p.sk_slot;
            tp.sk_flags = op->sk_flags;
            tp.sk_epoch = op->sk_epoch;
        }
        tp.cons_red = split_cluster ? p.cons_reduce : 0;
        if (ga) {
            tp.gather = ga->maps;
            tp.n_gather = ga->n;
            tp.gather_row0 = ga->row0;
            tp.mc = ga->mc;
            tp.mc_ld = ga->mc_ld;
            tp.mc_mode = ga->mc_mode;
        }
        const size_t trace_bytes = (size_t)kTraceCtas * kTraceSlots * 8;
        if (!op->trace_path.empty()) {
            if (!op->trace_dev) CU_TRY(cudaMalloc(&op->trace_dev, trace_bytes), "trace alloc");
            CU_TRY(cudaMemsetAsync(op->trace_dev, 0, trace_bytes, st), "trace clear");
            tp.trace = op->trace_dev;
        }
        if (p.halo) {
            tp.wp = p.halo_wp;
            tp.rt = p.halo_rt;
            tp.msub = p.halo_msub;
            tp.planes = p.halo_planes;
            tp.nbuf = p.halo_nbuf;
            tp.tpi = p.halo_tpi;
            tp.cl = p.halo_cl;
            tp.pair = p.halo_pair ? 1 : 0;
            tp.sfold = p.halo_sfold;
            tp.compact = p.halo_compact ? 1 : 0;
            tp.b64 = p.halo_b64 ? 1 : 0;
            if (p.halo_sfold > 1)                     // UMMA N = S * tile_n
                tp.idesc = (tp.idesc & ~(0x3Fu << 17)) | ((uint32_t)((p.halo_sfold * p.sch.tile_n) >> 3) << 17);
            tp.patch_bytes = (uint32_t)p.halo_patch_bytes;
            tp.plane_bytes = (uint32_t)(p.halo_patch_bytes / p.halo_planes);
            tp.patch_tx = (uint32_t)((int64_t)p.halo_planes * p.halo_pr * p.halo_wp * 128);
            CU_TRY(launch_tc_conv_halo(tf32, op->tmA, op->tmB, op->tmC, tp, p.grid_x, p.smem, st), "conv_halo launch");
            ++launches;
        } else {
            CU_TRY(launch_tc_gemm(tf32, d.kind == XTC_OP_CONV2D, p.cta_group, op->tmA, op->tmB, op->tmC, tp, p.grid_x,
                                  p.smem, st),
                   "tc_gemm launch");
            ++launches;
        }
        if (tp.trace) {
            std::vector<uint64_t> h((size_t)kTraceCtas * kTraceSlots);
            CU_TRY(cudaMemcpyAsync(h.data(), op->trace_dev, trace_bytes, cudaMemcpyDeviceToHost, st), "trace D2H");
            CU_TRY(cudaStreamSynchronize(st), "trace sync");
            if (FILE* f = fopen(op->trace_path.c_str(), "a")) {
                fprintf(f, "{\"M\":%lld,\"N\":%lld,\"K\":%lld,\"tile_n\":%d,\"tile_k\":%d,\"stages\":%d,\"cta_group\":%d,"
                           "\"grid\":%d,\"num_tiles\":%lld,\"kb_per_split\":%d,\"slots\":%d,\"kK\":%d,\"kT\":%d,\"t\":[",
                        (long long)p.M, (long long)p.N, (long long)p.K, p.sch.tile_n, p.sch.tile_k, p.sch.stages,
                        p.cta_group, p.grid_x, (long long)p.num_tiles, p.kb_per_split, kTraceSlots, kTraceK, kTraceTiles);
                for (size_t i = 0; i < h.size(); ++i) fprintf(f, "%s%llu", i ? "," : "", (unsigned long long)h[i]);
                fprintf(f, "]}\n");
                fclose(f);
            }
        }
    }
    if (split_out && !split_cluster) {
        CU_TRY(launch_splitk_reduce(op->ws, p.split_k, p.M, p.N, p.ws_ld, C, ldc, out_bf16, p.cons_reduce, op->bias, st),
               "splitk_reduce");
        ++launches;
    }
    if (p.has_tail) {
        const int64_t lda = d.lda ? d.lda : d.k;
        const int64_t ldb = d.ldb ? d.ldb : d.n;
        CU_TRY(launch_tail_gemm(A, B, d.in_dtype == XTC_BF16, C, out_bf16, p.cons_tail, op->bias, p.M, p.tail_n0,
                                p.tail_n, p.K, lda, ldb, ldc, p.tail_grid_x, p.tail_grid_y, st),
               "tail_gemm");
        ++launches;
    }
    if (p.cons_pass) {                       // fuse = 0: the consumer as its own pass
        CU_TRY(launch_consumer_pass(C, out_bf16, p.M, p.n_total, ldc, p.cons_pass, op->bias, st), "consumer pass");
        ++launches;
    }
    if (op->fault) {
        CU_TRY(launch_fault(C, out_bf16, p.M, p.n_total, ldc, op->fault, op->fault_row, op->fault_col, st), "fault");
        ++launches;
    }
    op->last_launches = launches;
    return XTC_OK;
}

// inputs[2] is the bias when the consumer has XTC_CONSUMER_BIAS (only then is it read)
static xtc_status bind_bias(xtc_op op, const void* const* inputs) {
    op->bias = nullptr;
    if (op->d.consumer & XTC_CONSUMER_BIAS) {
        if (!inputs[2]) return fail(XTC_E_INVALID_ARG, "consumer XTC_CONSUMER_BIAS needs inputs[2] (fp32 bias)");
        op->bias = static_cast<const float*>(inputs[2]);
    }
    return XTC_OK;
}

extern "C" xtc_status xtc_run(xtc_op op, const void* const* inputs, void* const* outputs, void* stream) {
    if (!op || !inputs || !outputs || !inputs[0] || !inputs[1] || !outputs[0])
        return fail(XTC_E_INVALID_ARG, "null op or tensor pointer");
    if (!op->has_plan) return fail(XTC_E_NO_SCHEDULE, "xtc_run before xtc_schedule_apply");
    if (bind_bias(op, inputs) != XTC_OK) return XTC_E_INVALID_ARG;
    DeviceGuard g(op->device);
    if (op->plan.engine == XTC_ENGINE_TCGEN05) {
        for (int i = 0; i < 2; ++i)
            if (reinterpret_cast<uintptr_t>(inputs[i]) & 15) return fail(XTC_E_INVALID_ARG, "TMA needs 16-byte aligned inputs");
        if (op->plan.sch.buffer_c && (reinterpret_cast<uintptr_t>(outputs[0]) & 15))
            return fail(XTC_E_INVALID_ARG, "TMA store needs a 16-byte aligned output");
    }
    return run_impl(op, inputs[0], inputs[1], outputs[0], (cudaStream_t)stream);
}

extern "C" xtc_status xtc_run_gather(xtc_op op, const void* const* inputs, void* const* dests, int32_t n_dest,
                                     int64_t row_offset, int64_t dest_rows, void* stream) {
    if (!op || !inputs || !dests || !inputs[0] || !inputs[1]) return fail(XTC_E_INVALID_ARG, "null op or tensor pointer");
    if (!op->has_plan) return fail(XTC_E_NO_SCHEDULE, "xtc_run_gather before xtc_schedule_apply");
    if (n_dest < 1 || n_dest > 8) return fail(XTC_E_INVALID_ARG, "xtc_run_gather: n_dest must be in [1, 8]");
    const Plan& p = op->plan;
    const xtc_op_desc& d = op->d;
    if (d.kind != XTC_OP_MATMUL || p.engine != XTC_ENGINE_TCGEN05 || !p.sch.buffer_c || p.split_k != 1 || p.halo ||
        p.has_tail || p.cons_pass || p.split3 || (d.consumer & XTC_CONSUMER_ACCUMULATE))
        return fail(XTC_E_UNSUPPORTED, "xtc_run_gather: needs a tcgen05 matmul schedule with buffer_c=1, split_k=1, "
                                       "no split_n_at root, fused consumers other than accumulate");
    const int64_t tile_rows = 128 * (int64_t)p.cta_group * p.msub;
    if (p.M % tile_rows) return fail(XTC_E_UNSUPPORTED, "xtc_run_gather: M must be a multiple of the CTA tile rows");
    if (row_offset < 0 || row_offset + p.M > dest_rows || dest_rows > INT32_MAX)
        return fail(XTC_E_INVALID_ARG, "xtc_run_gather: rows [row_offset, row_offset + M) must lie in [0, dest_rows)");
    for (int i = 0; i < 2; ++i)
        if (reinterpret_cast<uintptr_t>(inputs[i]) & 15) return fail(XTC_E_INVALID_ARG, "TMA needs 16-byte aligned inputs");
    for (int i = 0; i < n_dest; ++i)
        if (!dests[i] || (reinterpret_cast<uintptr_t>(dests[i]) & 15))
            return fail(XTC_E_INVALID_ARG, "xtc_run_gather: null or unaligned destination");
    if (bind_bias(op, inputs) != XTC_OK) return XTC_E_INVALID_ARG;
    DeviceGuard g(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int os = dsize(d.out_dtype);
    const int64_t ld = d.ldc ? d.ldc : p.n_total;
    bool same = op->n_gbound == n_dest && op->g_rows == dest_rows;
    for (int i = 0; same && i < n_dest; ++i) same = op->gbound[i] == dests[i];
    if (!same) {
        xtc_status s = load_driver_fns();
        if (s != XTC_OK) return s;
        const CUtensorMapDataType out_t = os == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        for (int i = 0; i < n_dest; ++i) {
            cuuint64_t dims[3] = {(cuuint64_t)p.N, (cuuint64_t)dest_rows, 1};
            cuuint64_t strides[2] = {(cuuint64_t)(ld * os), (cuuint64_t)(ld * os * dest_rows)};
            cuuint32_t box[3] = {(cuuint32_t)(128 / os), 32, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            CUresult r = g_encode_tiled(&op->gmaps[i], out_t, 3, dests[i], dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(XTC_E_CUDA, "cuTensorMapEncodeTiled(gather dest) failed: " + std::to_string((int)r));
        }
        if (!op->gmaps_dev) CU_TRY(cudaMalloc(&op->gmaps_dev, sizeof op->gmaps), "gather maps alloc");
        // pageable source: the call returns once the maps are staged, so op->gmaps may change afterwards
        CU_TRY(cudaMemcpyAsync(op->gmaps_dev, op->gmaps, n_dest * sizeof(CUtensorMap), cudaMemcpyHostToDevice, st),
               "gather maps upload");
        for (int i = 0; i < 8; ++i) op->gbound[i] = i < n_dest ? dests[i] : nullptr;
        op->n_gbound = n_dest;
        op->g_rows = dest_rows;
    }
    // C (for the unused local map) = this shard's rows of the first destination
    void* c_local = static_cast<uint8_t*>(dests[0]) + row_offset * ld * os;
    GatherArgs ga{op->gmaps_dev, n_dest, (int32_t)row_offset};
    return run_impl(op, inputs[0], inputs[1], c_local, st, &ga);
}

extern "C" xtc_status xtc_run_multicast(xtc_op op, const void* const* inputs, void* dest, int64_t row_offset,
                                        int64_t dest_rows, int32_t multimem, void* stream) {
    if (!op || !inputs || !dest || !inputs[0] || !inputs[1]) return fail(XTC_E_INVALID_ARG, "null op or tensor pointer");
    if (!op->has_plan) return fail(XTC_E_NO_SCHEDULE, "xtc_run_multicast before xtc_schedule_apply");
    if (multimem != 0 && multimem != 1) return fail(XTC_E_INVALID_ARG, "xtc_run_multicast: multimem must be 0 or 1");
    const Plan& p = op->plan;
    const xtc_op_desc& d = op->d;
    if (d.kind != XTC_OP_MATMUL || p.engine != XTC_ENGINE_TCGEN05 || !p.sch.buffer_c || p.split_k != 1 || p.halo ||
        p.has_tail || p.cons_pass || p.split3 || (d.consumer & XTC_CONSUMER_ACCUMULATE) || p.cluster_n > 1)
        return fail(XTC_E_UNSUPPORTED, "xtc_run_multicast: needs a tcgen05 matmul schedule with buffer_c=1, split_k=1, "
                                       "cluster_n 1, no split_n_at root, fused consumers other than accumulate");
    const int os = dsize(d.out_dtype);
    const int64_t ld = d.ldc ? d.ldc : p.n_total;
    const int64_t tile_rows = 128 * (int64_t)p.cta_group * p.msub;
    if (p.M % tile_rows) return fail(XTC_E_UNSUPPORTED, "xtc_run_multicast: M must be a multiple of the CTA tile rows");
    if ((p.N * os) % 16 || (ld * os) % 16)
        return fail(XTC_E_UNSUPPORTED, "xtc_run_multicast: N and the row pitch must be multiples of 16 bytes");
    if (row_offset < 0 || row_offset + p.M > dest_rows)
        return fail(XTC_E_INVALID_ARG, "xtc_run_multicast: rows [row_offset, row_offset + M) must lie in [0, dest_rows)");
    for (int i = 0; i < 2; ++i)
        if (reinterpret_cast<uintptr_t>(inputs[i]) & 15) return fail(XTC_E_INVALID_ARG, "TMA needs 16-byte aligned inputs");
    if (reinterpret_cast<uintptr_t>(dest) & 15) return fail(XTC_E_INVALID_ARG, "xtc_run_multicast: unaligned destination");
    if (bind_bias(op, inputs) != XTC_OK) return XTC_E_INVALID_ARG;
    DeviceGuard g(op->device);
    if (multimem) {
        typedef CUresult (*PFN_attr)(int*, CUdevice_attribute, CUdevice);
        static PFN_attr get_attr = nullptr;
        if (!get_attr) {
            cudaDriverEntryPointQueryResult q;
            void* fn = nullptr;
            CU_TRY(cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fn, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
            if (!fn || q != cudaDriverEntryPointSuccess) return fail(XTC_E_CUDA, "cuDeviceGetAttribute unavailable");
            get_attr = reinterpret_cast<PFN_attr>(fn);
        }
        int mc = 0;
        if (get_attr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)op->device) != CUDA_SUCCESS || !mc)
            return fail(XTC_E_UNSUPPORTED, "xtc_run_multicast: the device does not support multicast (NVLS)");
    }
    // the local C map is encoded on the shard's rows of the destination but never stored through:
    // the epilogue writes every staged tile with 16-byte (multimem) stores
    void* c_local = static_cast<uint8_t*>(dest) + row_offset * ld * os;
    GatherArgs ga{nullptr, 0, (int32_t)row_offset, dest, ld, multimem ? 2 : 1};
    return run_impl(op, inputs[0], inputs[1], c_local, (cudaStream_t)stream, &ga);
}

// --------------------------------------------------------------- measure --
static xtc_status ensure_flush(int device, cudaStream_t) {
    if (device < 0 || device >= 64) return fail(XTC_E_INVALID_ARG, "device index");
    if (g_flush_buf[device]) return XTC_OK;
    int l2 = 0;
    CU_TRY(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device), "L2 size");
    const int64_t bytes = std::max<int64_t>(2 * (int64_t)l2, 64 << 20);
    if (cudaMalloc(&g_flush_buf[device], bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(XTC_E_OOM, "L2 flush buffer allocation failed");
    }
    g_flush_bytes[device] = bytes;
    return XTC_OK;
}

static xtc_status compute_reference(xtc_op op, const void* A, const void* B, cudaStream_t st) {
    const xtc_op_desc& d = op->d;
    int64_t M, N, K, P, Q;
    gemm_view(d, M, N, K, P, Q);
    const int64_t elems = M * N;
    if (elems > op->ref_elems) {
        if (op->R) cudaFree(op->R);
        if (op->D) cudaFree(op->D);
        op->R = op->D = nullptr;
        op->ref_elems = 0;
        if (cudaMalloc(&op->R, elems * 8) != cudaSuccess || cudaMalloc(&op->D, elems * 8) != cudaSuccess) {
            cudaGetLastError();
            return fail(XTC_E_OOM, "reference buffers (2 x 8 B per output) allocation failed");
        }
        op->ref_elems = elems;
    }
    const int bf16 = d.in_dtype == XTC_BF16;
    if (d.kind == XTC_OP_MATMUL) {
        const int64_t lda = d.lda ? d.lda : d.k, ldb = d.ldb ? d.ldb : d.n;
        CU_TRY(launch_ref_gemm(A, B, bf16, M, N, K, lda, ldb, op->R, op->D, st), "ref_gemm");
    } else {
        CU_TRY(launch_ref_conv(A, B, bf16, conv_geom(d), d.batch, d.f, op->R, op->D, st), "ref_conv");
    }
    op->ref_inputs[0] = A;
    op->ref_inputs[1] = B;
    op->ref_valid = true;
    return XTC_OK;
}

static const int kCmpBlocks = 148 * 8;

// Copy the output (M rows of N elements, pitch ldc) into the op's snapshot buffer (same layout).
static xtc_status snapshot_output(xtc_op op, const void* C, int64_t M, int64_t N, int64_t ldc, int os, cudaStream_t st) {
    const int64_t bytes = M * ldc * os;
    if (op->c_old_bytes < bytes) {
        if (op->c_old) cudaFree(op->c_old);
        op->c_old = nullptr;
        op->c_old_bytes = 0;
        if (cudaMalloc(&op->c_old, bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(XTC_E_OOM, "accumulate snapshot");
        }
        op->c_old_bytes = bytes;
    }
    CU_TRY(cudaMemcpy2DAsync(op->c_old, ldc * os, C, ldc * os, N * os, M, cudaMemcpyDeviceToDevice, st), "snapshot C");
    return XTC_OK;
}

static xtc_status validate(xtc_op op, const void* A, const void* B, void* C, const xtc_measure_cfg* cfg,
                           xtc_metrics* m, cudaStream_t st) {
    const xtc_op_desc& d = op->d;
    int64_t M, N, K, P, Q;
    gemm_view(d, M, N, K, P, Q);
    const int64_t ldc = (d.kind == XTC_OP_MATMUL && d.ldc) ? d.ldc : N;
    const int os = dsize(d.out_dtype);
    CmpConsumer cc{d.consumer, op->bias, nullptr};
    if (d.consumer & XTC_CONSUMER_ACCUMULATE) {
        // C is an input: snapshot it (the reference is C_old + A*B ...) instead of the sentinel
        xtc_status s0 = snapshot_output(op, C, M, N, ldc, os, st);
        if (s0 != XTC_OK) return s0;
        cc.c_old = op->c_old;
    } else {
        // NaN sentinel: every output the schedule fails to write stays NaN (coverage)
        CU_TRY(cudaMemset2DAsync(C, ldc * os, 0xFF, N * os, M, st), "NaN fill");
    }
    xtc_status s = run_impl(op, A, B, C, st);
    if (s != XTC_OK) return s;
    if (!(cfg->reuse_reference && op->ref_valid && op->ref_inputs[0] == A && op->ref_inputs[1] == B)) {
        s = compute_reference(op, A, B, st);
        if (s != XTC_OK) return s;
    }
    if (!op->blk_err) {
        if (cudaMalloc(&op->blk_err, kCmpBlocks * 8) != cudaSuccess || cudaMalloc(&op->blk_idx, kCmpBlocks * 8) != cudaSuccess ||
            cudaMalloc(&op->counts, 16) != cudaSuccess) {
            cudaGetLastError();
            return fail(XTC_E_OOM, "compare buffers");
        }
    }
    CU_TRY(cudaMemsetAsync(op->counts, 0, 16, st), "memset counts");
    CU_TRY(launch_compare(C, d.out_dtype == XTC_BF16, cc, M, N, ldc, op->R, op->D, op->blk_err, op->blk_idx,
                          op->counts, kCmpBlocks, st),
           "compare");
    std::vector<double> be(kCmpBlocks);
    std::vector<int64_t> bi(kCmpBlocks);
    unsigned long long cnt[2];
    CU_TRY(cudaMemcpyAsync(be.data(), op->blk_err, kCmpBlocks * 8, cudaMemcpyDeviceToHost, st), "D2H err");
    CU_TRY(cudaMemcpyAsync(bi.data(), op->blk_idx, kCmpBlocks * 8, cudaMemcpyDeviceToHost, st), "D2H idx");
    CU_TRY(cudaMemcpyAsync(cnt, op->counts, 16, cudaMemcpyDeviceToHost, st), "D2H counts");
    CU_TRY(cudaStreamSynchronize(st), "validate sync");
    double best = -1;
    int64_t bidx = -1;
    for (int i = 0; i < kCmpBlocks; ++i)
        if (bi[i] >= 0 && (be[i] > best || (be[i] == best && bi[i] < bidx))) { best = be[i]; bidx = bi[i]; }
    m->max_norm_err = best < 0 ? 0.0 : best;
    m->err_row = bidx >= 0 ? bidx / N : -1;
    m->err_col = bidx >= 0 ? bidx % N : -1;
    m->n_mismatch = (int64_t)cnt[0];
    m->n_nan = (int64_t)cnt[1];
    double tol = cfg->tol;
    if (tol <= 0) tol = d.in_dtype == XTC_F32 ? 1e-5 : 5e-3;
    bool ok = m->n_nan == 0 && m->max_norm_err <= tol;
    if (cfg->exact) ok = ok && m->n_mismatch == 0;
    m->valid = ok ? 1 : 0;
    return XTC_OK;
}

static xtc_status measure_impl(xtc_op op, const void* A, const void* B, void* C, const xtc_measure_cfg* cfg,
                               xtc_metrics* m, cudaStream_t st) {
    memset(m, 0, sizeof *m);
    m->valid = -1;
    m->err_row = m->err_col = -1;
    if (cfg->repeats < 1 || cfg->warmup < 0) return fail(XTC_E_INVALID_ARG, "repeats must be >= 1, warmup >= 0");
    if (cfg->validate) {
        xtc_status s = validate(op, A, B, C, cfg, m, st);
        if (s != XTC_OK) return s;
    }
    for (int i = 0; i < cfg->warmup; ++i) {
        xtc_status s = run_impl(op, A, B, C, st);
        if (s != XTC_OK) return s;
    }
    if (cfg->flush_l2) {
        xtc_status s = ensure_flush(op->device, st);
        if (s != XTC_OK) return s;
    }
    const int R = cfg->repeats;
    while ((int)op->evs.size() < 2 * R) {
        cudaEvent_t e;
        CU_TRY(cudaEventCreate(&e), "cudaEventCreate");
        op->evs.push_back(e);
    }
    // keep the GPU busy while the reps are enqueued: if the host falls behind, a rep's start event
    // executes before its kernel is even submitted and the host's enqueue time lands inside the
    // measurement.  Host enqueue is ~3-6 us per rep (flush + 2 events + the launch) on a quiet host;
    // budget 30 us per rep + 20 us (XTC_MEASURE_DELAY_NS: per-rep budget, diagnostics)
    uint64_t per_rep = 30000ull;
    if (const char* e = getenv("XTC_MEASURE_DELAY_NS")) per_rep = strtoull(e, nullptr, 10);
    CU_TRY(launch_delay(std::min<uint64_t>(per_rep * (uint64_t)R + 20000ull, 20000000ull), st), "delay");
    for (int i = 0; i < R; ++i) {
        if (cfg->flush_l2) CU_TRY(launch_flush(g_flush_buf[op->device], g_flush_bytes[op->device], (uint32_t)i, st), "flush");
        CU_TRY(cudaEventRecord(op->evs[2 * i], st), "event");
        xtc_status s = run_impl(op, A, B, C, st);
        if (s != XTC_OK) return s;
        CU_TRY(cudaEventRecord(op->evs[2 * i + 1], st), "event");
    }
    CU_TRY(cudaEventSynchronize(op->evs[2 * R - 1]), "event sync");
    m->sm_clock_mhz = sm_clock_mhz(op->device);
    std::vector<double> t(R);
    for (int i = 0; i < R; ++i) {
        float ms = 0;
        CU_TRY(cudaEventElapsedTime(&ms, op->evs[2 * i], op->evs[2 * i + 1]), "elapsed");
        t[i] = ms * 1e6;
    }
    std::vector<double> srt = t;
    std::sort(srt.begin(), srt.end());
    m->t_min_ns = srt.front();
    m->t_max_ns = srt.back();
    m->t_med_ns = (R % 2) ? srt[R / 2] : 0.5 * (srt[R / 2 - 1] + srt[R / 2]);
    double sum = 0;
    for (double v : t) sum += v;
    m->t_mean_ns = sum / R;
    const double flops = xtc_op_flops(&op->d);
    m->tflops_med = flops / m->t_med_ns * 1e-3;
    m->tflops_min = flops / m->t_min_ns * 1e-3;
    m->frac_peak = cfg->peak_tflops > 0 ? m->tflops_med / cfg->peak_tflops : 0.0;
    m->n_reps = R;
    if (cfg->counters && *cfg->counters) {
        // separate pass, after the timed region: one range = one operator call
        std::vector<std::string> names = split_counter_names(cfg->counters);
        if (names.size() > 8) return fail(XTC_E_INVALID_ARG, "at most 8 counters per measurement");
        for (int i = 0; i < 8; ++i) m->counters[i] = std::nan("");
        std::vector<double> vals;
        std::string why;
        xtc_status rs = XTC_OK;
        auto prepare = [&] {  // same cache state as the timed reps: flushed before each replay
            if (cfg->flush_l2 &&
                launch_flush(g_flush_buf[op->device], g_flush_bytes[op->device], 0u, st) != cudaSuccess)
                return false;
            return cudaStreamSynchronize(st) == cudaSuccess;
        };
        auto once = [&] {
            rs = run_impl(op, A, B, C, st);
            return rs == XTC_OK && cudaStreamSynchronize(st) == cudaSuccess;
        };
        if (!names.empty() && collect_counters(op->device, names, prepare, once, vals, why)) {
            m->n_counters = (int32_t)names.size();
            for (size_t i = 0; i < names.size(); ++i) m->counters[i] = vals[i];
        } else {
            if (rs != XTC_OK) return rs;
            m->n_counters = -1;
            g_err = "counters unavailable: " + why;  // documented: readable although the status is XTC_OK
        }
    }
    m->status = XTC_OK;
    return XTC_OK;
}

extern "C" xtc_status xtc_measure(xtc_op op, const void* const* inputs, void* const* outputs,
                                  const xtc_measure_cfg* cfg, xtc_metrics* out, void* stream) {
    if (!op || !inputs || !outputs || !cfg || !out || !inputs[0] || !inputs[1] || !outputs[0])
        return fail(XTC_E_INVALID_ARG, "null argument");
    if (!op->has_plan) return fail(XTC_E_NO_SCHEDULE, "xtc_measure before xtc_schedule_apply");
    if (bind_bias(op, inputs) != XTC_OK) return XTC_E_INVALID_ARG;
    DeviceGuard g(op->device);
    xtc_status s = measure_impl(op, inputs[0], inputs[1], outputs[0], cfg, out, (cudaStream_t)stream);
    if (s != XTC_OK) { out->status = s; return s; }
    if (cfg->validate == 2 && out->valid == 0) return fail(XTC_E_VALIDATION_FAILED, "validation failed");
    return XTC_OK;
}

extern "C" xtc_status xtc_sweep(xtc_op op, const xtc_schedule* cands, int32_t n, const void* const* inputs,
                                void* const* outputs, const xtc_measure_cfg* cfg, xtc_metrics* out, void* stream) {
    if (!op || !cands || n < 0 || !out || !cfg || !inputs || !outputs) return fail(XTC_E_INVALID_ARG, "null argument");
    if (cfg->repeats < 1 || cfg->warmup < 0) return fail(XTC_E_INVALID_ARG, "repeats must be >= 1, warmup >= 0");
    if (bind_bias(op, inputs) != XTC_OK) return XTC_E_INVALID_ARG;
    DeviceGuard g(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    const void* A = inputs[0];
    const void* B = inputs[1];
    void* C = outputs[0];
    const xtc_op_desc& d = op->d;
    int64_t M, N, K, P, Q;
    gemm_view(d, M, N, K, P, Q);
    const int64_t ldc = (d.kind == XTC_OP_MATMUL && d.ldc) ? d.ldc : N;
    const int os = dsize(d.out_dtype);
    const int R = cfg->repeats;
    double tol = cfg->tol;
    if (tol <= 0) tol = d.in_dtype == XTC_F32 ? 1e-5 : 5e-3;

    // 1. plan every candidate on the host; illegal ones launch nothing
    std::vector<Plan> plans(n);
    std::vector<char> legal(n, 0);
    int64_t ws_max = 0;
    for (int i = 0; i < n; ++i) {
        memset(&out[i], 0, sizeof out[i]);
        out[i].valid = -1;
        out[i].err_row = out[i].err_col = -1;
        std::string why;
        xtc_status s = make_plan(d, cands[i], op->num_sms, plans[i], why);
        out[i].status = s;
        if (s == XTC_OK) {
            legal[i] = 1;
            ws_max = std::max(ws_max, plans[i].workspace_bytes);
        }
    }
    // 2. resources sized once for the whole sweep: no allocation (an implicit device
    //    synchronisation) between candidates
    if (ws_max > op->ws_bytes) {
        if (op->ws) cudaFree(op->ws);
        op->ws = nullptr;
        op->ws_bytes = 0;
        if (cudaMalloc(&op->ws, ws_max) != cudaSuccess) {
            cudaGetLastError();
            return fail(XTC_E_OOM, "split-K workspace allocation failed");
        }
        op->ws_bytes = ws_max;
    }
    if (cfg->flush_l2) {
        xtc_status s = ensure_flush(op->device, st);
        if (s != XTC_OK) return s;
    }
    if (cfg->validate) {
        if (!(cfg->reuse_reference && op->ref_valid && op->ref_inputs[0] == A && op->ref_inputs[1] == B)) {
            xtc_status s = compute_reference(op, A, B, st);
            if (s != XTC_OK) return s;
        }
        if (!op->blk_err) {
            if (cudaMalloc(&op->blk_err, kCmpBlocks * 8) != cudaSuccess ||
                cudaMalloc(&op->blk_idx, kCmpBlocks * 8) != cudaSuccess || cudaMalloc(&op->counts, 16) != cudaSuccess) {
                cudaGetLastError();
                return fail(XTC_E_OOM, "compare buffers");
            }
        }
        CU_TRY(cudaMemsetAsync(op->counts, 0, 16, st), "memset counts");
    }
    // accumulate: the output is an input; every candidate is validated from the same C_old
    const bool accum = (d.consumer & XTC_CONSUMER_ACCUMULATE) != 0;
    if (cfg->validate && accum) {
        xtc_status s = snapshot_output(op, C, M, N, ldc, os, st);
        if (s != XTC_OK) return s;
    }
    const CmpConsumer cc{d.consumer, op->bias, accum ? op->c_old : nullptr};
    // 3. chunks of candidates enqueued back to back, one synchronisation per chunk: the host
    //    stays ahead of the GPU, so the per-rep events bracket GPU work only (no delay kernel)
    const int CH = 64;
    double* slots = nullptr;
    if (cfg->validate && cudaMalloc(&slots, (size_t)CH * 4 * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(XTC_E_OOM, "sweep validation slots");
    }
    std::vector<cudaEvent_t> ev((size_t)CH * 2 * R);
    for (auto& e : ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            if (slots) cudaFree(slots);
            return cuda_fail(cudaGetLastError(), "cudaEventCreate");
        }
    auto cleanup = [&]() {
        for (auto e : ev) cudaEventDestroy(e);
        if (slots) cudaFree(slots);
    };
    const bool had_plan = op->has_plan;
    Plan saved = op->plan;
    const double flops = xtc_op_flops(&d);
    std::vector<double> hslots((size_t)CH * 4);
    for (int c0 = 0; c0 < n; c0 += CH) {
        const int c1 = std::min(n, c0 + CH);
        for (int i = c0; i < c1; ++i) {
            if (!legal[i]) continue;
            op->plan = plans[i];
            op->has_plan = true;
            op->maps_valid = false;           // TMA boxes depend on the schedule
            xtc_status s = XTC_OK;
            if (cfg->validate) {
                const cudaError_t pre =
                    accum ? cudaMemcpy2DAsync(C, ldc * os, op->c_old, ldc * os, N * os, M, cudaMemcpyDeviceToDevice, st)
                          : cudaMemset2DAsync(C, ldc * os, 0xFF, N * os, M, st);   // NaN sentinel
                if (pre != cudaSuccess) s = XTC_E_CUDA;
                if (s == XTC_OK) s = run_impl(op, A, B, C, st);
                if (s == XTC_OK && (launch_compare(C, d.out_dtype == XTC_BF16, cc, M, N, ldc, op->R, op->D, op->blk_err,
                                                   op->blk_idx, op->counts, kCmpBlocks, st) != cudaSuccess ||
                                    launch_compare_finalize(op->blk_err, op->blk_idx, kCmpBlocks, op->counts,
                                                            slots + (size_t)(i - c0) * 4, st) != cudaSuccess))
                    s = XTC_E_CUDA;
            }
            for (int w = 0; s == XTC_OK && w < cfg->warmup; ++w) s = run_impl(op, A, B, C, st);
            for (int r = 0; s == XTC_OK && r < R; ++r) {
                if (cfg->flush_l2 &&
                    launch_flush(g_flush_buf[op->device], g_flush_bytes[op->device], (uint32_t)r, st) != cudaSuccess) {
                    s = XTC_E_CUDA;
                    break;
                }
                cudaEventRecord(ev[((size_t)(i - c0) * R + r) * 2], st);
                s = run_impl(op, A, B, C, st);
                cudaEventRecord(ev[((size_t)(i - c0) * R + r) * 2 + 1], st);
            }
            out[i].status = s;
            if (s == XTC_E_CUDA) {
                cleanup();
                return s;
            }
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) {
            cleanup();
            return cuda_fail(cudaGetLastError(), "sweep chunk sync");
        }
        const double clk = sm_clock_mhz(op->device);
        if (cfg->validate &&
            cudaMemcpy(hslots.data(), slots, (size_t)(c1 - c0) * 4 * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cleanup();
            return cuda_fail(cudaGetLastError(), "sweep slots D2H");
        }
        for (int i = c0; i < c1; ++i) {
            if (!legal[i] || out[i].status != XTC_OK) continue;
            xtc_metrics& m = out[i];
            if (cfg->validate) {
                const double* sl = &hslots[(size_t)(i - c0) * 4];
                m.max_norm_err = sl[0];
                const int64_t idx = (int64_t)sl[1];
                m.err_row = idx >= 0 ? idx / N : -1;
                m.err_col = idx >= 0 ? idx % N : -1;
                m.n_mismatch = (int64_t)sl[2];
                m.n_nan = (int64_t)sl[3];
                bool ok = m.n_nan == 0 && m.max_norm_err <= tol;
                if (cfg->exact) ok = ok && m.n_mismatch == 0;
                m.valid = ok ? 1 : 0;
            }
            std::vector<double> t(R);
            for (int r = 0; r < R; ++r) {
                float ms = 0;
                cudaEventElapsedTime(&ms, ev[((size_t)(i - c0) * R + r) * 2], ev[((size_t)(i - c0) * R + r) * 2 + 1]);
                t[r] = ms * 1e6;
            }
            std::vector<double> srt = t;
            std::sort(srt.begin(), srt.end());
            m.t_min_ns = srt.front();
            m.t_max_ns = srt.back();
            m.t_med_ns = (R % 2) ? srt[R / 2] : 0.5 * (srt[R / 2 - 1] + srt[R / 2]);
            double sum = 0;
            for (double v : t) sum += v;
            m.t_mean_ns = sum / R;
            m.tflops_med = flops / m.t_med_ns * 1e-3;
            m.tflops_min = flops / m.t_min_ns * 1e-3;
            m.frac_peak = cfg->peak_tflops > 0 ? m.tflops_med / cfg->peak_tflops : 0.0;
            m.sm_clock_mhz = clk;
            m.n_reps = R;
        }
    }
    cleanup();
    // the op keeps the last legal candidate's schedule (or its previous one if none was legal)
    int last = -1;
    for (int i = n - 1; i >= 0; --i)
        if (legal[i]) { last = i; break; }
    if (last >= 0) {
        op->plan = plans[last];
        op->has_plan = true;
    } else {
        op->plan = saved;
        op->has_plan = had_plan;
    }
    op->maps_valid = false;
    return XTC_OK;
}
