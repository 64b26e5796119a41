"""paper_2512_16512_b200 -- B200-native hot path of XTC (arXiv 2512.16512).

A thin ctypes binding over ``libxtc.so`` (the C-ABI declared in
``include/xtc.h``).  Every step of the path runs in the library's sm_100a
kernels; this module only marshals arguments.  There is no CPU fallback:
if the library is missing or the device is not a B200, calls fail loudly.

Functions keep the C names (``xtc_op_create``, ``xtc_schedule_apply``,
``xtc_run``, ``xtc_measure``, ...).  ``Op`` is a small convenience wrapper
taking torch tensors (torch is used only for device memory and streams).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, byref, c_char_p, c_double, c_int32, c_int64, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libxtc.so")

# ----------------------------------------------------------------- enums ---
XTC_OK, XTC_E_INVALID_ARG, XTC_E_UNSUPPORTED, XTC_E_ILLEGAL_SCHEDULE = 0, 1, 2, 3
XTC_E_NO_SCHEDULE, XTC_E_CUDA, XTC_E_VALIDATION_FAILED, XTC_E_OOM = 4, 5, 6, 7
STATUS_NAMES = {0: "XTC_OK", 1: "XTC_E_INVALID_ARG", 2: "XTC_E_UNSUPPORTED", 3: "XTC_E_ILLEGAL_SCHEDULE",
                4: "XTC_E_NO_SCHEDULE", 5: "XTC_E_CUDA", 6: "XTC_E_VALIDATION_FAILED", 7: "XTC_E_OOM"}
XTC_OP_MATMUL, XTC_OP_CONV2D = 0, 1
XTC_F32, XTC_BF16, XTC_TF32 = 0, 1, 2
XTC_ENGINE_SIMT, XTC_ENGINE_TCGEN05, XTC_ENGINE_MMA = 0, 1, 2
XTC_ORDER_MN, XTC_ORDER_NM = 0, 1
XTC_SPLITK_ORDERED, XTC_SPLITK_ATOMIC, XTC_SPLITK_CLUSTER, XTC_SPLITK_STREAM = 0, 1, 2, 3
XTC_CONSUMER_NONE, XTC_CONSUMER_RELU, XTC_CONSUMER_BIAS, XTC_CONSUMER_ACCUMULATE = 0, 1, 2, 4
DTYPES = {"f32": XTC_F32, "bf16": XTC_BF16, "tf32": XTC_TF32}
CONSUMERS = {None: XTC_CONSUMER_NONE, "none": XTC_CONSUMER_NONE, "relu": XTC_CONSUMER_RELU,
             "bias": XTC_CONSUMER_BIAS, "accumulate": XTC_CONSUMER_ACCUMULATE}


def consumer_bits(consumer) -> int:
    """None / an int bitmask / a name / '+'-joined names ('bias+relu', 'accumulate+bias+relu')."""
    if consumer is None or isinstance(consumer, int):
        return int(consumer or 0)
    bits = 0
    for part in str(consumer).split("+"):
        bits |= CONSUMERS[part.strip()]
    return bits


# ------------------------------------------------------------- structs -----
class xtc_op_desc(Structure):
    _fields_ = [("kind", c_int32), ("in_dtype", c_int32), ("out_dtype", c_int32), ("consumer", c_int32),
                ("m", c_int64), ("n", c_int64), ("k", c_int64), ("lda", c_int64), ("ldb", c_int64), ("ldc", c_int64),
                ("batch", c_int64), ("h", c_int64), ("w", c_int64), ("c", c_int64), ("f", c_int64),
                ("r", c_int64), ("s", c_int64),
                ("stride_h", c_int64), ("stride_w", c_int64), ("pad_h", c_int64), ("pad_w", c_int64)]


SCHEDULE_FIELDS = ["engine", "tile_m", "tile_n", "tile_k", "inner_m", "inner_n", "order", "raster_group",
                   "unroll_k", "vector_n", "stages", "swizzle", "buffer_c", "acc_buffers", "split_k",
                   "split_k_mode", "cluster_m", "persistent", "split_n_at", "pack_warps", "b_resident", "fuse",
                   "pack_halo", "cluster_n", "grid_sms"]


class xtc_schedule(Structure):
    _fields_ = [(f, c_int32) for f in SCHEDULE_FIELDS]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f in SCHEDULE_FIELDS}


class xtc_plan_info(Structure):
    _fields_ = [("engine", c_int32), ("grid_x", c_int32), ("grid_y", c_int32), ("grid_z", c_int32),
                ("block_x", c_int32), ("cluster_x", c_int32), ("smem_bytes", c_int32), ("tmem_cols", c_int32),
                ("num_tiles", c_int64), ("k_blocks_per_split", c_int64), ("workspace_bytes", c_int64),
                ("tail_grid_x", c_int32), ("tail_grid_y", c_int32), ("reserved", c_int32 * 4)]


class xtc_measure_cfg(Structure):
    _fields_ = [("warmup", c_int32), ("repeats", c_int32), ("flush_l2", c_int32), ("validate", c_int32),
                ("exact", c_int32), ("reuse_reference", c_int32), ("tol", c_double), ("peak_tflops", c_double),
                ("counters", ctypes.c_char_p)]


class xtc_metrics(Structure):
    _fields_ = [("status", c_int32), ("valid", c_int32), ("max_norm_err", c_double), ("n_mismatch", c_int64),
                ("n_nan", c_int64), ("err_row", c_int64), ("err_col", c_int64),
                ("t_min_ns", c_double), ("t_med_ns", c_double), ("t_mean_ns", c_double), ("t_max_ns", c_double),
                ("tflops_med", c_double), ("tflops_min", c_double), ("frac_peak", c_double),
                ("sm_clock_mhz", c_double), ("n_reps", c_int32), ("n_counters", c_int32), ("counters", c_double * 8)]

    def as_dict(self):
        return {f: (getattr(self, f) if not isinstance(getattr(self, f), ctypes.Array) else None)
                for f, _ in self._fields_ if not f.startswith("reserved")}

    def counter_values(self, names) -> dict:
        """{name: value} for the names passed in measure_cfg(counters=...); {} if CUPTI was
        unavailable (n_counters == -1) or none were requested."""
        names = _counter_names(names)
        return {n: self.counters[i] for i, n in enumerate(names[:max(self.n_counters, 0)])}


def _counter_names(names) -> list:
    if not names:
        return []
    if isinstance(names, str):
        names = names.split(",")
    return [n.strip() for n in names if n.strip()]


xtc_op = c_void_p

# ------------------------------------------------------------- loading -----
_lib = None


class XtcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libxtc.so (built in-tree by __graft_entry__.build()).  No fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(the CUDA path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = POINTER
        L.xtc_op_create.argtypes = [P(xtc_op_desc), c_int32, P(xtc_op)]
        L.xtc_op_destroy.argtypes = [xtc_op]
        L.xtc_op_destroy.restype = None
        L.xtc_schedule_check.argtypes = [P(xtc_op_desc), P(xtc_schedule), c_int32, P(xtc_plan_info)]
        L.xtc_schedule_apply.argtypes = [xtc_op, P(xtc_schedule)]
        L.xtc_schedule_default.argtypes = [P(xtc_op_desc), c_int32, P(xtc_schedule)]
        L.xtc_run.argtypes = [xtc_op, P(c_void_p), P(c_void_p), c_void_p]
        L.xtc_run_gather.argtypes = [xtc_op, P(c_void_p), P(c_void_p), c_int32, c_int64, c_int64, c_void_p]
        L.xtc_run_multicast.argtypes = [xtc_op, P(c_void_p), c_void_p, c_int64, c_int64, c_int32, c_void_p]
        L.xtc_measure.argtypes = [xtc_op, P(c_void_p), P(c_void_p), P(xtc_measure_cfg), P(xtc_metrics), c_void_p]
        L.xtc_sweep.argtypes = [xtc_op, P(xtc_schedule), c_int32, P(c_void_p), P(c_void_p), P(xtc_measure_cfg),
                                P(xtc_metrics), c_void_p]
        L.xtc_fill.argtypes = [c_void_p, c_int64, c_int32, c_uint64, c_int32, c_int64, c_void_p]
        L.xtc_op_flops.argtypes = [P(xtc_op_desc)]
        L.xtc_op_flops.restype = c_double
        L.xtc_op_min_bytes.argtypes = [P(xtc_op_desc)]
        L.xtc_op_min_bytes.restype = c_double
        L.xtc_last_launch_count.argtypes = [xtc_op]
        L.xtc_last_launch_count.restype = c_int32
        L.xtc_last_error.restype = c_char_p
        L.xtc_abi_sizes.argtypes = [P(c_int64)]
        L.xtc_abi_sizes.restype = None
        for name in ("xtc_op_create", "xtc_schedule_check", "xtc_schedule_apply", "xtc_schedule_default",
                     "xtc_run", "xtc_run_gather", "xtc_measure", "xtc_sweep", "xtc_fill"):
            getattr(L, name).restype = c_int32
        sizes = (c_int64 * 5)()
        L.xtc_abi_sizes(sizes)
        ours = [ctypes.sizeof(t) for t in (xtc_op_desc, xtc_schedule, xtc_plan_info, xtc_measure_cfg, xtc_metrics)]
        if list(sizes) != ours:
            raise ImportError(f"libxtc struct sizes {list(sizes)} != binding {ours}: rebuild")
        _lib = L
    return _lib


def xtc_last_error() -> str:
    return lib().xtc_last_error().decode()


def _check(status):
    if status != XTC_OK:
        raise XtcError(status, xtc_last_error())
    return status


# ---------------------------------------------------- C-named functions ----
def xtc_op_create(desc: xtc_op_desc, device: int = 0) -> c_void_p:
    h = xtc_op()
    _check(lib().xtc_op_create(byref(desc), device, byref(h)))
    return h


def xtc_op_destroy(op) -> None:
    lib().xtc_op_destroy(op)


def xtc_schedule_check(desc: xtc_op_desc, sch: xtc_schedule, num_sms: int = 148):
    """Returns (status, plan_info, reason) without raising."""
    info = xtc_plan_info()
    st = lib().xtc_schedule_check(byref(desc), byref(sch), num_sms, byref(info))
    return st, info, ("" if st == XTC_OK else xtc_last_error())


def xtc_schedule_apply(op, sch: xtc_schedule) -> None:
    _check(lib().xtc_schedule_apply(op, byref(sch)))


def xtc_schedule_default(desc: xtc_op_desc, opt_level: int = 2) -> xtc_schedule:
    s = xtc_schedule()
    _check(lib().xtc_schedule_default(byref(desc), opt_level, byref(s)))
    return s


def _ptrs(ptrs):
    arr = (c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def xtc_run(op, inputs, outputs, stream=0) -> None:
    _check(lib().xtc_run(op, _ptrs(inputs), _ptrs(outputs), c_void_p(stream)))


def xtc_run_gather(op, inputs, dests, row_offset, dest_rows, stream=0) -> None:
    """xtc_run of an M-shard whose output tiles are TMA-stored to every pointer in ``dests``
    (the all-gather fused into the epilogue; include/xtc.h)."""
    _check(lib().xtc_run_gather(op, _ptrs(inputs), _ptrs(dests), len(dests), row_offset, dest_rows,
                                c_void_p(stream)))


def xtc_run_multicast(op, inputs, dest, row_offset, dest_rows, multimem, stream=0) -> None:
    _check(lib().xtc_run_multicast(op, _ptrs(inputs), c_void_p(dest), c_int64(row_offset), c_int64(dest_rows),
                                   c_int32(int(multimem)), c_void_p(stream)))


def xtc_measure(op, inputs, outputs, cfg: xtc_measure_cfg, stream=0) -> xtc_metrics:
    m = xtc_metrics()
    st = lib().xtc_measure(op, _ptrs(inputs), _ptrs(outputs), byref(cfg), byref(m), c_void_p(stream))
    if st not in (XTC_OK, XTC_E_VALIDATION_FAILED):
        _check(st)
    return m


def xtc_sweep(op, cands, inputs, outputs, cfg: xtc_measure_cfg, stream=0):
    n = len(cands)
    arr = (xtc_schedule * n)(*cands)
    out = (xtc_metrics * n)()
    _check(lib().xtc_sweep(op, arr, n, _ptrs(inputs), _ptrs(outputs), byref(cfg), out, c_void_p(stream)))
    return list(out)


def xtc_fill(ptr, count, dtype, seed, mode=0, first=0, stream=0) -> None:
    _check(lib().xtc_fill(c_void_p(ptr), count, dtype, seed, mode, first, c_void_p(stream)))


def xtc_op_flops(desc) -> float:
    return lib().xtc_op_flops(byref(desc))


def xtc_op_min_bytes(desc) -> float:
    return lib().xtc_op_min_bytes(byref(desc))


def xtc_last_launch_count(op) -> int:
    return int(lib().xtc_last_launch_count(op))


# ------------------------------------------------------------ helpers ------
def matmul_desc(m, n, k, in_dtype="bf16", out_dtype="bf16", lda=0, ldb=0, ldc=0, consumer=None) -> xtc_op_desc:
    d = xtc_op_desc()
    d.kind = XTC_OP_MATMUL
    d.in_dtype = DTYPES[in_dtype]
    d.out_dtype = DTYPES[out_dtype]
    d.consumer = consumer_bits(consumer)
    d.m, d.n, d.k, d.lda, d.ldb, d.ldc = m, n, k, lda, ldb, ldc
    return d


def conv2d_desc(batch, h, w, c, f, r=3, s=3, stride=1, pad=1, in_dtype="bf16", out_dtype="bf16",
                consumer=None) -> xtc_op_desc:
    d = xtc_op_desc()
    d.kind = XTC_OP_CONV2D
    d.in_dtype = DTYPES[in_dtype]
    d.out_dtype = DTYPES[out_dtype]
    d.consumer = consumer_bits(consumer)
    d.batch, d.h, d.w, d.c, d.f, d.r, d.s = batch, h, w, c, f, r, s
    d.stride_h = d.stride_w = stride
    d.pad_h = d.pad_w = pad
    return d


def gemm_view(d: xtc_op_desc):
    if d.kind == XTC_OP_CONV2D:
        P = (d.h + 2 * d.pad_h - d.r) // d.stride_h + 1
        Q = (d.w + 2 * d.pad_w - d.s) // d.stride_w + 1
        return d.batch * P * Q, d.f, d.r * d.s * d.c
    return d.m, d.n, d.k


def schedule(**kw) -> xtc_schedule:
    s = xtc_schedule()
    for k, v in kw.items():
        if k not in SCHEDULE_FIELDS:
            raise KeyError(k)
        setattr(s, k, int(v))
    return s


def measure_cfg(warmup=2, repeats=10, flush_l2=0, validate=1, exact=0, reuse_reference=0, tol=0.0,
                peak_tflops=0.0, counters=None) -> xtc_measure_cfg:
    """counters: None, a comma-separated string or a list of metric names (optionally
    "gpu."-prefixed), collected in a separate CUPTI pass after the timed reps."""
    c = xtc_measure_cfg()
    c.warmup, c.repeats, c.flush_l2, c.validate, c.exact, c.reuse_reference = (
        warmup, repeats, flush_l2, validate, exact, reuse_reference)
    c.tol, c.peak_tflops = tol, peak_tflops
    names = _counter_names(counters)
    c.counters = ",".join(names).encode() if names else None
    return c


class Op:
    """RAII wrapper: Op(desc, device).apply(sched); op.run(a, b, c); op.measure(...)."""

    def __init__(self, desc: xtc_op_desc, device: int = 0):
        self.desc = desc
        self.device = device
        self.handle = xtc_op_create(desc, device)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                xtc_op_destroy(h)
            except Exception:
                pass
            self.handle = None

    def apply(self, sch: xtc_schedule) -> "Op":
        xtc_schedule_apply(self.handle, sch)
        return self

    @staticmethod
    def _stream(stream):
        if stream is not None:
            return stream
        import torch
        return torch.cuda.current_stream().cuda_stream

    @staticmethod
    def _inputs(a, b, bias):
        # inputs[2] = the fp32 bias of an XTC_CONSUMER_BIAS consumer (include/xtc.h)
        return [a.data_ptr(), b.data_ptr()] + ([bias.data_ptr()] if bias is not None else [None])

    def run(self, a, b, c, stream=None, bias=None) -> None:
        xtc_run(self.handle, self._inputs(a, b, bias), [c.data_ptr()], self._stream(stream))

    def run_gather(self, a, b, dests, row_offset, dest_rows, stream=None, bias=None) -> None:
        """dests: device pointers (ints) of [dest_rows][N] outputs, local or peer-mapped."""
        xtc_run_gather(self.handle, self._inputs(a, b, bias), list(dests), row_offset, dest_rows,
                       self._stream(stream))

    def run_multicast(self, a, b, dest, row_offset, dest_rows, multimem=False, stream=None, bias=None) -> None:
        """dest: an int device address -- an NVLS multicast address (multimem=True) or a plain pointer."""
        xtc_run_multicast(self.handle, self._inputs(a, b, bias), int(dest), row_offset, dest_rows, multimem,
                          self._stream(stream))

    def measure(self, a, b, c, cfg: xtc_measure_cfg = None, stream=None, bias=None) -> xtc_metrics:
        cfg = cfg or measure_cfg()
        return xtc_measure(self.handle, self._inputs(a, b, bias), [c.data_ptr()], cfg, self._stream(stream))

    def sweep(self, cands, a, b, c, cfg: xtc_measure_cfg = None, stream=None, bias=None):
        cfg = cfg or measure_cfg()
        return xtc_sweep(self.handle, cands, self._inputs(a, b, bias), [c.data_ptr()], cfg, self._stream(stream))

    def launches(self) -> int:
        return xtc_last_launch_count(self.handle)
