"""Analytical traffic model of a schedule (the GPU analogue of the paper's
§VI-C cache-model study, where XTC's hardware-counter instrumentation is used
to check a model's predictions across schedule instances).

The paper's model predicts L1 misses of a CPU loop nest from a fully associative cache.  On
the tcgen05 engine the SM-local level is the SMEM ring fed by TMA, so the quantity the
schedule controls is the traffic between L2 and the SMs:

* operand loads: every output tile streams its K-range of A (tile_m rows) and of B
  (tile_n columns) once — M*N*K*s_in*(1/tile_n + 1/tile_m) for exact tiles (ragged edges
  load whole boxes: tile counts are rounded up); a CTA pair loads 256 rows of A and
  tile_n columns of B per pair tile, i.e. the same formula with tile_m = 256;
* output writes: M*N*s_out (TMA store or direct stores);
* split-K (ordered): S fp32 partial planes written and read back by the reduction, then
  the output; atomic split-K: S fp32 read-modify-writes of C.

Only the schedule's knobs and the descriptor enter; nothing is fitted.  The counters it is
compared with are collected by `xtc_measure(counters=...)` (CUPTI), see tools/model_study.py.
"""
from __future__ import annotations

import math
from typing import Dict

from . import XTC_BF16, XTC_SPLITK_ATOMIC, gemm_view, xtc_op_desc, xtc_schedule


def _es(dtype: int) -> int:
    return 2 if dtype == XTC_BF16 else 4


def predicted_l2_bytes(desc: xtc_op_desc, s: xtc_schedule) -> Dict[str, float]:
    """Bytes moved between L2 and the SMs by one run of `s` on `desc` (tcgen05 matmul)."""
    M, N, K = gemm_view(desc)
    es, os_ = _es(desc.in_dtype), _es(desc.out_dtype)
    tile_m = s.tile_m or 128
    tm, tn = math.ceil(M / tile_m), math.ceil(N / s.tile_n)
    kb = math.ceil(K / s.tile_k)
    split = max(1, s.split_k)
    kb_seg = math.ceil(kb / split)
    # every (tile, segment) loads its k-blocks of A and B; boxes are whole tiles
    seg_kb = [min(kb, (i + 1) * kb_seg) - i * kb_seg for i in range(split)]
    k_loaded = sum(max(0, x) for x in seg_kb) * s.tile_k
    loads = tm * tn * k_loaded * (tile_m + s.tile_n) * es
    out = M * N * os_
    if split > 1 and s.split_k_mode == XTC_SPLITK_ATOMIC:
        partial = 2.0 * split * M * N * 4          # red.global: read + write of C per segment
        out = 0.0
    elif split > 1:
        partial = 2.0 * split * M * N * 4          # workspace planes written, then read by the reduction
    else:
        partial = 0.0
    return {"loads": float(loads), "outputs": float(out), "partials": partial,
            "total": float(loads) + float(out) + partial}
