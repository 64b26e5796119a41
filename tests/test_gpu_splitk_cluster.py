"""-m gpu: split with the reduction inside the contraction kernel, split_k_mode 2
(XTC_SPLITK_CLUSTER, csrc/splitk_cluster.cuh): the split_k K segments of an output tile are the CTAs
of one thread-block cluster, and after all partials are written each CTA sums 1/split_k of the tile's
rows in ascending segment order.

Parity, element by element against the CPU oracle: bit-exact on integer data, <= 5e-3 of D on uniform
data (1e-5 for the 3xTF32 fp32 path).  Because the in-kernel reduction adds the partials in the order
of the separate reduction kernel (W[0] + W[1] + ...), the two modes must also agree BIT FOR BIT on
uniform data -- a second, stronger check that the segments, their order and the rows each CTA reduces
are right.  Cases cover ragged M / N / K, empty-row CTAs (rows < split_k), 2..16 segments (> 8 is a
non-portable cluster size), persistent clusters that stride over several tiles (the two alternating
signal barriers), the fused consumers, fp32 / bf16 output, tf32 and 3xTF32 inputs, and both conv
kernels (TMA im2col and the tile-level haloed patch).
"""
import numpy as np
import pytest
import torch

import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, MODE_UNIFORM
from gpu_util import (TORCH_DT, check_against_oracle, dev_tensor, oracle_conv, oracle_matmul, run_conv,
                      run_matmul, to_numpy_out)

pytestmark = pytest.mark.gpu
S = xtc.schedule
MODES = [MODE_INT, MODE_UNIFORM]


def mm(**kw):
    base = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, swizzle=128, buffer_c=0, acc_buffers=2,
                split_k_mode=xtc.XTC_SPLITK_CLUSTER)
    base.update(kw)
    return base


def plan(desc, sch):
    st, info, why = xtc.xtc_schedule_check(desc, S(**sch), 148)
    assert st == xtc.XTC_OK, why
    return info


MATMUL_CASES = [
    # (name, schedule, M, N, K, in, out)
    ("s2", mm(split_k=2), 256, 256, 512, "bf16", "bf16"),
    ("s3-ragged", mm(split_k=3), 300, 200, 520, "bf16", "bf16"),
    ("s8-512cube", mm(tile_n=64, tile_k=64, split_k=8), 512, 512, 512, "bf16", "bf16"),
    ("s3-uneven-segments", mm(split_k=3, tile_k=64), 256, 384, 448, "bf16", "f32"),
    ("s16-nonportable", mm(tile_n=64, split_k=16), 256, 128, 1024, "bf16", "bf16"),
    ("s5-rows-lt-128", mm(split_k=5), 40, 136, 640, "bf16", "bf16"),
    ("s4-persistent-multitile", mm(split_k=4, persistent=1, grid_sms=8), 640, 512, 512, "bf16", "bf16"),
    ("s2-persistent-acc1", mm(split_k=2, acc_buffers=1, persistent=1, grid_sms=4), 512, 640, 384, "bf16", "bf16"),
    ("s4-tf32", mm(tile_k=32, split_k=4), 256, 256, 512, "tf32", "f32"),
    ("s2-3xtf32", mm(tile_k=32, stages=3, split_k=2), 256, 256, 256, "f32", "f32"),
    ("s8-tile256", mm(tile_n=256, stages=3, split_k=8), 256, 512, 1024, "bf16", "bf16"),
    # partials staged in SMEM and written by TMA stores (buffer_c 1), completed before the signal
    ("s4-tma-partials", mm(split_k=4, buffer_c=1), 300, 256, 512, "bf16", "bf16"),
    ("s3-tma-partials-persistent", mm(split_k=3, buffer_c=1, tile_n=64, persistent=1, grid_sms=6), 512, 320, 576,
     "bf16", "f32"),
]


@pytest.mark.parametrize("case", MATMUL_CASES, ids=[c[0] for c in MATMUL_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_matmul_cluster_split_vs_oracle(case, mode):
    _, sch, M, N, K, idt, odt = case
    info = plan(xtc.matmul_desc(M, N, K, idt, odt), sch)
    assert info.cluster_x == sch["split_k"]
    tol = 1e-5 if idt == "f32" else 5e-3
    err, m = run_matmul(M, N, K, idt, odt, S(**sch), mode, seed=5, tol=tol)
    assert err <= tol


def _run(desc, sch, a, b, out_dt, shape, bias=None, c_init=None, launches=1):
    c = (c_init.clone() if c_init is not None
         else torch.full(shape, float("nan"), dtype=TORCH_DT[out_dt], device="cuda:0"))
    op = xtc.Op(desc).apply(S(**sch))
    op.run(a, b, c, bias=bias)
    torch.cuda.synchronize()
    assert op.launches() == launches          # the reduction runs inside the contraction kernel
    return c


@pytest.mark.parametrize("case", [c for c in MATMUL_CASES if c[5] != "f32"], ids=[c[0] for c in MATMUL_CASES
                                                                               if c[5] != "f32"])
def test_cluster_split_bitwise_equals_ordered_reduction(case):
    """Same partials, same summation order: split_k_mode 2 == split_k_mode 0, bit for bit (uniform data)."""
    _, sch, M, N, K, idt, odt = case
    desc = xtc.matmul_desc(M, N, K, idt, odt)
    a = dev_tensor((M, K), idt, 21, MODE_UNIFORM)
    b = dev_tensor((K, N), idt, 22, MODE_UNIFORM)
    got = _run(desc, sch, a, b, odt, (M, N))
    ordered = dict(sch, split_k_mode=xtc.XTC_SPLITK_ORDERED)
    ordered.pop("grid_sms", None)
    ordered.pop("persistent", None)
    want = _run(desc, ordered, a, b, odt, (M, N), launches=2)
    assert np.array_equal(to_numpy_out(got, odt), to_numpy_out(want, odt))


@pytest.mark.parametrize("cons", ["relu", "bias", "accumulate", "accumulate+bias+relu"])
@pytest.mark.parametrize("out_dt", ["bf16", "f32"])
def test_cluster_split_fused_consumers(cons, out_dt):
    """relu(C_old + A*B + bias) applied once, to the complete sums, in the in-kernel reduction."""
    M, N, K = 264, 192, 640
    sch = mm(split_k=5, tile_n=64, fuse=1)
    desc = xtc.matmul_desc(M, N, K, "bf16", out_dt, consumer=cons)
    a = dev_tensor((M, K), "bf16", 31, MODE_INT)
    b = dev_tensor((K, N), "bf16", 32, MODE_INT)
    bias = dev_tensor((N,), "f32", 33, MODE_INT)
    c0 = dev_tensor((M, N), out_dt, 34, MODE_INT)
    got = _run(desc, sch, a, b, out_dt, (M, N), bias=bias, c_init=c0)
    O, D = oracle_matmul(M, N, K, "bf16", MODE_INT, 31, 32)
    O = O.copy()
    if "accumulate" in cons:
        O += c0.double().cpu().numpy()
    if "bias" in cons:
        O += bias.double().cpu().numpy()[None, :]
    if "relu" in cons:
        O = np.maximum(O, 0.0)
    check_against_oracle(got, O, D, out_dt, exact=True, tol=0)


HALO = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, pack_halo=1, buffer_c=0, acc_buffers=2,
            split_k_mode=xtc.XTC_SPLITK_CLUSTER)
IM2COL = dict(engine=1, tile_m=128, tile_k=64, stages=4, swizzle=128, buffer_c=0, acc_buffers=2,
              split_k_mode=xtc.XTC_SPLITK_CLUSTER)
CONV_CASES = [
    # (name, (N, H, W, C, F, R, S, stride, pad), schedule)
    ("halo-L14-n1-s9", (1, 14, 14, 256, 256, 3, 3, 1, 1), dict(HALO, tile_n=128, tile_k=128, stages=3, split_k=9)),
    ("halo-L14-n2-s6-persistent", (2, 14, 14, 256, 256, 3, 3, 1, 1),
     dict(HALO, tile_n=64, tile_k=128, stages=3, split_k=6, persistent=1, grid_sms=12)),
    ("halo-L56-n1-s3", (1, 56, 56, 64, 64, 3, 3, 1, 1), dict(HALO, tile_n=64, stages=3, split_k=3)),
    ("halo-ragged-s4", (2, 11, 13, 128, 96, 3, 3, 1, 1), dict(HALO, tile_n=64, tile_k=64, stages=3, split_k=4)),
    ("im2col-L14-n1-s8", (1, 14, 14, 256, 256, 3, 3, 1, 1), dict(IM2COL, tile_n=128, split_k=8)),
    ("im2col-stride2-s3", (2, 15, 17, 64, 128, 3, 3, 2, 1), dict(IM2COL, tile_n=64, split_k=3)),
]


@pytest.mark.parametrize("case", CONV_CASES, ids=[c[0] for c in CONV_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_conv_cluster_split_vs_oracle(case, mode):
    _, (n, h, w, c, f, r, s, st, pd), sch = case
    d = xtc.conv2d_desc(n, h, w, c, f, r, s, st, pd, "bf16", "bf16")
    info = plan(d, sch)
    assert info.cluster_x == sch["split_k"]
    run_conv(d, "bf16", "bf16", S(**sch), mode, seed=41)
