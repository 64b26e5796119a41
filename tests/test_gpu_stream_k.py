"""-m gpu: stream-K (split_k_mode 3, csrc/stream_k.cuh) -- the split primitive applied to
the flattened (output tile, k-block) loop, with split points given by the persistent grid: CTA g of G
owns iterations [floor(I g / G), floor(I (g+1) / G)), I = tiles x k-blocks, so ranges start and end
inside tiles; the CTA whose range holds a tile's first k-blocks adds the partials of the CTAs holding
the rest, in ascending k order.

Element-by-element parity with the CPU oracle: bit-exact on integer data, <= 5e-3 of D on uniform data.
The cases force every shape of split: tiles cut in two, tiles spread over 3-6 CTAs (an owner waiting
for several contributors, CTAs whose whole range lies inside one tile), fewer iterations than SMs,
few SMs (grid_sms) so that every CTA crosses many tiles, ragged M / N / K, fused consumers, fp32 and
bf16 output, tf32 and 3xTF32, and both conv kernels (TMA im2col, haloed patch incl. two M-subtiles).
Repeated launches must agree bit for bit (the owner's summation order is fixed).
"""
import numpy as np
import pytest
import torch

import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, MODE_UNIFORM
from gpu_util import TORCH_DT, check_against_oracle, dev_tensor, oracle_matmul, run_conv, run_matmul, to_numpy_out

pytestmark = pytest.mark.gpu
S = xtc.schedule
SK = xtc.XTC_SPLITK_STREAM
MODES = [MODE_INT, MODE_UNIFORM]


def mm(**kw):
    base = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, swizzle=128, buffer_c=1, acc_buffers=2,
                persistent=1, split_k_mode=SK)
    base.update(kw)
    return base


def plan(desc, sch):
    st, info, why = xtc.xtc_schedule_check(desc, S(**sch), 148)
    assert st == xtc.XTC_OK, why
    return info


MATMUL_CASES = [
    # (name, schedule, M, N, K, in, out); I = tiles x k-blocks vs the grid G
    ("two-cuts-per-tile", mm(grid_sms=3), 256, 256, 512, "bf16", "bf16"),            # I=32, G=3
    ("six-ctas-per-tile", mm(grid_sms=12), 256, 256, 768, "bf16", "bf16"),           # I=48, G=12: 4 kb each
    ("fewer-iters-than-sms", mm(), 256, 128, 256, "bf16", "bf16"),                   # I=8 -> G=8
    ("wave-remainder-148", mm(tile_n=64), 1280, 960, 576, "bf16", "bf16"),            # 150 tiles x 9 kb on 148
    ("ragged-mnk", mm(grid_sms=7), 300, 200, 520, "bf16", "f32"),
    ("direct-stores", mm(buffer_c=0, grid_sms=5), 384, 320, 640, "bf16", "bf16"),
    ("acc1", mm(acc_buffers=1, grid_sms=4), 512, 384, 384, "bf16", "bf16"),
    ("tf32", mm(tile_k=32, grid_sms=6), 256, 256, 384, "tf32", "f32"),
    ("3xtf32", mm(tile_k=32, stages=3, grid_sms=5), 256, 256, 320, "f32", "f32"),
    ("tile256", mm(tile_n=256, stages=3, grid_sms=9), 384, 512, 512, "bf16", "bf16"),
]


@pytest.mark.parametrize("case", MATMUL_CASES, ids=[c[0] for c in MATMUL_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_matmul_stream_k_vs_oracle(case, mode):
    _, sch, M, N, K, idt, odt = case
    plan(xtc.matmul_desc(M, N, K, idt, odt), sch)
    tol = 1e-5 if idt == "f32" else 5e-3
    err, _ = run_matmul(M, N, K, idt, odt, S(**sch), mode, seed=8, tol=tol)
    assert err <= tol


def test_stream_k_repeated_launches_are_bit_identical():
    M, N, K = 640, 384, 832
    desc = xtc.matmul_desc(M, N, K, "bf16", "f32")
    a = dev_tensor((M, K), "bf16", 3, MODE_UNIFORM)
    b = dev_tensor((K, N), "bf16", 4, MODE_UNIFORM)
    op = xtc.Op(desc).apply(S(**mm(grid_sms=11)))
    outs = []
    for _ in range(3):
        c = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda:0")
        op.run(a, b, c)
        torch.cuda.synchronize()
        assert op.launches() == 1
        outs.append(to_numpy_out(c, "f32"))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    assert np.array_equal(outs[0].view(np.uint32), outs[2].view(np.uint32))


@pytest.mark.parametrize("cons", ["relu", "bias", "accumulate", "accumulate+bias+relu"])
def test_stream_k_fused_consumers(cons):
    """Owned tiles apply relu(C_old + sum of all k-ranges + bias) once, after the partials are added."""
    M, N, K = 384, 256, 704
    desc = xtc.matmul_desc(M, N, K, "bf16", "f32", consumer=cons)
    a = dev_tensor((M, K), "bf16", 71, MODE_INT)
    b = dev_tensor((K, N), "bf16", 72, MODE_INT)
    bias = dev_tensor((N,), "f32", 73, MODE_INT)
    c = dev_tensor((M, N), "f32", 74, MODE_INT)
    c_old = c.double().cpu().numpy()
    xtc.Op(desc).apply(S(**mm(grid_sms=7, fuse=1))).run(a, b, c, bias=bias)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", MODE_INT, 71, 72)
    O = O.copy()
    if "accumulate" in cons:
        O += c_old
    if "bias" in cons:
        O += bias.double().cpu().numpy()[None, :]
    if "relu" in cons:
        O = np.maximum(O, 0.0)
    check_against_oracle(c, O, D, "f32", exact=True, tol=0)


HALO = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, pack_halo=1, buffer_c=1, acc_buffers=2, persistent=1,
            split_k_mode=SK)
IM2COL = dict(engine=1, tile_m=128, tile_k=64, stages=4, swizzle=128, buffer_c=1, acc_buffers=2, persistent=1,
              split_k_mode=SK)
CONV_CASES = [
    # (name, (N, H, W, C, F, R, S, stride, pad), schedule)
    ("halo-L56-n2-wave", (2, 56, 56, 64, 64, 3, 3, 1, 1), dict(HALO, tile_n=64, stages=2, b_resident=1)),
    ("halo-L56-n1-few-sms", (1, 56, 56, 64, 64, 3, 3, 1, 1), dict(HALO, tile_n=64, stages=2, grid_sms=9)),
    ("halo-L14-n2", (2, 14, 14, 256, 256, 3, 3, 1, 1), dict(HALO, tile_n=128, tile_k=128, stages=3, grid_sms=10)),
    ("halo-msub2-direct", (2, 28, 28, 64, 64, 3, 3, 1, 1), dict(HALO, tile_m=256, tile_n=64, stages=2, buffer_c=0,
                                                               grid_sms=6)),
    ("halo-ragged", (2, 11, 13, 128, 96, 3, 3, 1, 1), dict(HALO, tile_n=64, stages=3, buffer_c=0, grid_sms=5)),
    ("im2col-L14-n1", (1, 14, 14, 256, 256, 3, 3, 1, 1), dict(IM2COL, tile_n=128, grid_sms=12)),
    ("im2col-stride2", (2, 15, 17, 64, 128, 3, 3, 2, 1), dict(IM2COL, tile_n=64, grid_sms=7)),
]


@pytest.mark.parametrize("case", CONV_CASES, ids=[c[0] for c in CONV_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_conv_stream_k_vs_oracle(case, mode):
    _, (n, h, w, c, f, r, s, st, pd), sch = case
    d = xtc.conv2d_desc(n, h, w, c, f, r, s, st, pd, "bf16", "bf16")
    plan(d, sch)
    run_conv(d, "bf16", "bf16", S(**sch), mode, seed=43)
