"""-m gpu: the warp-MMA engine (XTC_ENGINE_MMA, csrc/conv_mma.cu): mma.sync m16n8k16 bf16 tensor-core
tiles over an im2col gather, for operands TMA cannot address -- above all the paper's stem conv
"[112,112,16] x [7,7,3] step 2" (DESIGN reading 4: 224x224x3 input, 7x7 filter, stride 2,
pad 3, F = 16; K = 147, a 6-byte pixel).  Element-by-element parity with the CPU oracle: bit-exact on
integer data, <= 5e-3 of D on uniform data; ragged M / N / K, stride / pad variants, fused consumers,
fp32 and bf16 output, matmul through the same kernel, persistent grids.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, MODE_UNIFORM
from gpu_util import TORCH_DT, check_against_oracle, dev_tensor, oracle_conv, run_conv, run_matmul

pytestmark = pytest.mark.gpu
S = xtc.schedule
MODES = [MODE_INT, MODE_UNIFORM]


def mma(**kw):
    base = dict(engine=xtc.XTC_ENGINE_MMA, tile_m=128, tile_n=16, tile_k=32)
    base.update(kw)
    return S(**base)


CONV_CASES = [
    # (name, (N, H, W, C, F, R, S, stride, pad), schedule, out)
    ("stem-paper-n1", (1, 224, 224, 3, 16, 7, 7, 2, 3), mma(), "bf16"),
    ("stem-paper-n2-f32-persistent", (2, 224, 224, 3, 16, 7, 7, 2, 3), mma(persistent=1, tile_k=16), "f32"),
    ("stem-tile64-k64", (1, 64, 96, 3, 16, 7, 7, 2, 3), mma(tile_m=64, tile_k=64), "bf16"),
    ("c5-f24-ragged", (2, 19, 23, 5, 24, 3, 3, 1, 1), mma(tile_n=32), "bf16"),
    ("c8-f40-stride3", (1, 30, 31, 8, 40, 5, 5, 3, 2), mma(tile_n=64), "f32"),
    ("c64-f64-3x3", (1, 14, 14, 64, 64, 3, 3, 1, 1), mma(tile_n=64, tile_k=64), "bf16"),
]


def patch(**kw):
    """pack_halo = 1: the patch-staged kernel (tile_m / Q whole output rows per CTA, K resident), the
    input patch loaded by one TMA per tile where the layout allows; pack_halo = 2: filled by the threads."""
    base = dict(pack_halo=1, tile_k=16)
    base.update(kw)
    return mma(**base)


CONV_CASES += [
    ("patch-stem-n1-tp1", (1, 224, 224, 3, 16, 7, 7, 2, 3), patch(), "bf16"),
    ("patch-stem-n2-tp2-f32-persistent", (2, 224, 224, 3, 16, 7, 7, 2, 3), patch(tile_m=256, persistent=1), "f32"),
    ("patch-stem-ragged-p-tp4", (2, 100, 224, 3, 16, 7, 7, 2, 3), patch(tile_m=512), "bf16"),
    ("patch-stem-persistent-grid3", (1, 64, 96, 3, 16, 7, 7, 2, 3), patch(tile_m=256, persistent=1, grid_sms=3), "bf16"),
    ("patch-c1-5x5", (2, 28, 28, 1, 32, 5, 5, 1, 2), patch(tile_n=32), "bf16"),
    ("patch-c3-3x3-s1-ragged", (1, 33, 37, 3, 16, 3, 3, 1, 1), patch(tile_m=64), "f32"),
    ("patch-c5-f24-ragged-n", (2, 19, 23, 5, 24, 3, 3, 1, 1), patch(tile_n=32), "bf16"),
    ("patch-c8-f40-stride3", (1, 30, 31, 8, 40, 5, 5, 3, 2), patch(tile_n=64), "f32"),
    ("patch-c16-f48-two-n-tiles", (1, 20, 20, 16, 48, 3, 3, 1, 1), patch(tile_n=32, tile_m=256), "bf16"),
    # TMA patch layout (sw*C even, W*C % 16 == 0) -- the stem cases above take it; these force or avoid it
    ("tma-c8-s1-two-n-tiles-persistent", (2, 17, 18, 8, 40, 3, 3, 1, 1), patch(tile_n=32, persistent=1, grid_sms=2), "f32"),
    ("tma-c16-5x5-pad2-ragged-p", (1, 21, 24, 16, 16, 5, 5, 1, 2), patch(tile_m=64), "bf16"),
    ("tma-c4-stride2-pad0", (2, 31, 36, 4, 24, 3, 3, 2, 0), patch(tile_n=32, tile_m=256), "bf16"),
    ("tma-c2-7x7-pad3-wide-row", (1, 12, 480, 2, 16, 7, 7, 2, 3), patch(), "bf16"),
    ("thread-filled-stem-n2", (2, 224, 224, 3, 16, 7, 7, 2, 3), patch(pack_halo=2, tile_m=512), "bf16"),
    ("thread-filled-c16-persistent", (2, 20, 20, 16, 48, 3, 3, 1, 1), patch(pack_halo=2, tile_n=64, persistent=1,
                                                                             grid_sms=3), "f32"),
]


@pytest.mark.parametrize("case", CONV_CASES, ids=[c[0] for c in CONV_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_mma_engine_conv_vs_oracle(case, mode):
    _, (n, h, w, c, f, r, s, st, pd), sch, out = case
    d = xtc.conv2d_desc(n, h, w, c, f, r, s, st, pd, "bf16", out)
    run_conv(d, "bf16", out, sch, mode, seed=91)


@pytest.mark.parametrize("shape", [(256, 64, 128), (300, 40, 72), (129, 16, 1000)])
@pytest.mark.parametrize("mode", MODES)
def test_mma_engine_matmul_vs_oracle(shape, mode):
    M, N, K = shape
    err, _ = run_matmul(M, N, K, "bf16", "f32", mma(tile_n=64 if N > 32 else 16), mode, seed=93)
    assert err <= 5e-3


@pytest.mark.parametrize("pk", [0, 1])
@pytest.mark.parametrize("cons", ["relu", "bias", "accumulate+bias+relu"])
def test_mma_engine_stem_fused_consumers(cons, pk):
    d = xtc.conv2d_desc(1, 224, 224, 3, 16, 7, 7, 2, 3, "bf16", "f32", consumer=cons)
    M, N, K = xtc.gemm_view(d)
    x = dev_tensor((1, 224, 224, 3), "bf16", 95, MODE_INT)
    w = dev_tensor((7, 7, 3, 16), "bf16", 96, MODE_INT)
    bias = dev_tensor((16,), "f32", 97, MODE_INT)
    y = dev_tensor((M, N), "f32", 98, MODE_INT)
    y_old = y.double().cpu().numpy()
    xtc.Op(d).apply(patch(fuse=1, tile_m=256) if pk else mma(fuse=1)).run(x, w, y, bias=bias)
    torch.cuda.synchronize()
    O, D = oracle_conv(d, "bf16", MODE_INT, 95, 96)
    O = O.copy()
    if "accumulate" in cons:
        O += y_old
    if "bias" in cons:
        O += bias.double().cpu().numpy()[None, :]
    if "relu" in cons:
        O = np.maximum(O, 0.0)
    check_against_oracle(y, O, D, "f32", exact=True, tol=0)
