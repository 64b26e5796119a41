"""-m gpu: the CUDA path (through the C-ABI) against the CPU oracle."""
import numpy as np
import pytest
import torch

import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, MODE_UNIFORM, gen_tensor
from gpu_util import (TORCH_DT, check_against_oracle, dev_tensor, oracle_conv, oracle_matmul, out_as_f64, run_conv,
                      run_matmul, to_numpy_out)

pytestmark = pytest.mark.gpu

S = xtc.schedule


# ------------------------------------------------------------- generator --
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("mode", [MODE_UNIFORM, MODE_INT])
def test_gpu_generator_matches_seeded_inputs(dtype, mode):
    t = dev_tensor((1000, 37), dtype, 123, mode)
    got = to_numpy_out(t, dtype)
    want = gen_tensor(123, (1000, 37), dtype, mode)
    assert np.array_equal(got.view(np.uint16 if dtype == "bf16" else np.uint32),
                          want.view(np.uint16 if dtype == "bf16" else np.uint32))


# ------------------------------------------------------- config 1 (SIMT) --
CONFIG1 = dict(engine=0, tile_m=8, tile_n=8, tile_k=8, inner_m=1, inner_n=1, unroll_k=1, stages=1, order=0)


@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_config1_fp32_32cube_tile8_ijk(mode):
    err, m = run_matmul(32, 32, 32, "f32", "f32", S(**CONFIG1), mode)
    assert m.t_med_ns > 0


SIMT_SCHEDS = [
    dict(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, unroll_k=4, vector_n=4, stages=2, swizzle=4),
    dict(engine=0, tile_m=32, tile_n=64, tile_k=8, inner_m=2, inner_n=4, unroll_k=2, vector_n=1, stages=1, swizzle=1,
         order=1, raster_group=2),
    dict(engine=0, tile_m=128, tile_n=64, tile_k=32, inner_m=8, inner_n=8, unroll_k=8, vector_n=4, stages=2, swizzle=4,
         persistent=1),
    dict(engine=0, tile_m=16, tile_n=16, tile_k=16, inner_m=1, inner_n=1, unroll_k=4, stages=2, split_k=3),
    dict(engine=0, tile_m=16, tile_n=16, tile_k=16, inner_m=1, inner_n=2, split_k=4, split_k_mode=1),
]


@pytest.mark.parametrize("sch", SIMT_SCHEDS)
def test_simt_schedules_integer_bit_exact(sch):
    run_matmul(200, 136, 328, "f32", "f32", S(**sch), MODE_INT)


@pytest.mark.parametrize("sch", SIMT_SCHEDS[:3])
def test_simt_schedules_float_tolerance(sch):
    err, _ = run_matmul(256, 192, 512, "f32", "f32", S(**sch), MODE_UNIFORM)
    assert err <= 1e-5


def test_paper_fig4_split_j_at_256_remainder():
    """The paper's running example: I=256, J=258, K=512 with J split at 256,
    K1=4, J1=16 register tile: main root SIMT with a
    16-wide thread tile, remainder root [256,258) scalar."""
    sch = S(engine=0, tile_m=16, tile_n=128, tile_k=4, inner_m=1, inner_n=8, unroll_k=4, vector_n=4, stages=1,
            split_n_at=256)
    run_matmul(256, 258, 512, "f32", "f32", sch, MODE_INT)
    run_matmul(256, 258, 512, "f32", "f32", sch, MODE_UNIFORM)


def test_simt_bf16_output():
    run_matmul(96, 80, 64, "f32", "bf16", S(engine=0, tile_m=32, tile_n=16, tile_k=8, inner_m=2, inner_n=2),
               MODE_INT)


# --------------------------------------------------------- tcgen05 bf16 --
def tc(**kw):
    base = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, swizzle=128, buffer_c=1, acc_buffers=1)
    base.update(kw)
    return S(**base)


TC_SCHEDS = [
    dict(),
    dict(tile_n=64, stages=2),
    dict(tile_n=256, stages=3, acc_buffers=2, persistent=1),
    dict(tile_n=192, tile_k=128, stages=2, buffer_c=0),
    dict(tile_n=128, persistent=1, acc_buffers=2, raster_group=4, order=1),
    dict(tile_n=128, split_k=3),
    dict(tile_n=64, split_k=2, buffer_c=0),
]


@pytest.mark.parametrize("sch", TC_SCHEDS)
def test_tc_bf16_integer_bit_exact(sch):
    run_matmul(256, 512, 384, "bf16", "bf16", tc(**sch), MODE_INT)


@pytest.mark.parametrize("sch", TC_SCHEDS[:5])
def test_tc_bf16_f32_out_integer(sch):
    run_matmul(256, 256, 256, "bf16", "f32", tc(**sch), MODE_INT)


def test_tc_bf16_ragged_tails():
    # M, N, K not multiples of the tile: TMA zero-fill on loads, clipping on stores
    run_matmul(300, 328, 200, "bf16", "bf16", tc(tile_n=128), MODE_INT)
    run_matmul(300, 328, 200, "bf16", "f32", tc(tile_n=64, buffer_c=0, persistent=1, acc_buffers=2), MODE_INT)


@pytest.mark.parametrize("size", [512, 1024])
def test_tc_bf16_float_tolerance(size):
    err, m = run_matmul(size, size, size, "bf16", "bf16", tc(tile_n=256, stages=3, acc_buffers=2, persistent=1),
                        MODE_UNIFORM)
    assert err <= 5e-3


def test_tc_atomic_split_k():
    run_matmul(256, 256, 512, "bf16", "f32", tc(tile_n=128, split_k=4, split_k_mode=1, buffer_c=0), MODE_INT)


# ------------------------------------------------- tcgen05 fp32 (3xTF32) --
SPLIT3_SCHEDS = [dict(tile_k=32, tile_n=128, stages=3), dict(tile_k=32, tile_n=256, stages=2, persistent=1,
                                                             acc_buffers=2),
                 dict(tile_k=64, tile_n=64, stages=2, buffer_c=0), dict(tile_k=32, tile_n=128, stages=3, split_k=2)]


@pytest.mark.parametrize("sch", SPLIT3_SCHEDS)
def test_tc_fp32_3xtf32_at_the_fp32_tolerance(sch):
    """fp32 inputs on the tensor cores (a = hi + lo, C = hi*lo + lo*hi + hi*hi) meet the fp32
    bar of BASELINE (max |C - O| / D <= 1e-5), and are bit-exact on integer data."""
    run_matmul(256, 384, 320, "f32", "f32", tc(**sch), MODE_INT)
    err, _ = run_matmul(256, 384, 1024, "f32", "f32", tc(**sch), MODE_UNIFORM, tol=1e-5)
    assert err <= 1e-5


def test_tc_fp32_3xtf32_ragged_and_bf16_out():
    err, _ = run_matmul(300, 328, 200, "f32", "f32", tc(tile_k=32, tile_n=128, stages=3), MODE_UNIFORM, tol=1e-5)
    assert err <= 1e-5
    run_matmul(256, 256, 256, "f32", "bf16", tc(tile_k=32, tile_n=128, stages=3), MODE_INT)


# ---------------------------------------------------------- tcgen05 tf32 --
@pytest.mark.parametrize("sch", [dict(tile_k=32, tile_n=128), dict(tile_k=64, tile_n=96, stages=3, buffer_c=0),
                                 dict(tile_k=32, tile_n=256, persistent=1, acc_buffers=2)])
def test_tc_tf32_integer_and_float(sch):
    run_matmul(256, 384, 256, "tf32", "f32", tc(**sch), MODE_INT)
    err, _ = run_matmul(256, 384, 256, "tf32", "f32", tc(**sch), MODE_UNIFORM)
    assert err <= 5e-3


# ------------------------------------------------------------------ conv --
@pytest.mark.parametrize("shape", [(2, 56, 56, 64, 64), (3, 14, 14, 256, 256)])
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_tc_conv_resnet_layers(shape, mode):
    b, h, w, c, f = shape
    d = xtc.conv2d_desc(b, h, w, c, f, 3, 3, 1, 1, "bf16", "bf16")
    run_conv(d, "bf16", "bf16", tc(tile_n=min(f, 256), tile_k=64, stages=4, persistent=1, acc_buffers=2), mode)


def test_tc_conv_split_k_and_stride2():
    d = xtc.conv2d_desc(2, 14, 14, 256, 256, 3, 3, 1, 1, "bf16", "bf16")
    run_conv(d, "bf16", "bf16", tc(tile_n=128, split_k=3), MODE_INT)
    d2 = xtc.conv2d_desc(2, 15, 17, 64, 128, 3, 3, 2, 1, "bf16", "f32")
    run_conv(d2, "bf16", "f32", tc(tile_n=128, buffer_c=0), MODE_INT)


# pack_halo: the input packed once per output tile, filter taps as row-shifted views
PAIR_H = dict(tile_m=256, cluster_m=2, inner_m=256)
HALO_CASES = [
    # (batch, h, w, c, f, r, s, pad, in, out, schedule overrides)            Wp  rows/UMMA tile
    ((2, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(tile_n=64, b_resident=1, stages=2)),               # 64  2
    ((2, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(tile_m=256, tile_n=64, b_resident=1, stages=2)),   # 64  2x2
    ((3, 14, 14, 256, 256, 3, 3, 1, "bf16", "bf16"), dict(tile_n=128, stages=4)),                          # 16  8
    ((3, 14, 14, 256, 256, 3, 3, 1, "bf16", "bf16"), dict(tile_n=256, tile_k=64, stages=2, buffer_c=0)),
    ((2, 9, 13, 64, 64, 3, 3, 1, "bf16", "f32"), dict(tile_n=64, stages=3)),                               # 16  ragged
    ((1, 20, 20, 64, 128, 5, 5, 2, "bf16", "bf16"), dict(tile_n=128, stages=3, acc_buffers=1)),            # 32  4
    ((2, 7, 7, 128, 64, 1, 1, 0, "bf16", "bf16"), dict(tile_n=64, stages=2, tile_m=256)),                  # 8   16x2
    ((1, 10, 10, 64, 64, 3, 3, 0, "bf16", "f32"), dict(tile_n=64, stages=2, buffer_c=0)),                  # 16  pad 0
    ((1, 3, 100, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(tile_n=64, stages=2)),                             # 128 1
    ((2, 14, 14, 64, 64, 3, 3, 1, "tf32", "f32"), dict(tile_n=64, tile_k=32, stages=4)),                   # tf32: 2 planes
    # cluster_m 2: the filter stream shared by two CTAs through TMA multicast
    ((3, 14, 14, 256, 256, 3, 3, 1, "bf16", "bf16"), dict(cluster_m=2, tile_n=128, tile_k=128, stages=3)),
    ((2, 28, 28, 64, 256, 3, 3, 1, "bf16", "f32"), dict(cluster_m=2, tile_n=256, stages=3, persistent=0, buffer_c=0)),
    # inner_m 256: CTA pair (cta_group::2), M = 256 UMMAs over two CTAs' patches and filter halves
    ((3, 14, 14, 256, 256, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, tile_n=128, tile_k=128, stages=3)),
    ((2, 14, 14, 256, 256, 3, 3, 1, "bf16", "f32"), dict(PAIR_H, tile_n=256, stages=3, buffer_c=0, persistent=0)),
    ((2, 28, 28, 64, 128, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, tile_n=128, stages=2, b_resident=1)),     # 32  4
    ((2, 9, 13, 64, 128, 3, 3, 1, "bf16", "f32"), dict(PAIR_H, tile_n=128, stages=2, acc_buffers=1)),      # ragged
    ((2, 14, 14, 64, 128, 3, 3, 1, "tf32", "f32"), dict(PAIR_H, tile_n=64, tile_k=32, stages=4)),          # tf32
    # the pair at tile_n = 64 (bf16): 64-byte-swizzle filter halves (32 columns per CTA), resident and ring,
    # two N tiles (column offsets), ragged P / Q, direct stores, fp32 out
    ((2, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, tile_n=64, b_resident=1, stages=2)),
    ((2, 28, 28, 64, 128, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, tile_n=64, stages=3)),
    ((2, 9, 13, 64, 64, 3, 3, 1, "bf16", "f32"), dict(PAIR_H, tile_n=64, stages=2, buffer_c=0, acc_buffers=1)),
    ((2, 14, 14, 128, 64, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, tile_n=64, tile_k=128, b_resident=1, stages=2)),
    # split_k: K segments (runs of taps / channel planes) as CTAs, ordered reduction
    ((1, 14, 14, 256, 256, 3, 3, 1, "bf16", "bf16"), dict(tile_n=128, stages=4, split_k=3, buffer_c=0)),
    ((1, 14, 14, 256, 256, 3, 3, 1, "bf16", "bf16"), dict(tile_n=128, stages=4, split_k=9, buffer_c=0)),
    ((1, 56, 56, 64, 64, 3, 3, 1, "bf16", "f32"), dict(tile_n=64, stages=2, split_k=3, buffer_c=0, b_resident=1)),
    # s-fold (inner_n = S x tile_n): a filter row's S taps as the N blocks of one UMMA, the s shift applied in
    # the epilogue -- Wp 64 (output rows span two epilogue warps: cross-warp exchange), Wp 16 / 32 (no
    # exchange), Wp 128, S = 2 and 4, 2 channel planes, ragged P / Q, direct stores, many tiles per CTA
    ((4, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(tile_n=64, inner_n=192, b_resident=1, stages=2)),
    ((2, 30, 27, 64, 64, 3, 3, 1, "bf16", "f32"), dict(tile_n=64, inner_n=192, b_resident=1, stages=2, buffer_c=0)),
    ((3, 14, 14, 128, 64, 3, 3, 1, "bf16", "bf16"), dict(tile_n=64, inner_n=192, b_resident=1, stages=2)),
    ((2, 20, 21, 64, 64, 3, 4, 2, "bf16", "bf16"), dict(tile_n=64, inner_n=256, b_resident=1, stages=2)),
    ((2, 12, 100, 64, 64, 2, 2, 0, "bf16", "f32"), dict(tile_n=64, inner_n=128, b_resident=1, stages=2,
                                                        acc_buffers=1)),
    ((2, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(tile_n=64, inner_n=192, b_resident=1, stages=2,
                                                        persistent=1, grid_sms=5)),
    # pack_halo 2 (compact rows, Wc = Q + S - 1): tiles start mid-row, a warp's 32 rows wrap into the next
    # output row (direct stores); Wc 58 / 41 / 34 / 104 / 15, tile_m 128 / 256, ragged image ends, fp32
    # out, a 5x5 filter, 2 channel planes, tf32, several tiles per CTA (grid_sms)
    ((2, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(pack_halo=2, tile_n=64, b_resident=1, stages=2, buffer_c=0)),
    ((2, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(pack_halo=2, tile_n=64, b_resident=1, stages=2, buffer_c=0,
                                                        grid_sms=7)),
    ((3, 17, 39, 64, 128, 3, 3, 1, "bf16", "f32"), dict(pack_halo=2, tile_n=128, stages=3, buffer_c=0)),
    ((2, 11, 30, 128, 64, 5, 5, 2, "bf16", "bf16"), dict(pack_halo=2, tile_m=256, tile_n=64, stages=3, buffer_c=0)),
    ((2, 9, 102, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(pack_halo=2, tile_n=64, b_resident=1, stages=2,
                                                        buffer_c=0, grid_sms=3)),
    ((2, 13, 13, 64, 64, 3, 3, 1, "bf16", "f32"), dict(pack_halo=2, tile_n=64, stages=2, buffer_c=0)),
    ((2, 14, 14, 64, 64, 3, 3, 1, "tf32", "f32"), dict(pack_halo=2, tile_n=64, tile_k=32, stages=4, buffer_c=0)),
    # ragged N tiles (F = 96 / 160: the last tile's upper half partly or wholly past F) with direct stores, where
    # warps 0-3 drain the upper column half of each CTA's last tile; tile_m 256, compact rows, several tiles per CTA
    ((2, 20, 21, 64, 96, 3, 3, 1, "bf16", "f32"), dict(tile_m=256, tile_n=64, stages=3, buffer_c=0)),
    ((3, 17, 39, 64, 160, 3, 3, 1, "bf16", "bf16"), dict(pack_halo=2, tile_n=128, stages=3, buffer_c=0, grid_sms=5)),
    ((2, 14, 14, 128, 96, 3, 3, 1, "bf16", "bf16"), dict(tile_n=64, tile_k=128, stages=3, buffer_c=0, grid_sms=3)),
    # compact rows with the CTA pair (tile j of images 2i and 2i + 1): F = 64 halves, a two-N-tile ring, ragged
    ((4, 56, 56, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, pack_halo=2, tile_n=64, b_resident=1, stages=2,
                                                        buffer_c=0)),
    ((2, 17, 39, 64, 256, 3, 3, 1, "bf16", "f32"), dict(PAIR_H, pack_halo=2, tile_n=128, stages=3, buffer_c=0)),
    ((2, 9, 102, 64, 64, 3, 3, 1, "bf16", "bf16"), dict(PAIR_H, pack_halo=2, tile_n=64, stages=2, buffer_c=0,
                                                        grid_sms=4)),
]


@pytest.mark.parametrize("case", HALO_CASES, ids=[f"{c[0][:8]}-{i}" for i, c in enumerate(HALO_CASES)])
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_tc_conv_pack_halo(case, mode):
    (b, h, w, c, f, r, s, pad, idt, odt), kw = case
    d = xtc.conv2d_desc(b, h, w, c, f, r, s, 1, pad, idt, odt)
    base = dict(pack_halo=1, tile_m=128, tile_k=64, persistent=1, acc_buffers=2, buffer_c=1)
    base.update(kw)
    run_conv(d, idt, odt, tc(**base), mode)


def test_tc_conv_pack_halo_compact_fused_relu():
    d = xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16", consumer="relu")
    for extra in (dict(fuse=1), dict(fuse=1, acc_buffers=1)):
        run_conv_relu(d, tc(pack_halo=2, tile_n=64, stages=2, b_resident=1, persistent=1, buffer_c=0, **extra))


def run_conv_relu(d, sch, seed=30):
    import oracle as _o
    x = dev_tensor((d.batch, d.h, d.w, d.c), "bf16", seed, MODE_INT)
    w = dev_tensor((d.r, d.s, d.c, d.f), "bf16", seed + 1, MODE_INT)
    M, N, K = xtc.gemm_view(d)
    y = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0")
    xtc.Op(d).apply(sch).run(x, w, y)
    torch.cuda.synchronize()
    O, D = oracle_conv(d, "bf16", MODE_INT, seed, seed + 1)
    check_against_oracle(y, _o.relu(O), D, "bf16", True, 0.0)


def test_tc_conv_pack_halo_fused_relu_and_grid_modes():
    d = xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16", consumer="relu")
    for extra in (dict(fuse=1, persistent=1), dict(fuse=1, persistent=0, acc_buffers=1), dict(fuse=0)):
        run_conv_relu(d, tc(pack_halo=1, tile_n=64, stages=3, **extra))


# ------------------------------------------------ the paper's §VI-B workloads --
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_paper_tu_matmul_512x128x1024(mode):
    """[512,128] x [128,1024] (Fig.11): tcgen05 bf16 and SIMT fp32 schedules."""
    for sch in (tc(tile_n=64, tile_k=64, stages=2), tc(tile_n=128, tile_k=128, stages=2, persistent=1, acc_buffers=2),
                tc(tile_m=256, cluster_m=2, tile_n=256, tile_k=64, stages=2)):
        err, _ = run_matmul(512, 1024, 128, "bf16", "bf16", sch, mode)
        assert err <= 5e-3
    err, _ = run_matmul(512, 1024, 128, "f32", "f32", S(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4,
                                                          inner_n=4, unroll_k=4, vector_n=4, stages=2, swizzle=4), mode)
    assert err <= 1e-5


@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_paper_stem_conv_7x7_stride2(mode):
    """[112,112,16] x [7,7,3] step 2 (reading 4): 224x224x3 -> 112x112x16, pad 3.  C = 3 gives a 6-byte
    pixel pitch (no TMA, no tcgen05 operand): fp32 runs on the SIMT engine (here), bf16 on the warp-MMA tensor-core
    engine (tests/test_gpu_mma_engine.py); K = 147 is ragged for every tile_k."""
    d = xtc.conv2d_desc(1, 224, 224, 3, 16, 7, 7, 2, 3, "f32", "f32")
    assert xtc.gemm_view(d) == (112 * 112, 16, 147)
    for sch in (S(engine=0, tile_m=64, tile_n=16, tile_k=8, inner_m=4, inner_n=2, unroll_k=2, stages=1),
                S(engine=0, tile_m=64, tile_n=16, tile_k=21, inner_m=4, inner_n=4, stages=2, vector_n=4, swizzle=4)):
        err = run_conv(d, "f32", "f32", sch, mode)
        assert err <= 1e-5


def test_simt_conv_fp32():
    d = xtc.conv2d_desc(2, 14, 14, 16, 32, 3, 3, 1, 1, "f32", "f32")
    sch = S(engine=0, tile_m=64, tile_n=32, tile_k=16, inner_m=4, inner_n=4, unroll_k=4, vector_n=4, stages=2)
    run_conv(d, "f32", "f32", sch, MODE_INT)
    run_conv(d, "f32", "f32", sch, MODE_UNIFORM)


# ------------------------------------------------- CTA pair (cta_group::2) --
PAIR_SCHEDS = [
    dict(tile_m=256, cluster_m=2, tile_n=256, stages=4, acc_buffers=2, persistent=1),
    dict(tile_m=256, cluster_m=2, tile_n=128, stages=6, acc_buffers=2, persistent=0),
    dict(tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=2, buffer_c=0),
    dict(tile_m=256, cluster_m=2, tile_n=128, split_k=3, persistent=1, acc_buffers=2, order=1, raster_group=2),
]


@pytest.mark.parametrize("sch", PAIR_SCHEDS)
def test_tc_pair_bf16_integer_bit_exact(sch):
    run_matmul(512, 512, 384, "bf16", "bf16", tc(**sch), MODE_INT)


def test_tc_pair_ragged_and_float():
    run_matmul(300, 328, 200, "bf16", "f32", tc(**PAIR_SCHEDS[0]), MODE_INT)
    err, _ = run_matmul(1024, 1024, 1024, "bf16", "bf16", tc(**PAIR_SCHEDS[0]), MODE_UNIFORM)
    assert err <= 5e-3


def test_tc_pair_tf32():
    sch = tc(tile_m=256, cluster_m=2, tile_n=128, tile_k=32, stages=4, persistent=1, acc_buffers=2)
    run_matmul(512, 256, 256, "tf32", "f32", sch, MODE_INT)
    err, _ = run_matmul(512, 256, 256, "tf32", "f32", sch, MODE_UNIFORM)
    assert err <= 5e-3


@pytest.mark.parametrize("shape", [(2, 56, 56, 64, 128), (3, 14, 14, 256, 256)])
def test_tc_pair_conv(shape):
    b, h, w, c, f = shape
    d = xtc.conv2d_desc(b, h, w, c, f, 3, 3, 1, 1, "bf16", "bf16")
    run_conv(d, "bf16", "bf16", tc(tile_m=256, cluster_m=2, tile_n=128, stages=4, persistent=1, acc_buffers=2),
             MODE_INT)


# ------------------------------------------------------- fault injection --
@pytest.mark.parametrize("kind,expect", [(1, "value"), (2, "nan"), (3, "block")])
@pytest.mark.parametrize("in_dtype", ["bf16", "f32"])
def test_validation_catches_injected_faults(monkeypatch, kind, expect, in_dtype):
    """SPEC S:524 / SURVEY T4: a corrupted, unwritten or dropped output must fail
    on-chip validation and be located."""
    monkeypatch.setenv("XTC_DEBUG_FAULT", str(kind))
    monkeypatch.setenv("XTC_DEBUG_FAULT_AT", "70,37")
    M = N = K = 128
    desc = xtc.matmul_desc(M, N, K, in_dtype, "f32")
    a = dev_tensor((M, K), in_dtype, 3, MODE_INT)
    b = dev_tensor((K, N), in_dtype, 4, MODE_INT)
    c = torch.empty((M, N), dtype=torch.float32, device="cuda:0")
    sch = tc(tile_n=128) if in_dtype == "bf16" else S(engine=0, tile_m=32, tile_n=32, tile_k=8, inner_m=2, inner_n=2)
    op = xtc.Op(desc).apply(sch)
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=0, repeats=1, validate=1, exact=1))
    assert m.valid == 0
    if expect == "nan":
        assert m.n_nan == 1 and (m.err_row, m.err_col) == (70, 37)
    elif expect == "value":
        assert m.n_mismatch == 1 and (m.err_row, m.err_col) == (70, 37) and m.max_norm_err > 0
    else:
        assert m.n_mismatch >= 1 and 70 <= m.err_row < 102 and 37 <= m.err_col < 69
    # validate=2 turns the failure into a status
    with pytest.raises(xtc.XtcError):
        xtc._check(xtc.lib().xtc_measure(op.handle, xtc._ptrs([a.data_ptr(), b.data_ptr()]), xtc._ptrs([c.data_ptr()]),
                                         xtc.ctypes.byref(xtc.measure_cfg(warmup=0, repeats=1, validate=2, exact=1)),
                                         xtc.ctypes.byref(xtc.xtc_metrics()), xtc.c_void_p(0)))


def test_illegal_schedule_launches_nothing():
    desc = xtc.matmul_desc(256, 256, 256, "bf16", "bf16")
    op = xtc.Op(desc).apply(tc())
    with pytest.raises(xtc.XtcError) as e:
        op.apply(tc(tile_n=100))
    assert e.value.status == xtc.XTC_E_ILLEGAL_SCHEDULE
    # the previous (legal) schedule is still in effect
    a = dev_tensor((256, 256), "bf16", 1, MODE_INT)
    b = dev_tensor((256, 256), "bf16", 2, MODE_INT)
    c = torch.empty((256, 256), dtype=torch.bfloat16, device="cuda:0")
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=0, repeats=2, validate=1, exact=1))
    assert m.valid == 1


def test_sweep_records_and_illegal_candidates():
    desc = xtc.matmul_desc(512, 512, 512, "bf16", "bf16")
    a = dev_tensor((512, 512), "bf16", 1, MODE_INT)
    b = dev_tensor((512, 512), "bf16", 2, MODE_INT)
    c = torch.empty((512, 512), dtype=torch.bfloat16, device="cuda:0")
    cands = [tc(tile_n=128), tc(tile_n=100), tc(tile_m=256, cluster_m=2, tile_n=256, persistent=1, acc_buffers=2),
             S(engine=0, tile_m=32, tile_n=32, tile_k=8, inner_m=2, inner_n=2)]
    recs = xtc.Op(desc).sweep(cands, a, b, c, xtc.measure_cfg(warmup=1, repeats=3, validate=1, exact=1))
    assert [r.status for r in recs] == [0, xtc.XTC_E_ILLEGAL_SCHEDULE, 0, xtc.XTC_E_ILLEGAL_SCHEDULE]
    assert recs[0].valid == 1 and recs[2].valid == 1 and recs[1].valid == -1
    assert recs[0].tflops_med > 0 and recs[0].t_min_ns <= recs[0].t_med_ns <= recs[0].t_max_ns


# ----------------------------------------------- named hardware counters --
def test_measure_named_counters():
    """a9 counters by name: collected by CUPTI in a pass after the
    timed reps.  Pinned to physics: after an L2 flush every byte of A and B must come from
    DRAM at least once, the kernel time must agree with the event timing, and the timed
    numbers / validation are unaffected by the extra pass."""
    n = 2048
    desc = xtc.matmul_desc(n, n, n, "bf16", "bf16")
    a = dev_tensor((n, n), "bf16", 1, MODE_UNIFORM)
    b = dev_tensor((n, n), "bf16", 2, MODE_UNIFORM)
    c = torch.empty((n, n), dtype=torch.bfloat16, device="cuda:0")
    op = xtc.Op(desc)
    op.apply(tc(tile_n=256, stages=4, persistent=1, acc_buffers=2))
    names = ["gpu.dram__bytes_read.sum", "gpu__time_duration.sum", "dram__bytes_write.sum"]
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=2, repeats=5, flush_l2=1, validate=1, counters=names))
    assert m.valid == 1 and m.n_reps == 5
    assert m.n_counters == 3, xtc.xtc_last_error()
    v = m.counter_values(names)
    compulsory = 2 * n * n * 2                       # A + B in bf16
    assert compulsory <= v["gpu.dram__bytes_read.sum"] <= 8 * compulsory
    assert 0 <= v["dram__bytes_write.sum"] <= 4 * n * n * 2
    # the user range is pushed/popped on the host around the call, so its duration also
    # holds the launch's submission latency (tens of us under CUPTI's replay): the upper
    # bound allows that, the lower bound pins that the kernel itself is inside the range
    assert 0.5 * m.t_min_ns <= v["gpu__time_duration.sum"] <= 3.0 * m.t_max_ns + 200e3


def test_measure_unknown_counter_is_unavailable_not_failure():
    desc = xtc.matmul_desc(256, 256, 256, "bf16", "bf16")
    a = dev_tensor((256, 256), "bf16", 1, MODE_INT)
    b = dev_tensor((256, 256), "bf16", 2, MODE_INT)
    c = torch.empty((256, 256), dtype=torch.bfloat16, device="cuda:0")
    op = xtc.Op(desc)
    op.apply(tc())
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=0, repeats=2, validate=1, exact=1,
                                            counters="gpu.no_such__metric.sum"))
    assert m.valid == 1 and m.t_med_ns > 0
    assert m.n_counters == -1 and "counters unavailable" in xtc.xtc_last_error()
    assert m.counter_values("gpu.no_such__metric.sum") == {}


# ------------------------------------------- multi-rank bench rehearsal --
def test_bench_two_rank_rehearsal_on_one_gpu(tmp_path):
    """The N>1 bench path (M-sharded GEMM + all-gather + sharded sweep + max-over-ranks
    timing) run end to end with 2 ranks sharing one GPU over gloo."""
    import json, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, XTC_BENCH_DIST="gloo-shared")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--sweep-candidates", "32"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["validation"]["valid"] == 1 and rec["value"] > 0
    # the default N>1 gather is the fused one (xtc_run_gather into symmetric memory)
    assert "fused into the GEMM epilogue" in rec["config"]["parallelism"], rec["config"]["parallelism"]
    assert rec["validation"]["valid_all_ranks"] == 1 and rec["validation"]["gather_consistent_all_ranks"] == 1
    sw = rec["extras"]["sweep_1024_bf16_sharded"]
    assert sw["ranks"] == 2 and sw["candidates"] == 32 and sw["valid"] + sw["invalid"] == 32
    cv = rec["extras"]["conv_L56_batch_sharded"]
    assert cv["ranks"] == 2 and cv["images_per_rank"] == 16 and cv["valid_all_ranks"] == 1 and cv["step_us"] > 0
    # the NCCL-form (chunked all-gather overlap) path
    cmd2 = [x if x != "--master-port=29533" else "--master-port=29534" for x in cmd[:-2]]
    out = subprocess.run(cmd2 + ["--no-extras", "--gather", "nccl"], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    rec = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert "block-cyclic chunks" in rec["config"]["parallelism"]
    assert rec["validation"]["valid_all_ranks"] == 1 and rec["validation"]["gather_consistent_all_ranks"] == 1


@pytest.mark.parametrize("pw", [2, 3])
def test_tc_pack_warps(pw):
    """pack with 2-3 TMA-issuing warps (k-blocks dealt round-robin over the ring)."""
    run_matmul(256, 512, 640, "bf16", "bf16", tc(tile_n=128, stages=5, pack_warps=pw, persistent=1, acc_buffers=2),
               MODE_INT)
    run_matmul(512, 512, 384, "bf16", "bf16", tc(tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=3,
                                                 pack_warps=pw, persistent=1, acc_buffers=2), MODE_INT)
    d = xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16")
    run_conv(d, "bf16", "bf16", tc(tile_n=64, stages=8, pack_warps=pw, persistent=1, acc_buffers=2), MODE_INT)


def test_tc_b_resident():
    """pack of B at the outermost loop level (whole B resident in SMEM, ring streams A)."""
    run_matmul(512, 64, 576, "bf16", "bf16", tc(tile_n=64, stages=6, b_resident=1, persistent=1, acc_buffers=2,
                                                pack_warps=2), MODE_INT)
    run_matmul(640, 256, 256, "bf16", "f32", tc(tile_m=256, cluster_m=2, tile_n=256, stages=3, b_resident=1,
                                                persistent=1, acc_buffers=2), MODE_INT)
    d = xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16")
    run_conv(d, "bf16", "bf16", tc(tile_n=64, stages=7, b_resident=1, persistent=1, acc_buffers=2, pack_warps=3),
             MODE_INT)
    run_conv(d, "bf16", "bf16", tc(tile_n=64, stages=7, b_resident=1, persistent=1, acc_buffers=2, pack_warps=3),
             MODE_UNIFORM)


# --------------------------------------------------- schedule invariance --
def _invariance(desc, in_dtype, out_dtype, cands, seed=5):
    M, N, K = xtc.gemm_view(desc)
    a = dev_tensor((M, K), in_dtype, seed, MODE_INT)
    b = dev_tensor((K, N), in_dtype, seed + 1, MODE_INT)
    c = torch.empty((M, N), dtype=TORCH_DT[out_dtype], device="cuda:0")
    op = xtc.Op(desc)
    recs = op.sweep(cands, a, b, c, xtc.measure_cfg(warmup=0, repeats=1, validate=1, exact=1))
    bad = [(i, r.status, r.valid, r.n_mismatch, r.n_nan) for i, r in enumerate(recs)
           if r.status != 0 or r.valid != 1 or r.n_mismatch != 0]
    assert not bad, bad[:5]
    # the on-chip reference itself equals the oracle: check the last candidate's output
    O, D = oracle_matmul(M, N, K, in_dtype, MODE_INT, seed, seed + 1)
    check_against_oracle(c, O, D, out_dtype, True, 0.0)
    return len(recs)


def test_schedule_invariance_tcgen05_sampled():
    """BASELINE north_star: every legal schedule gives bit-identical results on
    small-integer inputs.  128 draws from the legal tcgen05 design space (both CTA
    shapes, split-K, raster orders, epilogue modes, persistence) plus pack_warps /
    b_resident variants."""
    from paper_2512_16512_b200.strategy import GpuStrategy
    desc = xtc.matmul_desc(512, 512, 512, "bf16", "bf16")
    st = GpuStrategy(desc, exact_divisors=False)
    cands = [st.generate(s) for s in st.sample(128, seed=11)]
    extra = []
    for i, c in enumerate(cands[:32]):
        d = c.as_dict()
        d["pack_warps"] = 1 + i % 3
        if d["pack_warps"] > d["stages"]:          # illegal: ring-slot parity aliasing (planner rule)
            assert xtc.xtc_schedule_check(desc, xtc.schedule(**d), 148)[0] == xtc.XTC_E_ILLEGAL_SCHEDULE
            d["pack_warps"] = d["stages"]
        extra.append(xtc.schedule(**d))
    n = _invariance(desc, "bf16", "bf16", cands + extra)
    assert n == 160


def test_schedule_invariance_conv_sampled():
    """north_star's invariance property for the conv2d kernels: 96 random LEGAL schedules of one ragged
    3x3 conv (Q + S - 1 = 25: power-of-two rows 32, compact rows 25) drawn over the halo patch layouts
    (pack_halo 0 = TMA im2col, 1, 2), tile shapes, stages, epilogues, accumulator buffers, persistence and
    grid size, resident / ring / multicast filters, the CTA pair, split-K (ordered and cluster-reduced) --
    every one bit-exact on integer data against the on-chip fp64 reference, which equals the oracle."""
    import random
    d = xtc.conv2d_desc(3, 19, 23, 64, 128, 3, 3, 1, 1, "bf16", "bf16")
    rng = random.Random(17)
    cands, seen = [], set()
    for _ in range(20000):
        k = dict(engine=1, swizzle=128, pack_halo=rng.choice([0, 1, 2]), tile_m=rng.choice([128, 256]),
                 tile_n=rng.choice([64, 128]), tile_k=rng.choice([64, 128]), stages=rng.choice([2, 3, 4]),
                 buffer_c=rng.choice([0, 1]), acc_buffers=rng.choice([1, 2]), persistent=rng.choice([0, 1]),
                 b_resident=rng.choice([0, 0, 1]), cluster_m=rng.choice([1, 1, 2]), inner_m=rng.choice([0, 0, 256]),
                 split_k=rng.choice([1, 1, 1, 2, 3]), split_k_mode=rng.choice([0, 2]), grid_sms=rng.choice([0, 0, 7]))
        key = tuple(sorted(k.items()))
        if key in seen:
            continue
        seen.add(key)
        sch = xtc.schedule(**k)
        if xtc.xtc_schedule_check(d, sch, 148)[0] == xtc.XTC_OK:
            cands.append(sch)
        if len(cands) == 96:
            break
    assert len(cands) == 96
    assert {c.pack_halo for c in cands} == {0, 1, 2}
    M, N, K = xtc.gemm_view(d)
    x = dev_tensor((d.batch, d.h, d.w, d.c), "bf16", 41, MODE_INT)
    w = dev_tensor((d.r, d.s, d.c, d.f), "bf16", 42, MODE_INT)
    y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda:0")
    recs = xtc.Op(d).sweep(cands, x, w, y, xtc.measure_cfg(warmup=0, repeats=1, validate=1, exact=1))
    bad = [(i, cands[i].as_dict(), r.status, r.valid, r.n_mismatch) for i, r in enumerate(recs)
           if r.status != 0 or r.valid != 1 or r.n_mismatch != 0]
    assert not bad, bad[:3]
    O, D = oracle_conv(d, "bf16", MODE_INT, 41, 42)
    check_against_oracle(y, O, D, "bf16", True, 0.0)


def test_schedule_invariance_simt_sampled():
    from paper_2512_16512_b200.strategy import GpuStrategy
    desc = xtc.matmul_desc(200, 136, 328, "f32", "f32")
    st = GpuStrategy(desc, engine=xtc.XTC_ENGINE_SIMT, exact_divisors=False)
    cands = [st.generate(s) for s in st.sample(96, seed=12)]
    assert _invariance(desc, "f32", "f32", cands) == 96


@pytest.mark.parametrize("mnk", [(130, 130, 131), (96, 132, 100), (64, 64, 4)])
def test_simt_fast_and_generic_pack_paths(mnk):
    """Aligned shapes take the vectorised pack (16-byte loads, partial vectors zero-filled);
    odd pitches fall back to the scalar pack.  Both must be exact."""
    M, N, K = mnk
    for stages in (1, 2):
        sch = S(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, unroll_k=4, vector_n=4,
                stages=stages, swizzle=4)
        run_matmul(M, N, K, "f32", "f32", sch, MODE_INT)


# ------------------------------------------------------- fuse (relu) --
def run_matmul_relu(M, N, K, in_dtype, out_dtype, sch, mode, seed=21):
    desc = xtc.matmul_desc(M, N, K, in_dtype, out_dtype, consumer="relu")
    a = dev_tensor((M, K), in_dtype, seed, mode)
    b = dev_tensor((K, N), in_dtype, seed + 1, mode)
    c = torch.full((M, N), float("nan"), dtype=TORCH_DT[out_dtype], device="cuda:0")
    op = xtc.Op(desc).apply(sch)
    op.run(a, b, c)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, in_dtype, mode, seed, seed + 1)
    exact = mode == MODE_INT
    tol = 1e-5 if in_dtype == "f32" else 5e-3
    import oracle as _o
    check_against_oracle(c, _o.relu(O), D, out_dtype, exact, tol)
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=0, repeats=2, validate=1, exact=int(exact), tol=tol))
    assert m.valid == 1, m.as_dict()
    return op.launches()


@pytest.mark.parametrize("fuse", [0, 1])
def test_fuse_relu_tcgen05(fuse):
    n1 = run_matmul_relu(256, 384, 320, "bf16", "bf16", tc(tile_n=128, fuse=fuse), MODE_INT)
    assert n1 == (1 if fuse else 2)            # fused: one kernel; unfused: GEMM + relu pass
    run_matmul_relu(256, 384, 320, "bf16", "f32", tc(tile_n=128, split_k=2, fuse=fuse), MODE_INT)
    run_matmul_relu(512, 256, 256, "bf16", "bf16", tc(tile_m=256, cluster_m=2, tile_n=256, fuse=fuse, persistent=1,
                                                      acc_buffers=2), MODE_UNIFORM)


def test_fuse_relu_atomic_splitk_unfused_and_simt_and_tail():
    run_matmul_relu(256, 256, 512, "bf16", "f32", tc(tile_n=128, split_k=4, split_k_mode=1, buffer_c=0, fuse=0),
                    MODE_INT)
    run_matmul_relu(200, 136, 328, "f32", "f32", S(engine=0, tile_m=32, tile_n=32, tile_k=8, inner_m=2, inner_n=2,
                                                   fuse=1), MODE_INT)
    run_matmul_relu(256, 258, 512, "f32", "f32", S(engine=0, tile_m=16, tile_n=128, tile_k=4, inner_m=1, inner_n=8,
                                                   unroll_k=4, vector_n=4, split_n_at=256, fuse=1), MODE_INT)


def test_fuse_relu_conv():
    d = xtc.conv2d_desc(2, 14, 14, 64, 128, 3, 3, 1, 1, "bf16", "bf16", consumer="relu")
    x = dev_tensor((2, 14, 14, 64), "bf16", 30, MODE_INT)
    w = dev_tensor((3, 3, 64, 128), "bf16", 31, MODE_INT)
    y = torch.empty((2 * 14 * 14, 128), dtype=torch.bfloat16, device="cuda:0")
    op = xtc.Op(d).apply(tc(tile_n=128, fuse=1))
    op.run(x, w, y)
    torch.cuda.synchronize()
    O, D = oracle_conv(d, "bf16", MODE_INT, 30, 31)
    import oracle as _o
    check_against_oracle(y, _o.relu(O), D, "bf16", True, 0.0)


# ------------------------------------------------- consumers: bias / accumulate --
def run_consumer(d, sch, cons, in_dtype, out_dtype, mode, seed=40):
    """One run of `sch` with the consumer bits `cons` (include/xtc.h) against
    oracle.consume(oracle result, relu, bias, C_old); then the library's own validation."""
    import oracle as _o
    from seeded_inputs import gen_tensor as _gen
    d.consumer = xtc.consumer_bits(cons)
    is_conv = d.kind == xtc.XTC_OP_CONV2D
    M, N, K = xtc.gemm_view(d)
    if is_conv:
        a = dev_tensor((d.batch, d.h, d.w, d.c), in_dtype, seed, mode)
        b = dev_tensor((d.r, d.s, d.c, d.f), in_dtype, seed + 1, mode)
        O, D = oracle_conv(d, in_dtype, mode, seed, seed + 1)
    else:
        a = dev_tensor((M, K), in_dtype, seed, mode)
        b = dev_tensor((K, N), in_dtype, seed + 1, mode)
        O, D = oracle_matmul(M, N, K, in_dtype, mode, seed, seed + 1)
    bits = d.consumer
    bias = dev_tensor((N,), "f32", seed + 7, mode) if bits & xtc.XTC_CONSUMER_BIAS else None
    if bits & xtc.XTC_CONSUMER_ACCUMULATE:
        c = dev_tensor((M, N), out_dtype, seed + 9, mode)
    else:
        c = torch.full((M, N), float("nan"), dtype=TORCH_DT[out_dtype], device="cuda:0")
    c_old = out_as_f64(to_numpy_out(c, out_dtype), out_dtype).reshape(M, N) if bits & xtc.XTC_CONSUMER_ACCUMULATE else None
    bias_np = _gen(seed + 7, (N,), "f32", mode).astype(np.float64) if bias is not None else None
    op = xtc.Op(d).apply(sch)
    op.run(a, b, c, bias=bias)
    torch.cuda.synchronize()
    want = _o.consume(O, bool(bits & xtc.XTC_CONSUMER_RELU), bias_np, c_old)
    Dn = D + (np.abs(c_old) if c_old is not None else 0) + (np.abs(bias_np)[None, :] if bias_np is not None else 0)
    exact = mode == MODE_INT
    tol = 1e-5 if in_dtype == "f32" else 5e-3
    check_against_oracle(c, want, Dn, out_dtype, exact, tol)
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=1, repeats=2, validate=1, exact=int(exact), tol=tol), bias=bias)
    assert m.valid == 1, m.as_dict()
    return op


CONS = ["bias", "accumulate", "bias+relu", "accumulate+bias+relu"]


@pytest.mark.parametrize("cons", CONS)
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_consumer_tcgen05_epilogue(cons, mode):
    d = lambda: xtc.matmul_desc(256, 320, 192, "bf16", "bf16")
    run_consumer(d(), tc(tile_n=64, fuse=1), cons, "bf16", "bf16", mode)                       # TMA-store epilogue
    run_consumer(d(), tc(tile_n=64, fuse=1, buffer_c=0), cons, "bf16", "bf16", mode)           # direct stores
    run_consumer(xtc.matmul_desc(256, 320, 192, "bf16", "f32"), tc(tile_n=64, fuse=1, persistent=1, acc_buffers=2),
                 cons, "bf16", "f32", mode)
    run_consumer(xtc.matmul_desc(512, 512, 256, "bf16", "bf16"),
                 tc(tile_m=256, cluster_m=2, tile_n=256, fuse=1, persistent=1, acc_buffers=2), cons, "bf16", "bf16", mode)


@pytest.mark.parametrize("cons", CONS)
def test_consumer_split_k_ordered_atomic_and_tail(cons):
    run_consumer(xtc.matmul_desc(256, 256, 512, "bf16", "bf16"), tc(tile_n=128, split_k=4, fuse=1), cons,
                 "bf16", "bf16", MODE_INT)                                                    # in the reduction
    if "relu" not in cons:                                                                    # relu + atomics: illegal
        run_consumer(xtc.matmul_desc(256, 256, 512, "bf16", "f32"),
                     tc(tile_n=128, split_k=4, split_k_mode=1, buffer_c=0, fuse=1), cons, "bf16", "f32", MODE_INT)
        run_consumer(xtc.matmul_desc(128, 96, 256, "f32", "f32"),
                     S(engine=0, tile_m=32, tile_n=32, tile_k=8, inner_m=2, inner_n=2, split_k=4, split_k_mode=1,
                       fuse=1), cons, "f32", "f32", MODE_INT)
    run_consumer(xtc.matmul_desc(256, 258, 512, "f32", "f32"),                                  # split_n_at remainder root
                 S(engine=0, tile_m=16, tile_n=128, tile_k=4, inner_m=1, inner_n=8, unroll_k=4, vector_n=4, stages=1,
                   split_n_at=256, fuse=1), cons, "f32", "f32", MODE_INT)


@pytest.mark.parametrize("cons", CONS)
def test_consumer_conv_simt_and_unfused(cons):
    run_consumer(xtc.conv2d_desc(2, 14, 14, 64, 128, 3, 3, 1, 1, "bf16", "bf16"), tc(tile_n=128, fuse=1), cons,
                 "bf16", "bf16", MODE_INT)                                                    # im2col conv
    run_consumer(xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16"),
                 tc(pack_halo=1, tile_n=64, stages=2, b_resident=1, persistent=1, acc_buffers=2, fuse=1), cons,
                 "bf16", "bf16", MODE_INT)                                                    # halo conv, TMA store
    run_consumer(xtc.conv2d_desc(1, 9, 13, 64, 64, 3, 3, 1, 1, "bf16", "f32"),
                 tc(pack_halo=1, tile_n=64, stages=3, buffer_c=0, fuse=1), cons, "bf16", "f32", MODE_INT)
    run_consumer(xtc.matmul_desc(200, 136, 328, "f32", "f32"),
                 S(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, unroll_k=4, vector_n=4, stages=2,
                   swizzle=4, fuse=1), cons, "f32", "f32", MODE_UNIFORM)
    if "accumulate" not in cons:                                                              # unfused: its own pass
        run_consumer(xtc.matmul_desc(256, 384, 320, "bf16", "bf16"), tc(tile_n=128, fuse=0), cons, "bf16", "bf16",
                     MODE_INT)


@pytest.mark.parametrize("cons", CONS)
def test_consumer_halo_compact_rows_and_pair64(cons):
    """The round-2 halo layouts with every consumer combination (bias, relu, accumulate): compact rows
    (direct stores at a mid-row tile start), the F = 64 CTA pair (64-byte filter halves; TMA store and direct),
    and compact rows with the pair (images 2i, 2i+1)."""
    L56 = lambda: xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16")
    pair = dict(tile_m=256, cluster_m=2, inner_m=256, tile_n=64, stages=2, b_resident=1, persistent=1, fuse=1)
    run_consumer(L56(), tc(pack_halo=2, tile_n=64, stages=2, b_resident=1, buffer_c=0, persistent=1, acc_buffers=2,
                           fuse=1), cons, "bf16", "bf16", MODE_INT)
    run_consumer(L56(), tc(pack_halo=1, acc_buffers=2, **pair), cons, "bf16", "bf16", MODE_INT)
    run_consumer(xtc.conv2d_desc(2, 9, 13, 64, 64, 3, 3, 1, 1, "bf16", "f32"),
                 tc(pack_halo=1, buffer_c=0, acc_buffers=1, **pair), cons, "bf16", "f32", MODE_INT)
    run_consumer(L56(), tc(pack_halo=2, buffer_c=0, acc_buffers=2, **pair), cons, "bf16", "bf16", MODE_INT)


def test_consumer_halo_split_last_ragged_n():
    """bias + relu on a ragged N tile drained by both warp groups (warps 0-3 take the upper half of the last tile)."""
    run_consumer(xtc.conv2d_desc(2, 20, 21, 64, 96, 3, 3, 1, 1, "bf16", "f32"),
                 tc(pack_halo=1, tile_n=64, stages=3, buffer_c=0, persistent=1, acc_buffers=2, fuse=1, grid_sms=3),
                 "bias+relu", "bf16", "f32", MODE_INT)
    run_consumer(xtc.conv2d_desc(2, 20, 21, 64, 96, 3, 3, 1, 1, "bf16", "bf16"),
                 tc(pack_halo=2, tile_n=64, stages=3, buffer_c=0, persistent=1, acc_buffers=1, fuse=1),
                 "accumulate+bias+relu", "bf16", "bf16", MODE_INT)


def test_consumer_halo_split_k_in_the_reduction():
    run_consumer(xtc.conv2d_desc(1, 14, 14, 256, 256, 3, 3, 1, 1, "bf16", "bf16"),
                 tc(pack_halo=1, tile_n=128, stages=4, split_k=4, buffer_c=0, fuse=1), "bias+relu", "bf16", "bf16",
                 MODE_INT)


def test_consumer_bias_pointer_required_and_sweep_with_accumulate():
    d = xtc.matmul_desc(256, 256, 256, "bf16", "bf16", consumer="bias")
    a = dev_tensor((256, 256), "bf16", 1, MODE_INT)
    b = dev_tensor((256, 256), "bf16", 2, MODE_INT)
    c = torch.empty((256, 256), dtype=torch.bfloat16, device="cuda:0")
    op = xtc.Op(d).apply(tc())
    with pytest.raises(xtc.XtcError, match="INVALID_ARG"):
        op.run(a, b, c)
    d2 = xtc.matmul_desc(256, 256, 256, "bf16", "f32", consumer="accumulate+bias")
    bias = dev_tensor((256,), "f32", 3, MODE_INT)
    c2 = dev_tensor((256, 256), "f32", 4, MODE_INT)
    recs = xtc.Op(d2).sweep([tc(tile_n=128, fuse=1), tc(tile_n=64, split_k=2, fuse=1),
                             tc(tile_n=128, split_k=2, split_k_mode=1, buffer_c=0, fuse=1)], a, b, c2,
                            xtc.measure_cfg(warmup=1, repeats=2, validate=1, exact=1), bias=bias)
    assert [r.valid for r in recs] == [1, 1, 1], [r.as_dict() for r in recs]


# ------------------------------------- fused all-gather (xtc_run_gather, N2) --
GATHER_CASES = [
    # (schedule, W virtual ranks, out dtype, N)
    (dict(tile_n=128, stages=4, persistent=1, acc_buffers=2), 4, "bf16", 384),
    (dict(tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=3, persistent=1, acc_buffers=2,
          raster_group=16), 4, "bf16", 512),
    (dict(tile_n=64, stages=6), 8, "f32", 328),          # ragged N: every destination's store is clipped
    (dict(tile_n=256, stages=3, acc_buffers=2, persistent=1), 1, "bf16", 256),
    # the bench headline tile: CTA pair with two M-subtiles (512-row tiles)
    (dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=4, persistent=1, raster_group=8), 2, "bf16", 512),
    (dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=3, persistent=1, raster_group=8), 2, "bf16", 512),
    # overlapped epilogue + gather with a ragged last N tile (576 = 2 x 256 + 64)
    (dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=3, persistent=1, raster_group=2), 2, "bf16", 576),
]


@pytest.mark.parametrize("sch,W,out,N", GATHER_CASES)
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_run_gather_every_destination_holds_the_gathered_matmul(sch, W, out, N, mode):
    """The M-sharded matmul with its all-gather fused into the epilogue, W ranks simulated on one
    GPU: rank r's op computes rows [r*M/W, (r+1)*M/W) and TMA-stores each tile to all W
    destinations.  Afterwards EVERY destination must equal the oracle's full C (bit-exact on
    integers, <= 5e-3 of D on uniform data) -- the all-gather's result."""
    M, K = 1024, 320
    Ms = M // W
    a = dev_tensor((M, K), "bf16", 11, mode)
    b = dev_tensor((K, N), "bf16", 12, mode)
    dests = [torch.full((M, N), float("nan"), dtype=TORCH_DT[out], device="cuda:0") for _ in range(W)]
    ptrs = [d.data_ptr() for d in dests]
    for r in range(W):
        op = xtc.Op(xtc.matmul_desc(Ms, N, K, "bf16", out)).apply(tc(**sch))
        op.run_gather(a[r * Ms:(r + 1) * Ms], b, ptrs, r * Ms, M)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", mode, 11, 12)
    for d in dests:
        check_against_oracle(d, O, D, out, exact=(mode == MODE_INT), tol=5e-3)


def test_run_gather_fused_relu_and_rerun_with_new_destinations():
    """A fused consumer (relu) applies before the multi-destination store; a second call with
    other destination pointers re-encodes the destination maps."""
    M, N, K, W = 512, 256, 192, 2
    Ms = M // W
    a = dev_tensor((M, K), "bf16", 21, MODE_INT)
    b = dev_tensor((K, N), "bf16", 22, MODE_INT)
    ops = [xtc.Op(xtc.matmul_desc(Ms, N, K, "bf16", "bf16", consumer="relu")).apply(tc(tile_n=128, fuse=1))
           for _ in range(W)]
    O, D = oracle_matmul(M, N, K, "bf16", MODE_INT, 21, 22)
    import oracle
    O = oracle.relu(O)
    for _ in range(2):
        dests = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0") for _ in range(W)]
        for r in range(W):
            ops[r].run_gather(a[r * Ms:(r + 1) * Ms], b, [d.data_ptr() for d in dests], r * Ms, M)
        torch.cuda.synchronize()
        for d in dests:
            check_against_oracle(d, O, D, "bf16", exact=True, tol=0)


def test_run_gather_rejects_unsupported_schedules_and_ranges():
    a = dev_tensor((256, 128), "bf16", 1, MODE_INT)
    b = dev_tensor((128, 128), "bf16", 2, MODE_INT)
    c = torch.zeros((512, 128), dtype=torch.bfloat16, device="cuda:0")
    ok = xtc.Op(xtc.matmul_desc(256, 128, 128)).apply(tc(tile_n=128))
    for bad in (dict(tile_n=128, split_k=2), dict(tile_n=128, buffer_c=0)):
        op = xtc.Op(xtc.matmul_desc(256, 128, 128)).apply(tc(**bad))
        with pytest.raises(xtc.XtcError):
            op.run_gather(a, b, [c.data_ptr()], 0, 512)
    with pytest.raises(xtc.XtcError):                       # rows past the destination
        ok.run_gather(a, b, [c.data_ptr()], 384, 512)
    with pytest.raises(xtc.XtcError):                       # more than 8 destinations
        ok.run_gather(a, b, [c.data_ptr()] * 9, 0, 512)
    ragged = xtc.Op(xtc.matmul_desc(200, 128, 128)).apply(tc(tile_n=128))
    with pytest.raises(xtc.XtcError):                       # ragged shard would spill into a neighbour
        ragged.run_gather(a[:200], b, [c.data_ptr()], 0, 512)


# ------------------------- cluster_n: A stages multicast across N-adjacent CTAs --
CLUSTER_N_SCHEDS = [
    dict(tile_n=64, stages=8, cluster_n=2),
    dict(tile_n=64, stages=6, cluster_n=4, persistent=1, acc_buffers=2, raster_group=2),
    dict(tile_n=128, tile_k=128, stages=3, cluster_n=2, persistent=1, acc_buffers=2, pack_warps=2),
    dict(tile_n=64, stages=4, cluster_n=2, split_k=2),
    dict(tile_n=64, stages=4, cluster_n=4, buffer_c=0, order=1),
]


@pytest.mark.parametrize("sch", CLUSTER_N_SCHEDS)
def test_tc_cluster_n_multicast_integer_bit_exact(sch):
    run_matmul(384, 512, 448, "bf16", "bf16", tc(**sch), MODE_INT)
    run_matmul(300, 512, 200, "bf16", "f32", tc(**sch), MODE_INT)     # ragged M and K


@pytest.mark.parametrize("size", [512, 1024])
def test_tc_cluster_n_float_tolerance(size):
    err, _ = run_matmul(size, size, size, "bf16", "bf16", tc(tile_n=64, stages=8, cluster_n=2, persistent=1,
                                                             acc_buffers=2), MODE_UNIFORM)
    assert err <= 5e-3


def test_tc_cluster_n_tf32():
    run_matmul(256, 256, 192, "tf32", "f32", tc(tile_n=64, tile_k=32, stages=6, cluster_n=2), MODE_INT)


# ------------------- two 128-row M-subtiles per CTA sharing B (tile_m = 256 * cta_group) --
MSUB_SCHEDS = [
    dict(tile_m=256, tile_n=128, stages=4),
    dict(tile_m=256, tile_n=256, tile_k=64, stages=3, persistent=1, raster_group=4),
    dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=4),
    dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=4, persistent=1, raster_group=16, order=1),
    dict(tile_m=512, cluster_m=2, tile_n=128, tile_k=64, stages=4, persistent=1, acc_buffers=2, pack_warps=2),
    dict(tile_m=256, tile_n=128, stages=3, split_k=2),
    dict(tile_m=256, tile_n=64, stages=4, buffer_c=0),
    # overlapped epilogue (bf16 out, 256 columns, 3 stages leave room for the 64 KB SMEM tile)
    dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=3, persistent=1, raster_group=8),
    dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=3),
]


@pytest.mark.parametrize("sch", MSUB_SCHEDS)
def test_tc_two_m_subtiles_integer_bit_exact(sch):
    run_matmul(1024, 512, 384, "bf16", "bf16", tc(**sch), MODE_INT)
    run_matmul(700, 512, 200, "bf16", "f32", tc(**sch), MODE_INT)      # ragged M (partial subtiles) and K


def test_tc_two_m_subtiles_float_and_tf32():
    err, _ = run_matmul(1024, 1024, 1024, "bf16", "bf16", tc(tile_m=512, cluster_m=2, tile_n=256, tile_k=64,
                                                             stages=4), MODE_UNIFORM)
    assert err <= 5e-3
    run_matmul(512, 256, 192, "tf32", "f32", tc(tile_m=256, tile_n=128, tile_k=32, stages=4), MODE_INT)
    desc_relu = dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=4, fuse=1)
    M, N, K = 512, 256, 128
    import oracle
    d = xtc.matmul_desc(M, N, K, "bf16", "bf16", consumer="relu")
    a = dev_tensor((M, K), "bf16", 31, MODE_INT)
    b = dev_tensor((K, N), "bf16", 32, MODE_INT)
    c = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0")
    xtc.Op(d).apply(tc(**desc_relu)).run(a, b, c)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", MODE_INT, 31, 32)
    check_against_oracle(c, oracle.relu(O), D, "bf16", exact=True, tol=0)


# ------------------------------------------------------- degenerate shapes --
@pytest.mark.parametrize("mnk", [(1, 1, 1), (1, 7, 3), (5, 1, 9), (3, 5, 1)])
def test_simt_degenerate_shapes(mnk):
    """Single rows/columns and a one-term reduction on the fp32 SIMT engine (bit-exact on integers)."""
    M, N, K = mnk
    run_matmul(M, N, K, "f32", "f32", S(engine=0, tile_m=8, tile_n=8, tile_k=8, inner_m=1, inner_n=1), MODE_INT)


@pytest.mark.parametrize("mnk", [(1, 64, 64), (1, 8, 8), (130, 64, 8), (3, 200, 24)])
@pytest.mark.parametrize("sch", [dict(tile_n=64, stages=2), dict(tile_m=256, cluster_m=2, tile_n=128, stages=2),
                                 dict(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=4)])
def test_tc_degenerate_shapes(mnk, sch):
    """One output row, the narrowest TMA-legal N (8 bf16 = 16 B rows), K smaller than one k-block (TMA
    zero-fills the rest of the box): one partial tile, every schedule family."""
    M, N, K = mnk
    run_matmul(M, N, K, "bf16", "bf16", tc(**sch), MODE_INT)


def test_conv_degenerate_single_pixel():
    """1x1 image, 3x3 filter with pad 1: only the centre tap meets data (P = Q = 1, M = batch)."""
    d = xtc.conv2d_desc(3, 1, 1, 64, 64, 3, 3, 1, 1, "bf16", "f32")
    run_conv(d, "bf16", "f32", tc(tile_n=64, stages=3), MODE_INT)
    d = xtc.conv2d_desc(1, 1, 1, 64, 128, 1, 1, 1, 0, "bf16", "bf16")
    run_conv(d, "bf16", "bf16", tc(tile_n=128, stages=2), MODE_INT)


def test_tc_overlapped_epilogue_ragged():
    """The overlapped epilogue (persistent, TMEM released before the stores) with ragged M and N; integer data
    bit-exact, uniform data within 5e-3.  These shapes give 45 and 60 tiles to 74 CTA pairs, i.e. ONE tile per
    pair: the cross-tile paths (SMEM tile reuse, TMEM phase flips) are covered by tests/test_gpu_multitile.py."""
    sch = tc(tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=3, persistent=1, raster_group=2)
    run_matmul(2048 + 300, 2048 + 64, 512, "bf16", "bf16", sch, MODE_INT)
    err, _ = run_matmul(3072, 2560, 1024, "bf16", "bf16", sch, MODE_UNIFORM)
    assert err <= 5e-3


def test_headline_schedule_with_fused_consumers():
    """The headline schedule with fused relu / bias: applied per 32-column chunk before the rounding inside
    the overlapped epilogue (both the SMEM-tile and the register-held subtile); exact on integers."""
    import bench
    import oracle
    M, N, K = 1024, 512, 256
    for cons in ("relu", "relu+bias"):
        d = xtc.matmul_desc(M, N, K, "bf16", "bf16", consumer=cons)
        a = dev_tensor((M, K), "bf16", 41, MODE_INT)
        b = dev_tensor((K, N), "bf16", 42, MODE_INT)
        bias = torch.arange(N, dtype=torch.float32, device="cuda:0") % 7 - 3
        c = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0")
        xtc.Op(d).apply(xtc.schedule(**dict(bench.HEADLINE_SCHEDULE, fuse=1))).run(
            a, b, c, bias=bias if "bias" in cons else None)
        torch.cuda.synchronize()
        O, D = oracle_matmul(M, N, K, "bf16", MODE_INT, 41, 42)
        O = oracle.consume(O, relu_=True, bias=bias.cpu().numpy().astype(np.float64) if "bias" in cons else None)
        check_against_oracle(c, O, D, "bf16", exact=True, tol=0)


# ------------------------------------- N3: descript / primitive-log front-ends --
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_fig4_and_fig8_schedules_run_on_the_gpu(mode):
    """The schedule built call for call from Fig.4 (imperative, primitive log) and from Fig.8 (descript)
    lowers to ONE xtc_schedule (tests/test_host.py pins that); it runs on the SIMT engine -- a 1 x 16
    register row with K1 = 4 unrolled and the [256, 258) remainder root -- against the oracle."""
    import test_host
    from paper_2512_16512_b200.scheduler import Scheduler
    desc = xtc.matmul_desc(256, 258, 512, "f32", "f32")
    s = Scheduler(desc)
    s.descript(test_host.FIG8)
    assert s.knobs() == test_host._fig4(desc).knobs()
    err, _ = run_matmul(256, 258, 512, "f32", "f32", s.schedule(), mode)
    assert err <= 1e-5


def test_descript_headline_runs_on_the_gpu():
    from paper_2512_16512_b200.scheduler import Scheduler
    desc = xtc.matmul_desc(1024, 768, 320, "bf16", "bf16")
    s = Scheduler(desc)
    s.descript({"I": ["parallelize"], "J": ["parallelize"], "K": ["pack=3"], "K#64": [], "I#512": [],
                "J#256": ["buffer"]})
    run_matmul(1024, 768, 320, "bf16", "bf16", s.schedule(dict(cluster_m=2, persistent=1, raster_group=8)),
               MODE_INT)
