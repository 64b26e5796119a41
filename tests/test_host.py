"""Host-side tests (no GPU): the C-ABI library loads and exports every symbol
of include/xtc.h, the planner's legality rules, the tile-order mapping and the
strategy pins (Fig.9 and the §VI-A 594-instance count)."""
import ctypes
import os
import re

import pytest

import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200 import strategy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
S = xtc.schedule


def header_functions():
    src = open(os.path.join(ROOT, "include", "xtc.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(xtc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 14, names
    lib = xtc.lib()
    for n in names:
        assert hasattr(lib, n), f"libxtc.so does not export {n}"


def test_struct_sizes_match_binding():
    sizes = (ctypes.c_int64 * 5)()
    xtc.lib().xtc_abi_sizes(sizes)
    assert list(sizes) == [ctypes.sizeof(t) for t in (xtc.xtc_op_desc, xtc.xtc_schedule, xtc.xtc_plan_info,
                                                       xtc.xtc_measure_cfg, xtc.xtc_metrics)]


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2512_16512_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "xtc_oracle" not in txt, f


def test_flops_and_bytes():
    d = xtc.matmul_desc(8192, 8192, 8192, "bf16", "bf16")
    assert xtc.xtc_op_flops(d) == 2 * 8192 ** 3
    assert xtc.xtc_op_min_bytes(d) == 3 * 8192 * 8192 * 2
    c = xtc.conv2d_desc(32, 56, 56, 64, 64)
    assert xtc.xtc_op_flops(c) == 2 * 32 * 56 * 56 * 64 * 9 * 64
    assert xtc.gemm_view(c) == (32 * 56 * 56, 64, 576)


# ------------------------------------------------------------- planner ----
def chk(desc, **kw):
    st, info, why = xtc.xtc_schedule_check(desc, S(**kw))
    return st, info, why


MM = xtc.matmul_desc(1024, 1024, 1024, "bf16", "bf16")
TCB = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, buffer_c=1)


def test_config1_plan():
    d = xtc.matmul_desc(32, 32, 32, "f32", "f32")
    st, info, why = chk(d, engine=0, tile_m=8, tile_n=8, tile_k=8, inner_m=1, inner_n=1)
    assert st == xtc.XTC_OK, why
    assert info.block_x == 64 and info.grid_x == 16 and info.num_tiles == 16


@pytest.mark.parametrize("kw,frag", [
    (dict(tile_n=100), "tile_n"),
    (dict(tile_m=64), "tile_m"),
    (dict(tile_k=32), "tile_k"),
    (dict(stages=1), "stages"),
    (dict(stages=9), "stages"),
    (dict(tile_n=256, tile_k=128, stages=4), "SMEM"),
    (dict(tile_n=256, acc_buffers=2, tile_k=64, stages=2), None),
    (dict(split_k=17), "empty K segment"),
    (dict(split_k=2, split_k_mode=1), "fp32 output"),
    (dict(unroll_k=2), "unroll_k"),
    (dict(order=2), "order"),
])
def test_tc_legality(kw, frag):
    args = dict(TCB)
    args.update(kw)
    st, info, why = chk(MM, **args)
    if frag is None:
        assert st == xtc.XTC_OK, why
        assert info.tmem_cols == 512
    else:
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (st, why)


def test_tc_fp32_is_the_3xtf32_split_and_simt_rejects_bf16():
    d32 = xtc.matmul_desc(256, 256, 256, "f32", "f32")
    st, info, why = chk(d32, **dict(TCB, tile_k=32, stages=3))
    assert st == xtc.XTC_OK, why
    assert info.smem_bytes == 3 * 2 * (128 * 32 * 4 + 32 * 128 * 4) + 32768 + 2048   # hi + lo per stage
    for kw, frag in ((dict(tile_m=256, cluster_m=2, tile_n=256), "cluster_m"), (dict(pack_warps=2), "pack_warps")):
        st, _, why = chk(d32, **dict(TCB, tile_k=32, stages=2, **kw))
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, why
    st, _, why = chk(xtc.conv2d_desc(1, 14, 14, 64, 64, 3, 3, 1, 1, "f32", "f32"), **dict(TCB, tile_k=32, stages=2))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "matmul only" in why
    st, _, why = chk(MM, engine=0, tile_m=16, tile_n=16, tile_k=8, inner_m=1, inner_n=1)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "fp32" in why


@pytest.mark.parametrize("kw,frag", [
    (dict(inner_m=3), "inner"),
    (dict(tile_m=64, inner_m=1, tile_n=64, inner_n=1), "threads"),
    (dict(unroll_k=3), "unroll_k"),
    (dict(tile_k=12, unroll_k=8), "divide"),
    (dict(vector_n=4, inner_n=2), "vector_n"),
    (dict(buffer_c=1), "buffer_c"),
])
def test_simt_legality(kw, frag):
    d = xtc.matmul_desc(256, 256, 256, "f32", "f32")
    args = dict(engine=0, tile_m=32, tile_n=32, tile_k=8, inner_m=2, inner_n=2)
    args.update(kw)
    st, _, why = chk(d, **args)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (st, why)


def test_tma_pitch_rule():
    d = xtc.matmul_desc(256, 258, 512, "bf16", "bf16")       # 516-byte B rows: not 16-byte aligned
    st, _, why = chk(d, **TCB)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "16-byte" in why
    d32 = xtc.matmul_desc(256, 258, 512, "f32", "f32")       # the paper's shape runs on the SIMT engine
    st, _, why = chk(d32, engine=0, tile_m=16, tile_n=64, tile_k=4, inner_m=1, inner_n=4, split_n_at=256)
    assert st == xtc.XTC_OK, why


def test_conv_legality_and_plan():
    c = xtc.conv2d_desc(32, 14, 14, 256, 256)
    st, info, why = chk(c, engine=1, tile_m=128, tile_n=256, tile_k=64, stages=4, buffer_c=1, split_k=3)
    assert st == xtc.XTC_OK, why
    assert info.num_tiles == 49 * 3 and info.k_blocks_per_split == 12
    c3 = xtc.conv2d_desc(1, 112, 112, 3, 16, 7, 7, 2, 3)    # C=3: not a 128-byte channel block
    st, _, why = chk(c3, engine=1, tile_m=128, tile_n=64, tile_k=64, stages=4)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE


HALO = dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2, buffer_c=1, acc_buffers=2, persistent=1,
            pack_halo=1)


def test_pack_halo_plan():
    """Tile counts follow from Wp = pow2 >= Q+S-1 slots and 128/Wp output rows per UMMA tile."""
    l56 = xtc.conv2d_desc(32, 56, 56, 64, 64)
    st, info, why = chk(l56, **dict(HALO, b_resident=1))
    assert st == xtc.XTC_OK, why
    assert info.num_tiles == 32 * 28 and info.grid_x == 148 and info.tmem_cols == 128
    # resident filter 9 x 8 KiB + 2 patches of 4 rows x 64 slots x 128 B + epilogue staging
    # resident filter + 3 patch buffers + epilogue staging + barriers + the SMEM tile table (64 x 32 B + 16)
    assert info.smem_bytes == 9 * 8192 + 3 * 4 * 64 * 128 + 32768 + 2048 + 64 * 32 + 16
    st, info, why = chk(l56, **dict(HALO, tile_m=256, b_resident=1))
    assert st == xtc.XTC_OK and info.num_tiles == 32 * 14 and info.tmem_cols == 256, why
    l14 = xtc.conv2d_desc(32, 14, 14, 256, 256)
    st, info, why = chk(l14, **dict(HALO, tile_n=128, stages=4))
    assert st == xtc.XTC_OK and info.num_tiles == 32 * 2 * 2, why
    # the CTA pair: the tile loop runs over M-tile pairs, two CTAs (one cluster) per pair tile
    st, info, why = chk(l14, **dict(HALO, tile_m=256, cluster_m=2, inner_m=256, tile_n=128, tile_k=128, stages=3))
    assert st == xtc.XTC_OK and info.num_tiles == 32 * 2 * 2 // 2 and info.cluster_x == 2, why
    one = xtc.conv2d_desc(2, 7, 7, 128, 64, 1, 1, 1, 0)        # 1x1: Wp = 8, 16 rows per tile
    st, info, why = chk(one, **HALO)
    assert st == xtc.XTC_OK and info.num_tiles == 2, why


def test_pack_halo_pair_64byte_filter_halves():
    """The CTA pair at tile_n = 64 (bf16): each CTA holds a 32-column half of every filter k-block
    (64-byte rows), so the resident L56 filter takes 9 x 64 x 32 x 2 = 36 KiB per CTA."""
    l56 = xtc.conv2d_desc(32, 56, 56, 64, 64)
    P = dict(HALO, tile_m=256, cluster_m=2, inner_m=256, tile_n=64)
    st, info, why = chk(l56, **dict(P, b_resident=1))
    assert st == xtc.XTC_OK and info.num_tiles == 32 * 28 // 2 and info.cluster_x == 2, why
    assert info.smem_bytes == 9 * 64 * 32 * 2 + 3 * 4 * 64 * 128 + 32768 + 2048 + 64 * 32 + 16
    st, info, why = chk(xtc.conv2d_desc(2, 28, 28, 64, 128), **dict(P, stages=3))     # ring, two N tiles
    assert st == xtc.XTC_OK and info.num_tiles == 2 * 7 * 2 // 2, why


def test_pack_halo_compact_plan():
    """pack_halo 2: Wc = Q + S - 1 slots per row, tiles of 128 consecutive virtual rows per image
    (ceil(P*Wc / 128) per image), patch rows = the rows spanned by a tile's largest read, + 1."""
    l56 = xtc.conv2d_desc(32, 56, 56, 64, 64)
    C = dict(HALO, pack_halo=2, buffer_c=0)
    st, info, why = chk(l56, **dict(C, b_resident=1))
    assert st == xtc.XTC_OK, why
    tpi = -(-56 * 58 // 128)                                     # 26 tiles per image (25 full + 48 rows)
    assert tpi == 26 and info.num_tiles == 32 * tpi and info.grid_x == 148
    pr = (57 + 127 + 2 * 58 + 2) // 58 + 1                       # 6 patch rows of 58 slots
    assert pr == 6 and pr * 58 * 128 == 44544
    # resident filter + 3 patch planes rounded up to the 1024-byte swizzle atom (44544 -> 45056 bytes),
    # no epilogue staging (direct stores), barriers + the SMEM tile table
    assert info.smem_bytes == 9 * 8192 + 3 * 45056 + 2048 + 64 * 32 + 16
    st, info, why = chk(l56, **dict(C, tile_m=256, b_resident=1))
    assert st == xtc.XTC_OK and info.num_tiles == 32 * (-(-56 * 58 // 256)), why
    # with the CTA pair (tile j of images 2i, 2i+1): 16 x 26 pair tiles
    st, info, why = chk(l56, **dict(C, tile_m=256, cluster_m=2, inner_m=256, b_resident=1))
    assert st == xtc.XTC_OK and info.num_tiles == 16 * 26 and info.cluster_x == 2, why
    # a power-of-two width gains nothing but stays legal: L14 (Wc = 16)
    l14 = xtc.conv2d_desc(4, 14, 14, 256, 256)
    st, info, why = chk(l14, **dict(C, tile_n=128, stages=4))
    assert st == xtc.XTC_OK and info.num_tiles == 4 * 2 * 2, why


@pytest.mark.parametrize("desc,kw,frag", [
    (xtc.conv2d_desc(2, 15, 17, 64, 128, 3, 3, 2, 1), {}, "stride 1"),
    (xtc.matmul_desc(256, 256, 256), {}, "conv2d only"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(cluster_m=4), "cluster_m"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(cluster_m=2, b_resident=1), "b_resident"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(cluster_m=2), "even number of 128-byte filter blocks"),
    (xtc.conv2d_desc(1, 14, 14, 256, 256), dict(cluster_m=2, tile_n=128, tile_m=256), "even number of M tiles"),
    (xtc.conv2d_desc(2, 14, 14, 256, 256), dict(inner_m=256, tile_n=128), "cluster_m 2 and tile_m 256"),
    (xtc.conv2d_desc(2, 56, 56, 64, 256), dict(inner_m=256, cluster_m=2, tile_m=256, tile_n=192), "tile_n % 128"),
    (xtc.conv2d_desc(2, 14, 14, 64, 64, 3, 3, 1, 1, "tf32", "f32"), dict(inner_m=256, cluster_m=2, tile_m=256, tile_n=32,
                                                                      tile_k=32), "64-byte filter halves"),
    (xtc.conv2d_desc(1, 7, 7, 256, 256), dict(inner_m=256, cluster_m=2, tile_m=256, tile_n=128), "even number of M tiles"),
    (xtc.conv2d_desc(2, 14, 14, 256, 256), dict(inner_m=256, cluster_m=2, tile_m=256, tile_n=128, split_k=2,
                                                buffer_c=0), "split_k 1"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(inner_m=64), "inner_m"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(split_k=3), "buffer_c 0"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(split_k=10, buffer_c=0), "empty K segment"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(pack_warps=2), "pack_warps"),
    (xtc.conv2d_desc(1, 4, 200, 64, 64), {}, "slots"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(tile_m=384), "tile_m"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(pack_halo=3), "pack_halo"),
    # pack_halo 2 (compact rows): one CTA per tile, no s-fold, no split, TMA-store staging needs Wc >= 32
    (xtc.conv2d_desc(2, 56, 56, 64, 128), dict(pack_halo=2, cluster_m=2, tile_n=128, buffer_c=0), "compact rows"),
    (xtc.conv2d_desc(3, 56, 56, 64, 64), dict(pack_halo=2, cluster_m=2, inner_m=256, tile_m=256, buffer_c=0),
     "even batch"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(pack_halo=2, inner_n=192, b_resident=1, buffer_c=0), "compact rows"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(pack_halo=2, split_k=3, buffer_c=0), "split_k must be 1"),
    (xtc.conv2d_desc(2, 56, 56, 64, 64), dict(pack_halo=2, buffer_c=1), "buffer_c 0"),
    (xtc.conv2d_desc(2, 56, 56, 256, 256), dict(tile_m=256, tile_n=256, acc_buffers=1, stages=8), "SMEM"),
])
def test_pack_halo_legality(desc, kw, frag):
    args = dict(HALO)
    args.update(kw)
    st, _, why = chk(desc, **args)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (st, why)
    st, _, why = chk(desc, engine=0, tile_m=32, tile_n=32, tile_k=8, inner_m=2, inner_n=2, pack_halo=1)
    assert st != xtc.XTC_OK


def test_consumer_bitmask_legality():
    """bias / accumulate: accumulate must be fused; relu cannot ride atomic split-K."""
    acc = xtc.matmul_desc(256, 256, 256, "bf16", "f32", consumer="accumulate+bias")
    st, _, why = chk(acc, **dict(TCB, fuse=0))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "accumulate must be fused" in why
    for kw in (dict(fuse=1), dict(fuse=1, split_k=2), dict(fuse=1, split_k=2, split_k_mode=1, buffer_c=0)):
        st, _, why = chk(acc, **dict(TCB, **kw))
        assert st == xtc.XTC_OK, (kw, why)
    br = xtc.matmul_desc(256, 256, 256, "bf16", "f32", consumer="bias+relu")
    st, _, why = chk(br, **dict(TCB, fuse=1, split_k=2, split_k_mode=1, buffer_c=0))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "atomic" in why
    st, _, why = chk(br, **dict(TCB, fuse=0))
    assert st == xtc.XTC_OK, why
    assert xtc.consumer_bits("accumulate+bias+relu") == 7 and xtc.consumer_bits(None) == 0


def test_default_schedules_are_legal():
    for d in (MM, xtc.matmul_desc(8192, 8192, 8192), xtc.conv2d_desc(32, 56, 56, 64, 64),
              xtc.conv2d_desc(32, 14, 14, 256, 256), xtc.matmul_desc(32, 32, 32, "f32", "f32"),
              xtc.matmul_desc(512, 512, 512, "tf32", "f32")):
        for lvl in (0, 2):
            if lvl == 0 and d.in_dtype != xtc.XTC_F32:
                continue
            s = xtc.xtc_schedule_default(d, lvl)
            st, _, why = xtc.xtc_schedule_check(d, s)
            assert st == xtc.XTC_OK, why


def test_invalid_descriptors():
    st, _, why = xtc.xtc_schedule_check(xtc.matmul_desc(0, 4, 4, "f32", "f32"), S(engine=0))
    assert st == xtc.XTC_E_INVALID_ARG


# --------------------------------------------------- tile order mapping ----
def _order_python(tiles_m, tiles_n, order, group):
    """Independent restatement: grouped raster = strip-mine the outer tile loop
    by `group`, then interchange so the inner loop runs inside the strip."""
    outer_n, inner_n = (tiles_m, tiles_n) if order == 0 else (tiles_n, tiles_m)
    seq = []
    for g0 in range(0, outer_n, group):
        for inner in range(inner_n):
            for outer in range(g0, min(g0 + group, outer_n)):
                seq.append((outer, inner) if order == 0 else (inner, outer))
    return seq


def test_tile_order_is_a_permutation():
    # the C mapping is exercised through the plan on the GPU; here we pin the
    # rule itself: every order/group visits each tile exactly once
    for tm, tn in [(3, 5), (8, 8), (7, 2)]:
        for order in (0, 1):
            for g in (1, 2, 4, 8):
                seq = _order_python(tm, tn, order, g)
                assert sorted(seq) == [(i, j) for i in range(tm) for j in range(tn)]
    assert _order_python(2, 3, 0, 1)[:3] == [(0, 0), (0, 1), (0, 2)]      # MN: N fastest


# ------------------------------------------------------------ strategy ----
def test_goto_space_594():
    """§VI-A: register tile 4x32, outer tiles free under divisibility, 1024^2 -> 594."""
    assert strategy.divisor_tiles(1024, 4) == [4, 8, 16, 32, 64, 128, 256, 512, 1024]
    assert strategy.goto_space_size(1024, 1024, 1024, 4, 32) == 594


def test_fig9_prt_sample_semantics():
    t = strategy.prt_tiles([1, 16, 4, 4, 1, 16, 16, 1])
    assert (t["i1"], t["i2"], t["i3"]) == (64, 64, 4)
    assert (t["j1"], t["j2"], t["j3"]) == (64, 16, 16)
    assert t["k1"] == 16 and t["W"] is True


def test_gpu_strategy_sampling_is_seeded_and_legal():
    st = strategy.GpuStrategy(MM)
    legal = st.legal_samples()
    assert len(legal) > 500
    a = st.sample(64, seed=3)
    assert a == st.sample(64, seed=3) and a != st.sample(64, seed=4)
    for smp in a:
        s = st.generate(smp)
        code, _, why = xtc.xtc_schedule_check(MM, s)
        assert code == xtc.XTC_OK, why


def test_fuse_legality():
    d = xtc.matmul_desc(256, 256, 256, "bf16", "f32", consumer="relu")
    st, _, why = chk(d, **dict(TCB, split_k=2, split_k_mode=1, buffer_c=0, fuse=1))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "atomic" in why
    for kw in (dict(fuse=1), dict(fuse=0), dict(split_k=2, fuse=1), dict(split_k=2, split_k_mode=1, buffer_c=0, fuse=0)):
        args = dict(TCB)
        args.update(kw)
        st, _, why = chk(d, **args)
        assert st == xtc.XTC_OK, (kw, why)
    bad = xtc.matmul_desc(64, 64, 64, "bf16", "f32")
    bad.consumer = 8                                  # not an XTC_CONSUMER_* bit
    st, _, why = xtc.xtc_schedule_check(bad, S(**TCB))
    assert st == xtc.XTC_E_INVALID_ARG


# ------------------------------------------------------- traffic model (N3) ----
def test_traffic_model_closed_forms():
    from paper_2512_16512_b200.model import predicted_l2_bytes
    d = xtc.matmul_desc(1024, 1024, 1024, "bf16", "bf16")
    # 128x128 tiles: A and B each streamed N/128 resp. M/128 times -> 2 * 1024^3 * 2 B / 128
    p = predicted_l2_bytes(d, S(**dict(TCB, tile_n=128)))
    assert p["loads"] == 2 * 1024 ** 3 * 2 / 128 and p["outputs"] == 1024 * 1024 * 2 and p["partials"] == 0
    # a CTA pair (tile_m 256) with tile_n 256 halves the operand traffic of 128x128
    p2 = predicted_l2_bytes(d, S(**dict(TCB, tile_m=256, cluster_m=2, tile_n=256)))
    assert p2["loads"] == p["loads"] / 2
    # split-K does not change the operand loads, adds S fp32 planes written and read
    p3 = predicted_l2_bytes(d, S(**dict(TCB, tile_n=128, split_k=4)))
    assert p3["loads"] == p["loads"] and p3["partials"] == 2 * 4 * 1024 * 1024 * 4
    # ragged: M = 300 -> 3 tiles of 128 rows are loaded in full boxes
    pr = predicted_l2_bytes(xtc.matmul_desc(300, 128, 64, "bf16", "bf16"), S(**dict(TCB, tile_n=128)))
    assert pr["loads"] == 3 * 1 * 64 * (128 + 128) * 2


def test_cluster_n_legality():
    """cluster_n (A multicast across N-adjacent CTAs): legal values and the rules of include/xtc.h."""
    d = xtc.matmul_desc(1024, 1024, 1024)
    base = dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=8, swizzle=128, buffer_c=1)
    for cn in (0, 1, 2, 4):
        st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**base, cluster_n=cn))
        assert st == xtc.XTC_OK, why
        if cn > 1:
            assert info.cluster_x == cn and info.grid_x == 128 and info.num_tiles == 128 // cn
    for bad in (dict(cluster_n=3), dict(cluster_n=8), dict(cluster_n=2, cluster_m=2, tile_m=256, tile_n=128),
                dict(cluster_n=2, b_resident=1)):
        st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, **bad)))
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE, bad
    # N tiles not divisible by cluster_n
    st, _, why = xtc.xtc_schedule_check(xtc.matmul_desc(1024, 192, 1024), xtc.schedule(**base, cluster_n=2))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "divide" in why
    # SIMT and conv reject it
    st, _, _ = xtc.xtc_schedule_check(d, xtc.schedule(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4,
                                                      inner_n=4, cluster_n=2))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE
    dc = xtc.conv2d_desc(2, 14, 14, 64, 64, 3, 3, 1, 1)
    st, _, _ = xtc.xtc_schedule_check(dc, xtc.schedule(**base, cluster_n=2))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE


def test_two_m_subtiles_legality():
    """tile_m = 256 x cluster_m: two 128-row UMMA subtiles per CTA (matmul only), TMEM = 2 x tile_n x acc."""
    d = xtc.matmul_desc(8192, 8192, 8192)
    ok = dict(engine=1, tile_m=512, cluster_m=2, tile_n=256, tile_k=64, stages=4, swizzle=128, buffer_c=1)
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**ok))
    assert st == xtc.XTC_OK, why
    assert info.tmem_cols == 512 and info.num_tiles == 16 * 32 and info.grid_x == 1024
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(ok, tile_m=256, cluster_m=1, tile_n=128)))
    assert st == xtc.XTC_OK, why
    for bad in (dict(acc_buffers=2),                       # 2 x 2 x 256 TMEM columns
                dict(tile_m=384),                          # not 128 or 256 per CTA
                dict(stages=5),                            # 5 x 48 KB stages exceed SMEM
                dict(inner_m=512)):                        # the UMMA M is 256
        st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(ok, **bad)))
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE, bad
    dc = xtc.conv2d_desc(2, 14, 14, 64, 64, 3, 3, 1, 1)
    st, _, why = xtc.xtc_schedule_check(dc, xtc.schedule(engine=1, tile_m=256, tile_n=64, tile_k=64, stages=4,
                                                         swizzle=128, buffer_c=1))
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "matmul only" in why


def test_bench_schedule_for_rows_wave_rule():
    """bench.py picks the 512-row pair tile unless a small shard's last wave wastes more of the GPU."""
    import bench
    assert bench.schedule_for_rows(8192) is bench.HEADLINE_SCHEDULE       # 512 tiles: 7 waves vs 14 half-size
    assert bench.schedule_for_rows(4096) is bench.PAIR256_SCHEDULE        # 256 tiles: 4 waves (8) vs 7
    assert bench.schedule_for_rows(2048) is bench.HEADLINE_SCHEDULE
    assert bench.schedule_for_rows(1024) is bench.HEADLINE_SCHEDULE
    for s in (bench.HEADLINE_SCHEDULE, bench.PAIR256_SCHEDULE):
        st, _, why = xtc.xtc_schedule_check(xtc.matmul_desc(8192, 8192, 8192), xtc.schedule(**s))
        assert st == xtc.XTC_OK, why


def test_overlapped_epilogue_smem_placement():
    """The headline plan reserves the 64 KB SMEM output tile of the overlapped epilogue (3 x 48 KB stages +
    64 KB + 2 KB); 4 stages leave no room (32 KB staging, plain epilogue); f32 output never overlaps."""
    import bench
    d = xtc.matmul_desc(8192, 8192, 8192)
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**bench.HEADLINE_SCHEDULE))
    assert st == xtc.XTC_OK, why
    assert info.smem_bytes == 3 * (256 * 64 * 2 + 64 * 128 * 2) + 65536 + 2048
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(bench.HEADLINE_SCHEDULE, stages=4)))
    assert st == xtc.XTC_OK and info.smem_bytes == 4 * 49152 + 32768 + 2048, why
    d32 = xtc.matmul_desc(8192, 8192, 8192, "bf16", "f32")
    st, info, why = xtc.xtc_schedule_check(d32, xtc.schedule(**bench.HEADLINE_SCHEDULE))
    assert st == xtc.XTC_OK and info.smem_bytes == 3 * 49152 + 32768 + 2048, why


# --------------------------------------------------------- the knob itself --
def test_grid_sms_plan_and_legality():
    import bench
    HEADLINE = bench.HEADLINE_SCHEDULE
    """grid_sms caps the persistent grid (parallelize over a number of cores, P:542-547)."""
    d = xtc.matmul_desc(4096, 4096, 256)
    st, info, _ = xtc.xtc_schedule_check(d, xtc.schedule(**HEADLINE), 148)
    assert st == 0 and info.grid_x == 148 and info.num_tiles == 128
    st, info, _ = xtc.xtc_schedule_check(d, xtc.schedule(**dict(HEADLINE, grid_sms=9)), 148)
    assert st == 0 and info.grid_x == 8          # whole CTA pairs only
    for bad in (dict(HEADLINE, grid_sms=1), dict(HEADLINE, grid_sms=8, persistent=0), dict(HEADLINE, grid_sms=-1)):
        st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**bad), 148)
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "grid_sms" in why


# ------------------------------------------- split with the in-kernel reduction --
def test_cluster_split_plan_and_legality():
    """split_k_mode 2: one cluster of split_k CTAs per output tile, reduced in the kernel."""
    CL = xtc.XTC_SPLITK_CLUSTER
    base = dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=4, buffer_c=0, acc_buffers=2, split_k_mode=CL)
    d = xtc.matmul_desc(512, 512, 512)
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, split_k=8)), 148)
    # 4 x 8 output tiles, each one cluster of 8 CTAs (one K segment of one k-block each)
    assert st == 0 and info.num_tiles == 32 and info.cluster_x == 8 and info.grid_x == 256, why
    assert info.k_blocks_per_split == 1 and info.workspace_bytes == 8 * 512 * 512 * 4
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, split_k=8, persistent=1)), 148)
    assert st == 0 and info.grid_x == 144, why          # whole clusters only: 18 x 8
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, split_k=4, persistent=1, grid_sms=10)), 148)
    assert st == 0 and info.grid_x == 8, why
    st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, split_k=4, buffer_c=1)), 148)
    assert st == 0, why                                  # partials through SMEM + TMA stores
    for bad, frag in ((dict(tile_m=256, cluster_m=2, tile_n=128), "cluster_m"),
                      (dict(split_k=17), "<= 16"), (dict(cluster_n=2), "cluster_n"), (dict(tile_m=256), "tile_m"),
                      (dict(split_k=16), "empty K segment"), (dict(b_resident=1, split_k=2), "b_resident")):
        kw = dict(base, split_k=4)
        kw.update(bad)
        st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**kw), 148)
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (bad, why)
    simt = dict(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, stages=2, split_k=2,
                split_k_mode=CL)
    st, _, why = xtc.xtc_schedule_check(xtc.matmul_desc(256, 256, 256, "f32", "f32"), xtc.schedule(**simt), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "tcgen05" in why
    # the haloed-patch conv: L14 at batch 1 = 2 x 2 tiles, 9 segments of 2 k-blocks
    dc = xtc.conv2d_desc(1, 14, 14, 256, 256, 3, 3, 1, 1)
    halo = dict(base, pack_halo=1, tile_n=128, tile_k=128, stages=3, split_k=9)
    st, info, why = xtc.xtc_schedule_check(dc, xtc.schedule(**halo), 148)
    assert st == 0 and info.num_tiles == 4 and info.cluster_x == 9 and info.grid_x == 36, why
    st, _, why = xtc.xtc_schedule_check(dc, xtc.schedule(**dict(halo, cluster_m=2)), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE


def test_stream_k_plan_and_legality():
    """split_k_mode 3: the persistent grid splits tiles x k-blocks into equal ranges."""
    SK = xtc.XTC_SPLITK_STREAM
    base = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, buffer_c=1, acc_buffers=2, persistent=1,
                split_k_mode=SK)
    d = xtc.matmul_desc(1280, 960, 576)                  # 10 x 8 = 80 tiles x 9 k-blocks = 720 iterations
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**base), 148)
    assert st == 0 and info.grid_x == 148 and info.num_tiles == 80, why
    assert info.workspace_bytes == 148 * 128 * 128 * 4      # one fp32 partial slot per CTA
    st, info, why = xtc.xtc_schedule_check(xtc.matmul_desc(256, 128, 256), xtc.schedule(**base), 148)
    assert st == 0 and info.grid_x == 8, why                 # 2 tiles x 4 k-blocks: one iteration per CTA
    for bad, frag in ((dict(persistent=0), "persistent"), (dict(split_k=2), "split_k"),
                      (dict(tile_m=256, cluster_m=2), "cluster_m"), (dict(tile_m=256), "tile_m"),
                      (dict(cluster_n=2), "cluster_n")):
        st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, **bad)), 148)
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (bad, why)
    # the haloed-patch conv (L56 at batch 2: 56 tiles x 9 k-blocks over 148 CTAs)
    dc = xtc.conv2d_desc(2, 56, 56, 64, 64, 3, 3, 1, 1)
    halo = dict(base, pack_halo=1, tile_n=64, stages=2)
    st, info, why = xtc.xtc_schedule_check(dc, xtc.schedule(**halo), 148)
    assert st == 0 and info.grid_x == 148 and info.num_tiles == 56, why
    st, _, why = xtc.xtc_schedule_check(dc, xtc.schedule(**dict(halo, cluster_m=2)), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE


def test_mma_engine_plan_and_legality():
    """Engine 2 (warp-MMA tiles over an im2col gather): the paper's C = 3 stem conv plans on it."""
    stem = xtc.conv2d_desc(1, 224, 224, 3, 16, 7, 7, 2, 3)
    base = dict(engine=xtc.XTC_ENGINE_MMA, tile_m=128, tile_n=16, tile_k=32)
    st, info, why = xtc.xtc_schedule_check(stem, xtc.schedule(**base), 148)
    assert st == 0 and info.num_tiles == 98 and info.grid_x == 98, why      # 112*112/128 tiles, F = 16
    assert xtc.xtc_schedule_check(stem, xtc.schedule(**dict(base, persistent=1)), 148)[0] == 0
    # the same conv cannot take the tcgen05 engine (C = 3: no 128-byte channel block for TMA)
    tc = dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=4, swizzle=128)
    assert xtc.xtc_schedule_check(stem, xtc.schedule(**tc), 148)[0] == xtc.XTC_E_ILLEGAL_SCHEDULE
    for bad, frag in ((dict(tile_m=256), "tile_m"), (dict(tile_n=48), "tile_n"), (dict(tile_k=8), "tile_k"),
                      (dict(split_k=2), "split_k"), (dict(buffer_c=1), "buffer_c"), (dict(inner_m=4), "inner_m")):
        st, _, why = xtc.xtc_schedule_check(stem, xtc.schedule(**dict(base, **bad)), 148)
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (bad, why)
    f32 = xtc.conv2d_desc(1, 224, 224, 3, 16, 7, 7, 2, 3, "f32", "f32")
    assert xtc.xtc_schedule_check(f32, xtc.schedule(**base), 148)[0] == xtc.XTC_E_ILLEGAL_SCHEDULE
    # pack_halo = 1: tile_m / Q whole output rows per CTA, the patch staged once (tile_k = the 16-deep step)
    pk = dict(base, pack_halo=1, tile_k=16)
    for tm, rows in ((128, 1), (256, 2), (512, 4)):
        st, info, why = xtc.xtc_schedule_check(stem, xtc.schedule(**dict(pk, tile_m=tm)), 148)
        assert st == 0 and info.num_tiles == 112 // rows and info.block_x == 32 * (-(-112 * rows // 32)), why
        # TMA layout (sw*C = 6 even, W*C = 672 = 42 chunks of 16): the row starts at element x0 = -16, delta = 1
        # makes every pixel run start even, kpr = 32 (21 taps + 1), 44 chunks of 32 B per row; 2 patch buffers
        # + filter 16 x (7*32 + 8) + staging + 2 mbarriers
        pr = (rows - 1) * 2 + 7
        px_w = -(-112 * rows // 32) * 32
        rnd = lambda b: -(-b // 128) * 128
        assert info.smem_bytes == 2 * rnd(pr * 44 * 32) + rnd(16 * 232 * 2) + px_w * 16 * 2 + 16 + 4 * 224, info.smem_bytes
        # pack_halo 2: thread-filled pixel slots of 4 channels, taps padded 7 -> 8, 230 slots per row, 1 buffer
        st, info2, why = xtc.xtc_schedule_check(stem, xtc.schedule(**dict(pk, tile_m=tm, pack_halo=2)), 148)
        assert st == 0 and info2.num_tiles == info.num_tiles, why
        assert info2.smem_bytes == rnd(pr * 230 * 8) + rnd(16 * 232 * 2) + px_w * 16 * 2 + 16 + 4 * 224, info2.smem_bytes
    for bad, frag in ((dict(tile_k=32), "tile_k"), (dict(tile_m=1024), "tile_m"), (dict(pack_halo=3), "pack_halo")):
        st, _, why = xtc.xtc_schedule_check(stem, xtc.schedule(**dict(pk, **bad)), 148)
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (bad, why)
    wide_c = xtc.conv2d_desc(1, 14, 14, 32, 16, 3, 3, 1, 1)
    st, _, why = xtc.xtc_schedule_check(wide_c, xtc.schedule(**pk), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "C must be" in why
    mm = xtc.matmul_desc(256, 64, 128)
    st, _, why = xtc.xtc_schedule_check(mm, xtc.schedule(**pk), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "conv2d" in why


# --------------------------------------------- N3: descript + primitive log --
def _fig4(desc):
    """PAPER.md Fig.4, call for call."""
    from paper_2512_16512_b200.scheduler import Scheduler
    sch = Scheduler(desc)
    sch.dims = ["I", "J", "K"]
    sch.split(root="mm0", dim="J", segments={"J[0]": 0, "J[1]": 256})
    sch.strip_mine(root="J[0]", dim="K", tiles={"K1": 4})
    sch.strip_mine(root="J[0]", dim="J", tiles={"J1": 16})
    sch.unroll(root="J[0]", unrolls={"J1": 16, "K1": 4})
    sch.vectorize(root="J[0]", axes=["J1"])
    sch.interchange(root="mm0", permutation=["I", "J[0]", "J[1]"])
    sch.interchange(root="J[0]", permutation=["K", "K1", "J1"])
    sch.interchange(root="J[1]", permutation=["K"])
    return sch


FIG8 = {"I": [], "J[0:256]": {"K": [], "K#4": ["unroll"], "J#16": ["vectorize"]}, "J[256:258]": {"K": []}}


def test_fig4_primitive_log_and_fig8_descript_give_one_schedule():
    """§V-A: Fig.8 is 'the reimplementation of the example in Fig.4'; both front-ends must build
    the same loop nest and lower to the same legal schedule: the SIMT engine with the 1 x 16 register row
    (J1 = 16, vectorized), K1 = 4 unrolled, and the [256, 258) remainder root."""
    from paper_2512_16512_b200.scheduler import Scheduler
    desc = xtc.matmul_desc(256, 258, 512, "f32", "f32")
    imp = _fig4(desc)
    dec = Scheduler(desc)
    dec.dims = ["I", "J", "K"]
    dec.descript(FIG8)
    want_nest = (("I", 256, ()),
                 ("split", "J", ((0, 256, (("K", 512, ()), ("K", 4, (("unroll", 4),)),
                                           ("J", 16, (("unroll", 16), ("vectorize", 1))))),
                                 (256, 258, (("K", 512, ()),)))))
    assert imp.nest() == want_nest
    assert dec.nest() == want_nest
    kn = imp.knobs()
    assert kn == dec.knobs()
    assert kn == dict(engine=0, split_n_at=256, order=0, tile_m=1, tile_n=16, inner_m=1, inner_n=16, tile_k=4,
                      unroll_k=4, stages=1, vector_n=4)
    st, info, why = imp.check()
    assert st == xtc.XTC_OK, why
    assert info.tail_grid_x == 1 and info.num_tiles == 256 * 16      # 1 x 16 tiles of [0, 256) + the remainder
    # the primitive log replays to the same state
    assert [p for p, _ in imp.log] == ["dims", "split", "strip_mine", "strip_mine", "unroll", "vectorize",
                                        "interchange", "interchange", "interchange"]
    again = Scheduler.replay(desc, imp.log)
    assert again.nest() == want_nest and again.knobs() == kn


def test_descript_and_primitives_lower_the_headline_schedule():
    """The bench's tcgen05 schedule written as a loop nest: I, J parallelized over the grid with steps 512 x 256
    (the CTA-pair tile), K staged in 64-deep blocks through a 3-stage pack, the output bufferized."""
    import bench
    from paper_2512_16512_b200.scheduler import Scheduler
    desc = xtc.matmul_desc(8192, 8192, 8192, "bf16", "bf16")
    target = dict(cluster_m=2, persistent=1, raster_group=8, acc_buffers=1)
    dec = Scheduler(desc)
    dec.descript({"I": ["parallelize"], "J": ["parallelize"], "K": ["pack=3"], "K#64": [], "I#512": [],
                  "J#256": ["buffer"]})
    imp = Scheduler(desc)
    imp.strip_mine(root="mm0", dim="I", tiles={"I1": 512})
    imp.strip_mine(root="mm0", dim="J", tiles={"J1": 256})
    imp.strip_mine(root="mm0", dim="K", tiles={"K1": 64})
    imp.interchange(root="mm0", permutation=["I", "J", "K", "K1", "I1", "J1"])
    imp.parallelize(root="mm0", axes=["I", "J"])
    imp.pack(root="mm0", at="K", stages=3)
    imp.bufferize(root="mm0", at="J1")
    assert imp.nest() == dec.nest()
    want = {k: v for k, v in bench.HEADLINE_SCHEDULE.items()}
    got = dec.knobs(target)
    assert {k: got.get(k, 0) for k in want} == want
    assert imp.knobs(target) == got
    assert dec.check(target)[0] == xtc.XTC_OK
    again = Scheduler.replay(desc, imp.log)
    assert again.knobs(target) == got


def test_scheduler_rejects_malformed_primitives():
    from paper_2512_16512_b200.scheduler import Scheduler, ScheduleError
    desc = xtc.matmul_desc(256, 258, 512, "f32", "f32")
    s = Scheduler(desc)
    with pytest.raises(ScheduleError):
        s.interchange(root="mm0", permutation=["I", "K"])               # not a permutation
    with pytest.raises(ScheduleError):
        s.strip_mine(root="nope", dim="K", tiles={"K1": 4})              # unknown root
    with pytest.raises(ScheduleError):
        s.unroll(root="mm0", unrolls={"K": 3})                           # 3 does not divide 512
    s.interchange(root="mm0", permutation=["K", "I", "J"])                # K outermost: no GPU lowering
    with pytest.raises(ScheduleError):
        s.knobs()
    with pytest.raises(ScheduleError):
        Scheduler(desc).descript({"I": [], "J": ["fuse"], "K": []})       # unknown annotation
    with pytest.raises(ScheduleError):
        Scheduler(desc).descript({"I": [], "J[0:100]": {"K": []}, "J[120:258]": {"K": []}})   # gap
    with pytest.raises(ScheduleError):
        Scheduler(xtc.conv2d_desc(1, 8, 8, 64, 64))


def test_sweep_resume_matches_the_full_key(tmp_path):
    """A resume file is matched on everything the candidate list depends on: records of
    another shape / dtype / engine / count under the same seed are refused, not merged."""
    import json
    from paper_2512_16512_b200.sweep import load_resume, sweep_key
    k1 = sweep_key(1024, 1024, 1024, 4096, 0, "bf16", "bf16", 1)
    k2 = sweep_key(512, 512, 512, 4096, 0, "bf16", "bf16", 1)
    p = tmp_path / "r.jsonl"
    assert load_resume(str(p), k1) == {}
    p.write_text("".join(json.dumps({"id": i, "key": k1, "tflops_med": 1.0}) + "\n" for i in (3, 7)))
    assert sorted(load_resume(str(p), k1)) == [3, 7]
    with pytest.raises(ValueError):
        load_resume(str(p), k2)
    p.write_text(json.dumps({"id": 0, "seed": 0, "tflops_med": 1.0}) + "\n")   # the round-1 format
    with pytest.raises(ValueError):
        load_resume(str(p), k1)


def test_pack_warps_bounded_by_stages():
    """pack_warps producers rotate over the ring; a producer only knows k-block g - pack_warps - stages
    was consumed, so pack_warps > stages could refill a slot two rounds behind (parity aliasing)."""
    d = xtc.matmul_desc(512, 512, 512)
    base = dict(engine=1, tile_m=256, tile_n=64, tile_k=64, swizzle=128, buffer_c=1, acc_buffers=2)
    st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, stages=2, pack_warps=3)), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and "pack_warps" in why, why
    for stages, pw in ((2, 2), (3, 3), (4, 3)):
        assert xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, stages=stages, pack_warps=pw)), 148)[0] == 0


def test_pack_halo_sfold_plan_and_legality():
    """inner_n = S x tile_n folds a filter row's S taps into one UMMA (TMEM: S accumulator blocks)."""
    d = xtc.conv2d_desc(32, 56, 56, 64, 64, 3, 3, 1, 1)
    base = dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2, swizzle=128, pack_halo=1, buffer_c=1,
                acc_buffers=2, persistent=1, b_resident=1)
    st, info, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, inner_n=192)), 148)
    assert st == 0 and info.tmem_cols == 512, why               # 2 buffers x 3 blocks x 64 columns -> 512
    st0, info0, _ = xtc.xtc_schedule_check(d, xtc.schedule(**base), 148)
    # the exchange rows for the warp above: 4 warps x 2 parities x 3 rows x 128 B
    assert info.smem_bytes == info0.smem_bytes + 4 * 2 * 3 * 128
    for bad, frag in ((dict(inner_n=128), "inner_n"), (dict(inner_n=192, b_resident=0), "b_resident"),
                      (dict(inner_n=192, tile_m=256), "tile_m"), (dict(inner_n=192, split_k=3, buffer_c=0), "split_k")):
        st, _, why = xtc.xtc_schedule_check(d, xtc.schedule(**dict(base, **bad)), 148)
        assert st == xtc.XTC_E_ILLEGAL_SCHEDULE and frag in why, (bad, why)
    d14 = xtc.conv2d_desc(32, 14, 14, 256, 256, 3, 3, 1, 1)       # S x tile_n must stay <= 256
    st, _, why = xtc.xtc_schedule_check(d14, xtc.schedule(**dict(base, tile_n=128, inner_n=384, b_resident=0)), 148)
    assert st == xtc.XTC_E_ILLEGAL_SCHEDULE
