"""-m gpu: oracle parity on the paths a persistent CTA (or CTA pair / cluster) takes when it strides over
SEVERAL output tiles -- the cross-tile state the full-size bench configs run through:

  * the overlapped epilogue's reuse of its 64 KB SMEM tile (bulk_wait_read before the next tile's
    drain) and TMEM released while the previous tile's TMA stores are still in flight;
  * the TMEM accumulator ping-pong (acc_buffers = 2) and the tfull / tempty phase flips;
  * the SMEM ring's slot / parity bookkeeping carried from one tile into the next (single CTA, CTA
    pair, two M-subtiles, A-multicast clusters, split-K segments as extra tiles);
  * the halo conv's patch-buffer phase flips and the im2col conv's per-tile (n, p, q) origin.

Every case asserts, from the planner's own plan (xtc_schedule_check on the 148-SM B200), that some
persistent CTA / pair / cluster processes >= 2 tiles, then compares the GPU output with the CPU oracle
element by element: bit-exact on integer data, <= 5e-3 of D on uniform data.  Some cases reach this at
the natural size (more tiles than SM pairs, like the 8192^3 headline's 7 tiles per pair); the others use
the schedule's ``grid_sms`` knob (parallelize over fewer SMs, include/xtc.h) so a small problem strides
over many tiles per CTA.  The Executor contract: PAPER.md P:792-795 (§IV-B).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, MODE_UNIFORM, gen_tensor
from gpu_util import TORCH_DT, check_against_oracle, dev_tensor, oracle_matmul, run_conv, run_matmul

pytestmark = pytest.mark.gpu

S = xtc.schedule
NUM_SMS = 148
HEADLINE = dict(engine=1, tile_m=512, tile_n=256, tile_k=64, stages=3, swizzle=128, buffer_c=1, acc_buffers=1,
                persistent=1, raster_group=8, order=0, cluster_m=2)
PAIR256 = dict(engine=1, tile_m=256, tile_n=256, tile_k=128, stages=3, swizzle=128, buffer_c=1, acc_buffers=2,
               persistent=1, raster_group=16, order=0, cluster_m=2)


def tc(**kw):
    base = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, swizzle=128, buffer_c=1, acc_buffers=1)
    base.update(kw)
    return S(**base)


def tiles_per_cluster(desc, sch):
    """Most tiles any persistent CTA / pair / cluster processes under the plan (the kernels stride
    t = cluster_id, cluster_id + #clusters, ...)."""
    st, info, why = xtc.xtc_schedule_check(desc, sch, NUM_SMS)
    assert st == xtc.XTC_OK, why
    clusters = info.grid_x // max(1, info.cluster_x)
    return -(-int(info.num_tiles) // clusters)


def multi(desc, sch, at_least=2):
    n = tiles_per_cluster(desc, sch)
    assert n >= at_least, f"plan gives {n} tile(s) per persistent cluster; this test needs >= {at_least}"
    return n


MODES = [MODE_INT, MODE_UNIFORM]


# ------------------------------------------------------------- matmul --
# (schedule, M, N, K, in dtype, out dtype): natural sizes first, then grid_sms-limited ones
MATMUL_CASES = [
    # the bench headline schedule (CTA pair, two M-subtiles, overlapped epilogue) at its natural grid:
    # 8 x 16 = 128 tiles over 74 pairs; then ragged M, N, K (9 x 17 = 153 tiles: up to 3 per pair)
    ("headline-4096", HEADLINE, 4096, 4096, 256, "bf16", "bf16"),
    ("headline-ragged", HEADLINE, 4096 + 200, 4096 + 64, 200, "bf16", "bf16"),
    # the same on 8 SMs (4 pairs): 45 tiles, 11-12 per pair
    ("headline-8sm", dict(HEADLINE, grid_sms=8), 2048 + 300, 2048 + 64, 512, "bf16", "bf16"),
    ("headline-8sm-order-nm", dict(HEADLINE, grid_sms=8, order=1, raster_group=2), 1536, 1280, 320, "bf16", "bf16"),
    # the previous headline: CTA pair, 256 x 256, double-buffered TMEM accumulator
    ("pair256-8sm", dict(PAIR256, grid_sms=8), 1280, 1088, 384, "bf16", "bf16"),
    ("pair256-8sm-f32", dict(PAIR256, grid_sms=8), 1000, 1024, 448, "bf16", "f32"),
    ("pair-direct-store-6sm", dict(engine=1, tile_m=256, cluster_m=2, tile_n=128, tile_k=64, stages=4, buffer_c=0,
                                   acc_buffers=2, persistent=1, grid_sms=6), 1024, 640, 256, "bf16", "bf16"),
    # two M-subtiles on one CTA (tile_m 256, no pair)
    ("msub-3sm", dict(engine=1, tile_m=256, tile_n=128, tile_k=64, stages=4, buffer_c=1, acc_buffers=1,
                      persistent=1, grid_sms=3), 1024, 768, 256, "bf16", "bf16"),
    ("msub-ovl-1cta-4sm", dict(engine=1, tile_m=256, tile_n=256, tile_k=64, stages=3, buffer_c=1, acc_buffers=1,
                               persistent=1, grid_sms=4, raster_group=4), 1280, 1024, 192, "bf16", "bf16"),
    # single-CTA tiles, TMEM ping-pong, split-K segments as extra tiles, odd SM counts
    ("1cta-acc2-5sm", tc(tile_n=256, stages=3, acc_buffers=2, persistent=1, grid_sms=5).as_dict(),
     640, 1024, 384, "bf16", "bf16"),
    ("1cta-splitk-7sm", tc(tile_n=128, stages=4, acc_buffers=2, persistent=1, split_k=3, grid_sms=7).as_dict(),
     512, 512, 576, "bf16", "bf16"),
    ("1cta-direct-tf32-3sm", tc(tile_n=128, tile_k=32, stages=4, acc_buffers=2, persistent=1, buffer_c=0,
                                grid_sms=3).as_dict(), 384, 384, 160, "tf32", "f32"),
    # A multicast across N-adjacent CTAs (cluster_n), persistent
    ("cluster-n2-8sm", tc(tile_n=128, stages=4, cluster_n=2, persistent=1, acc_buffers=2, grid_sms=8).as_dict(),
     1024, 1024, 320, "bf16", "bf16"),
    ("cluster-n4-8sm", tc(tile_n=64, stages=6, cluster_n=4, persistent=1, acc_buffers=2, raster_group=2,
                          grid_sms=8).as_dict(), 768, 1024, 256, "bf16", "bf16"),
    # fp32 on the tensor cores (3xTF32 split), persistent
    ("3xtf32-4sm", tc(tile_n=128, tile_k=32, stages=3, persistent=1, acc_buffers=2, grid_sms=4).as_dict(),
     512, 384, 256, "f32", "f32"),
    # SIMT engine, persistent (2 resident CTAs per SM)
    ("simt-2sm", dict(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, unroll_k=4, vector_n=4,
                      stages=2, swizzle=4, persistent=1, grid_sms=2), 520, 328, 200, "f32", "f32"),
]


@pytest.mark.parametrize("case", MATMUL_CASES, ids=[c[0] for c in MATMUL_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_matmul_many_tiles_per_persistent_cluster(case, mode):
    _, sch, M, N, K, idt, odt = case
    sch = S(**sch)
    multi(xtc.matmul_desc(M, N, K, idt, odt), sch)
    tol = 1e-5 if idt == "f32" else 5e-3
    err, _ = run_matmul(M, N, K, idt, odt, sch, mode, seed=3, tol=tol)
    assert err <= tol


def _run_consumer(M, N, K, sch, cons, mode, seed=51):
    d = xtc.matmul_desc(M, N, K, "bf16", "bf16", consumer=cons)
    multi(d, sch)
    a = dev_tensor((M, K), "bf16", seed, mode)
    b = dev_tensor((K, N), "bf16", seed + 1, mode)
    bits = d.consumer
    bias = dev_tensor((N,), "f32", seed + 7, mode) if bits & xtc.XTC_CONSUMER_BIAS else None
    c = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0")
    op = xtc.Op(d).apply(sch)
    op.run(a, b, c, bias=bias)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", mode, seed, seed + 1)
    bias_np = gen_tensor(seed + 7, (N,), "f32", mode).astype(np.float64) if bias is not None else None
    want = oracle.consume(O, bool(bits & xtc.XTC_CONSUMER_RELU), bias_np, None)
    Dn = D + (np.abs(bias_np)[None, :] if bias_np is not None else 0)
    check_against_oracle(c, want, Dn, "bf16", mode == MODE_INT, 5e-3)
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=1, repeats=2, validate=1, exact=int(mode == MODE_INT)),
                   bias=bias)
    assert m.valid == 1, m.as_dict()


@pytest.mark.parametrize("cons", ["relu", "bias+relu"])
@pytest.mark.parametrize("mode", MODES)
def test_headline_fused_consumers_many_tiles(cons, mode):
    """relu / bias applied per 32-column chunk inside the overlapped epilogue, 11-12 tiles per pair."""
    _run_consumer(2048 + 300, 2048 + 64, 256, S(**dict(HEADLINE, grid_sms=8, fuse=1)), cons, mode)


@pytest.mark.parametrize("sch,W", [(dict(HEADLINE, grid_sms=8), 2), (dict(PAIR256, grid_sms=4), 4),
                                   (tc(tile_n=128, stages=4, persistent=1, acc_buffers=2, grid_sms=3).as_dict(), 2)])
@pytest.mark.parametrize("mode", MODES)
def test_run_gather_many_tiles_per_cluster(sch, W, mode):
    """The fused all-gather (every staged tile TMA-stored to all W destinations) while each persistent
    pair strides over several tiles: every destination must hold the oracle's full C."""
    M, N, K = 2048, 1280, 256
    Ms = M // W
    sch = S(**sch)
    multi(xtc.matmul_desc(Ms, N, K, "bf16", "bf16"), sch)
    a = dev_tensor((M, K), "bf16", 61, mode)
    b = dev_tensor((K, N), "bf16", 62, mode)
    dests = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0") for _ in range(W)]
    ptrs = [d.data_ptr() for d in dests]
    for r in range(W):
        op = xtc.Op(xtc.matmul_desc(Ms, N, K, "bf16", "bf16")).apply(sch)
        op.run_gather(a[r * Ms:(r + 1) * Ms], b, ptrs, r * Ms, M)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", mode, 61, 62)
    for d in dests:
        check_against_oracle(d, O, D, "bf16", exact=(mode == MODE_INT), tol=5e-3)


# --------------------------------------------------------------- conv --
HALO = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, pack_halo=1, buffer_c=1, acc_buffers=2, persistent=1)
CONV_CASES = [
    # BASELINE config 3's L56 at batch 8: 8 images x 28 tiles = 224 halo tiles over 148 CTAs (natural size)
    ("halo-L56-n8", (8, 56, 56, 64, 64), dict(HALO, tile_n=64, stages=2, b_resident=1)),
    ("halo-L56-n2-12sm", (2, 56, 56, 64, 64), dict(HALO, tile_n=64, stages=2, b_resident=1, grid_sms=12)),
    # the CTA pair with 64-byte filter halves (tile_n 64): 112 pair tiles over 5 pairs
    ("halo-pair64-L56-n8-10sm", (8, 56, 56, 64, 64), dict(HALO, tile_m=256, cluster_m=2, inner_m=256, tile_n=64,
                                                          stages=2, b_resident=1, grid_sms=10)),
    ("halo-pair64-compact-L56-n8-10sm", (8, 56, 56, 64, 64), dict(HALO, tile_m=256, cluster_m=2, inner_m=256,
                                                                  tile_n=64, stages=2, b_resident=1, pack_halo=2,
                                                                  buffer_c=0, grid_sms=10)),
    # compact rows (pack_halo 2) at batch 8: 8 x 26 = 208 tiles over 148 CTAs, and 52 tiles on 11 SMs
    ("halo-compact-L56-n8", (8, 56, 56, 64, 64), dict(HALO, pack_halo=2, buffer_c=0, tile_n=64, stages=2,
                                                      b_resident=1)),
    ("halo-compact-L56-n2-11sm", (2, 56, 56, 64, 64), dict(HALO, pack_halo=2, buffer_c=0, tile_n=64, stages=2,
                                                           b_resident=1, grid_sms=11)),
    ("halo-L56-msub2-n4-10sm", (4, 56, 56, 64, 64), dict(HALO, tile_m=256, tile_n=64, stages=2, b_resident=1,
                                                           grid_sms=10)),
    ("halo-L14-ring-n8-9sm", (8, 14, 14, 256, 256), dict(HALO, tile_n=128, stages=4, grid_sms=9)),
    # the L14 bench schedule: CTA pair (cta_group::2) over two CTAs' patches and filter halves
    ("halo-L14-pair-n8-8sm", (8, 14, 14, 256, 256), dict(HALO, tile_m=256, cluster_m=2, inner_m=256, tile_n=128,
                                                         tile_k=128, stages=3, grid_sms=8)),
    ("halo-L14-mcast-n8-6sm", (8, 14, 14, 256, 256), dict(HALO, cluster_m=2, tile_n=128, tile_k=128, stages=3,
                                                          grid_sms=6)),
    ("halo-L14-direct-acc1-n4-5sm", (4, 14, 14, 256, 256), dict(HALO, tile_n=256, stages=2, buffer_c=0,
                                                                acc_buffers=1, grid_sms=5)),
    # im2col conv (TMA im2col per k-block), natural size and few SMs
    ("im2col-L56-n8", (8, 56, 56, 64, 64), dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=8, swizzle=128,
                                                buffer_c=1, acc_buffers=2, persistent=1, raster_group=8,
                                                pack_warps=3)),
    ("im2col-L14-pair-n4-6sm", (4, 14, 14, 256, 256), dict(engine=1, tile_m=256, cluster_m=2, tile_n=256,
                                                           tile_k=128, stages=3, swizzle=128, buffer_c=1,
                                                           acc_buffers=2, persistent=1, pack_warps=2, grid_sms=6)),
]


@pytest.mark.parametrize("case", CONV_CASES, ids=[c[0] for c in CONV_CASES])
@pytest.mark.parametrize("mode", MODES)
def test_conv_many_tiles_per_persistent_cluster(case, mode):
    _, (b, h, w, c, f), sch = case
    d = xtc.conv2d_desc(b, h, w, c, f, 3, 3, 1, 1, "bf16", "bf16")
    sch = S(**sch)
    multi(d, sch)
    run_conv(d, "bf16", "bf16", sch, mode, seed=71)
