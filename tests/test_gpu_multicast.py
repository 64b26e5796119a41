"""-m gpu: the fused all-gather through one multicast destination (xtc_run_multicast, SURVEY §8(f) N2,
the NVLS form; BASELINE.json north_star "sharded by M ... all-gather").

On sm_100a `multimem.st.global.v4` and `st.global.v4` assemble to the same STG.E.128 instruction (the
multicast replication is a property of the destination's mapping, not of the store), so the write-out
path -- SMEM read-back of every staged tile, 16-byte row-segment stores at the shard's global rows -- is
checked here with multimem = 0 on one GPU: W rank shards store into ONE shared destination, which must
then hold the oracle's full C (bit-exact on integers, <= 5e-3 of D on uniform data).  Multicast objects
cannot be created on the single-GPU boxes this suite runs on (cuMulticastCreate -> invalid value,
profiles/r02_multicast_probe.json); the W > 1 NVLS run is the bench's N > 1 path.
"""
import pytest
import torch

import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, MODE_UNIFORM
from gpu_util import TORCH_DT, check_against_oracle, dev_tensor, oracle_matmul

pytestmark = pytest.mark.gpu
S = xtc.schedule
HEADLINE = dict(engine=1, tile_m=512, tile_n=256, tile_k=64, stages=3, swizzle=128, buffer_c=1, acc_buffers=1,
                persistent=1, raster_group=8, order=0, cluster_m=2)
PAIR256 = dict(engine=1, tile_m=256, tile_n=256, tile_k=128, stages=3, swizzle=128, buffer_c=1, acc_buffers=2,
               persistent=1, raster_group=16, order=0, cluster_m=2)
ONE_CTA = dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=4, swizzle=128, buffer_c=1, acc_buffers=2,
               persistent=1)

CASES = [
    # (name, schedule, M, N, K, W, out): the overlapped epilogue (4 boxes per warp read back), the plain
    # epilogue's 32-row boxes (bf16 64-column and fp32 32-column), several tiles per persistent CTA / pair
    ("headline-w4", HEADLINE, 2048, 512, 256, 4, "bf16"),
    ("headline-w8-4sm", dict(HEADLINE, grid_sms=4), 4096, 768, 128, 8, "bf16"),
    ("pair256-w2", PAIR256, 1024, 512, 384, 2, "bf16"),
    ("pair256-w2-f32", PAIR256, 1024, 512, 256, 2, "f32"),
    ("1cta-w4-ragged-n", dict(ONE_CTA, grid_sms=3), 1024, 328, 192, 4, "bf16"),
    ("1cta-w8-f32", ONE_CTA, 1024, 256, 160, 8, "f32"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("mode", [MODE_INT, MODE_UNIFORM])
def test_multicast_writeout_assembles_the_gathered_matmul(case, mode):
    _, sch, M, N, K, W, out = case
    Ms = M // W
    a = dev_tensor((M, K), "bf16", 51, mode)
    b = dev_tensor((K, N), "bf16", 52, mode)
    dest = torch.full((M, N), float("nan"), dtype=TORCH_DT[out], device="cuda:0")
    for r in range(W):
        op = xtc.Op(xtc.matmul_desc(Ms, N, K, "bf16", out)).apply(S(**sch))
        op.run_multicast(a[r * Ms:(r + 1) * Ms], b, dest.data_ptr(), r * Ms, M, multimem=False)
        assert op.launches() == 1
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", mode, 51, 52)
    check_against_oracle(dest, O, D, out, exact=(mode == MODE_INT), tol=5e-3)


def test_multicast_fused_relu_bias():
    """Fused consumers are applied before the write-out (relu(A*B + bias) in every rank's rows)."""
    M, N, K, W = 1024, 256, 192, 2
    Ms = M // W
    a = dev_tensor((M, K), "bf16", 61, MODE_INT)
    b = dev_tensor((K, N), "bf16", 62, MODE_INT)
    bias = dev_tensor((N,), "f32", 63, MODE_INT)
    dest = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0")
    for r in range(W):
        op = xtc.Op(xtc.matmul_desc(Ms, N, K, "bf16", "bf16", consumer="bias+relu")).apply(S(**dict(HEADLINE, fuse=1)))
        op.run_multicast(a[r * Ms:(r + 1) * Ms], b, dest.data_ptr(), r * Ms, M, bias=bias)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, "bf16", MODE_INT, 61, 62)
    O = (O + bias.double().cpu().numpy()[None, :]).clip(min=0.0)
    check_against_oracle(dest, O, D, "bf16", exact=True, tol=0)


def test_multicast_rejects_unsupported_requests():
    a = dev_tensor((256, 128), "bf16", 1, MODE_INT)
    b = dev_tensor((128, 128), "bf16", 2, MODE_INT)
    c = torch.zeros((512, 128), dtype=torch.bfloat16, device="cuda:0")
    one = dict(ONE_CTA, tile_n=128)
    for desc, sch in ((xtc.matmul_desc(256, 128, 128), dict(one, split_k=2)),        # split-K partials
                      (xtc.matmul_desc(256, 128, 128), dict(one, buffer_c=0)),       # nothing staged
                      (xtc.matmul_desc(200, 128, 128), one)):                        # ragged shard
        op = xtc.Op(desc).apply(S(**sch))
        with pytest.raises(xtc.XtcError):
            op.run_multicast(a[:desc.m], b, c.data_ptr(), 0, 512)
    ok = xtc.Op(xtc.matmul_desc(256, 128, 128)).apply(S(**one))
    with pytest.raises(xtc.XtcError):                                                # rows past the destination
        ok.run_multicast(a, b, c.data_ptr(), 384, 512)
