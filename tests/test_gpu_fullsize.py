"""-m gpu: oracle parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

  * config 5's 8192^3 bf16 matmul with bench.HEADLINE_SCHEDULE (CTA pair, two M-subtiles, overlapped
    epilogue; 512 tiles over 74 pairs = 7 tiles per pair): the CPU oracle on 64 sampled output rows (one in
    every 128-row UMMA subtile, at varying lanes) and on 4096 random elements, bit-exact on integer data
    and within 5e-3 of D on uniform data; plus the library's on-chip validation of the whole output;
  * config 3's ResNet-50 layers at batch 32 (L56: 56x56x64 -> 64, L14: 14x14x256 -> 256, 3x3 s1 p1) with the
    bench's schedules, against the full CPU oracle;
  * config 4's sweep: the bench's 4096 seeded candidates at 1024^3, every one run on integer data with
    exact = 1 (BASELINE north_star: every legal schedule bit-identical).

The Executor contract: PAPER.md P:792-795 (§IV-B).  BASELINE.md §5 plans the sampled-row check.
"""
import numpy as np
import pytest
import torch

import bench
import oracle
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import CONV_SCHEDS
from paper_2512_16512_b200.strategy import GpuStrategy
from seeded_inputs import MODE_INT, MODE_UNIFORM, gen_rows, gen_tensor
from gpu_util import TORCH_DT, check_against_oracle, dev_tensor, run_conv, to_numpy_out

pytestmark = pytest.mark.gpu

MODES = [MODE_INT, MODE_UNIFORM]


def sampled_rows(M, n=64, sub=128):
    """n rows, one per 128-row UMMA subtile block (spread over all of them), at varying lanes."""
    blocks = M // sub
    return [min(M - 1, (i * blocks // n) * sub + (37 * i + 5) % sub) for i in range(n)]


def tiles_per_pair(desc, sch):
    st, info, why = xtc.xtc_schedule_check(desc, sch, 148)
    assert st == 0, why
    return -(-int(info.num_tiles) // (info.grid_x // max(1, info.cluster_x)))


@pytest.mark.parametrize("mode", MODES)
def test_headline_8192_sampled_rows_and_random_elements(mode):
    M = N = K = 8192
    seed = 101
    desc = xtc.matmul_desc(M, N, K, "bf16", "bf16")
    sch = xtc.schedule(**bench.HEADLINE_SCHEDULE)
    assert tiles_per_pair(desc, sch) == 7            # the bench's launch configuration
    a = dev_tensor((M, K), "bf16", seed, mode)
    b = dev_tensor((K, N), "bf16", seed + 1, mode)
    c = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda:0")
    op = xtc.Op(desc).apply(sch)
    op.run(a, b, c)
    torch.cuda.synchronize()
    exact = mode == MODE_INT
    # 64 sampled rows, full N, full K
    rows = sampled_rows(M)
    B = oracle.to_f64(gen_tensor(seed + 1, (K, N), "bf16", mode), "bf16")
    Ar = oracle.to_f64(gen_rows(seed, (M, K), rows, "bf16", mode), "bf16")
    O, D = oracle.matmul(Ar, B)
    check_against_oracle(c[rows], O, D, "bf16", exact, 5e-3)
    # 4096 random elements (grouped by row: the oracle over that row and the sampled columns)
    rng = np.random.default_rng(7)
    ii = rng.integers(0, M, 4096)
    jj = rng.integers(0, N, 4096)
    got_all = to_numpy_out(c, "bf16")
    uniq = np.unique(ii)
    A_u = oracle.to_f64(gen_rows(seed, (M, K), uniq, "bf16", mode), "bf16")
    for r_idx, i in enumerate(uniq):
        cols = jj[ii == i]
        Oe, De = oracle.matmul(A_u[r_idx:r_idx + 1], np.ascontiguousarray(B[:, cols]))
        got = got_all[i, cols][None, :]
        if exact:
            assert np.array_equal(got, oracle.round_out(Oe, "bf16")), (i, cols)
        else:
            g = oracle.to_f64(got, "bf16")
            assert np.max(np.abs(g - Oe) / De) <= 5e-3, (i, cols)
    # the library's own on-chip validation of all 67M outputs (fp64 GPU reference)
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=0, repeats=1, validate=1, exact=int(exact)))
    assert m.valid == 1 and m.n_nan == 0, m.as_dict()
    if exact:
        assert m.n_mismatch == 0


# (layer, index into the bench's candidate list, tiles per persistent CTA / pair at batch 32):
# L56 compact rows: 32 x 26 = 832 tiles over 148 CTAs (6 per CTA); L56 power-of-two rows: 896 tiles (7);
# L14's CTA-pair schedule: 64 pair tiles for 74 pairs (one each; its multi-tile form is in test_gpu_multitile.py)
@pytest.mark.parametrize("layer,idx,per_cta", [("L56", 0, 6), ("L56", 1, 7), ("L14", 0, 1)])
@pytest.mark.parametrize("mode", MODES)
def test_conv_resnet_layers_batch32_bench_schedule(layer, idx, per_cta, mode):
    h, c = {"L56": (56, 64), "L14": (14, 256)}[layer]
    d = xtc.conv2d_desc(32, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
    sch = xtc.schedule(**CONV_SCHEDS[layer][idx])
    assert tiles_per_pair(d, sch) == per_cta
    run_conv(d, "bf16", "bf16", sch, mode, seed=111)


def test_sweep_4096_candidates_integer_bit_exact():
    """The bench's 4096-candidate sweep (1024^3 bf16, seed 0, the legal set of GpuStrategy's slots), each
    candidate validated on integer data with exact = 1 against the on-chip fp64 reference, which itself
    equals the CPU oracle (checked on the output the last candidate left behind)."""
    n = 1024
    desc = xtc.matmul_desc(n, n, n, "bf16", "bf16")
    strat = GpuStrategy(desc)
    cands = [strat.generate(s) for s in strat.sample(4096, seed=0)]
    a = dev_tensor((n, n), "bf16", 121, MODE_INT)
    b = dev_tensor((n, n), "bf16", 122, MODE_INT)
    c = torch.empty((n, n), dtype=torch.bfloat16, device="cuda:0")
    recs = xtc.Op(desc).sweep(cands, a, b, c, xtc.measure_cfg(warmup=0, repeats=1, validate=1, exact=1))
    bad = [(i, r.status, r.valid, r.n_mismatch, r.n_nan) for i, r in enumerate(recs)
           if r.status != 0 or r.valid != 1 or r.n_mismatch != 0 or r.n_nan != 0]
    assert not bad, (len(bad), bad[:5])
    A = oracle.to_f64(gen_tensor(121, (n, n), "bf16", MODE_INT), "bf16")
    B = oracle.to_f64(gen_tensor(122, (n, n), "bf16", MODE_INT), "bf16")
    O, D = oracle.matmul(A, B)
    check_against_oracle(c, O, D, "bf16", True, 0.0)
