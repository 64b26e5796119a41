"""Helpers for the -m gpu parity tests: seeded inputs on both sides, oracle
comparison.  Inputs reach the GPU through the library's own generator
(xtc_fill) and the oracle side through seeded_inputs; a dedicated test checks
the two generators agree bit for bit."""
import numpy as np
import torch

import oracle
import paper_2512_16512_b200 as xtc
from seeded_inputs import MODE_INT, gen_tensor

TORCH_DT = {"bf16": torch.bfloat16, "f32": torch.float32, "tf32": torch.float32}


def dev_tensor(shape, dtype, seed, mode, device=0):
    n = int(np.prod(shape))
    t = torch.empty(shape, dtype=TORCH_DT[dtype], device=f"cuda:{device}")
    xtc.xtc_fill(t.data_ptr(), n, xtc.DTYPES[dtype], seed, mode, 0, torch.cuda.current_stream().cuda_stream)
    return t


def to_numpy_out(c: torch.Tensor, out_dtype: str) -> np.ndarray:
    c = c.detach().cpu().contiguous()
    if out_dtype == "bf16":
        return c.view(torch.int16).numpy().view(np.uint16)
    return c.numpy()


def out_as_f64(arr: np.ndarray, out_dtype: str) -> np.ndarray:
    return oracle.to_f64(arr, "bf16" if out_dtype == "bf16" else "f32")


def oracle_matmul(M, N, K, in_dtype, mode, seed_a, seed_b):
    A = gen_tensor(seed_a, (M, K), "bf16" if in_dtype == "bf16" else "f32", mode)
    B = gen_tensor(seed_b, (K, N), "bf16" if in_dtype == "bf16" else "f32", mode)
    ia = "bf16" if in_dtype == "bf16" else "f32"
    return oracle.matmul(oracle.to_f64(A, ia), oracle.to_f64(B, ia))


def oracle_conv(d, in_dtype, mode, seed_x, seed_w):
    ia = "bf16" if in_dtype == "bf16" else "f32"
    x = gen_tensor(seed_x, (d.batch, d.h, d.w, d.c), ia, mode)
    w = gen_tensor(seed_w, (d.r, d.s, d.c, d.f), ia, mode)
    y, D = oracle.conv2d(oracle.to_f64(x, ia), oracle.to_f64(w, ia), (d.stride_h, d.stride_w), (d.pad_h, d.pad_w))
    return y.reshape(-1, d.f), D.reshape(-1, d.f)


def check_against_oracle(c_dev, O, D, out_dtype, exact, tol):
    """exact: bits(C) == bits(round_out(O)) everywhere; else max |C-O|/D <= tol."""
    got = to_numpy_out(c_dev, out_dtype).reshape(O.shape)
    if exact:
        want = oracle.round_out(O, out_dtype)
        if out_dtype == "f32":
            bad = got.view(np.uint32) != want.view(np.uint32)
        else:
            bad = got != want
        nbad = int(bad.sum())
        if nbad:
            i, j = np.argwhere(bad)[0]
            raise AssertionError(f"{nbad} mismatches; first at ({i},{j}): got {out_as_f64(got, out_dtype)[i, j]} "
                                 f"want {O[i, j]}")
        return 0.0
    g = out_as_f64(got, out_dtype)
    assert np.all(np.isfinite(g)), "non-finite output"
    with np.errstate(divide="ignore", invalid="ignore"):
        err = np.where(D > 0, np.abs(g - O) / D, np.where(g == O, 0.0, np.inf))
    e = float(err.max())
    assert e <= tol, f"max normalised error {e} > {tol} at {np.unravel_index(err.argmax(), err.shape)}"
    return e


def run_matmul(M, N, K, in_dtype, out_dtype, sch, mode, seed=0, measure=True, exact=None, tol=None):
    """Runs one schedule through the C-ABI and checks it element by element
    against the CPU oracle; also checks the library's own on-chip validation."""
    desc = xtc.matmul_desc(M, N, K, in_dtype, out_dtype)
    a = dev_tensor((M, K), in_dtype, seed, mode)
    b = dev_tensor((K, N), in_dtype, seed + 1, mode)
    c = torch.full((M, N), float("nan"), dtype=TORCH_DT[out_dtype], device="cuda:0")
    op = xtc.Op(desc).apply(sch)
    op.run(a, b, c)
    torch.cuda.synchronize()
    O, D = oracle_matmul(M, N, K, in_dtype, mode, seed, seed + 1)
    if exact is None:
        exact = mode == 1
    if tol is None:
        tol = 1e-5 if in_dtype == "f32" else 5e-3
    err = check_against_oracle(c, O, D, out_dtype, exact, tol)
    m = None
    if measure:
        m = op.measure(a, b, c, xtc.measure_cfg(warmup=1, repeats=3, validate=1, exact=int(exact), tol=tol))
        assert m.valid == 1, m.as_dict()
        assert m.n_nan == 0
        if exact:
            assert m.n_mismatch == 0
    return err, m


def run_conv(d, in_dtype, out_dtype, sch, mode, seed=10):
    x = dev_tensor((d.batch, d.h, d.w, d.c), in_dtype, seed, mode)
    w = dev_tensor((d.r, d.s, d.c, d.f), in_dtype, seed + 1, mode)
    M, N, K = xtc.gemm_view(d)
    y = torch.full((M, N), float("nan"), dtype=TORCH_DT[out_dtype], device="cuda:0")
    op = xtc.Op(d).apply(sch)
    op.run(x, w, y)
    torch.cuda.synchronize()
    O, D = oracle_conv(d, in_dtype, mode, seed, seed + 1)
    exact = mode == MODE_INT
    tol = 1e-5 if in_dtype == "f32" else 5e-3
    err = check_against_oracle(y, O, D, out_dtype, exact, tol)
    m = op.measure(x, w, y, xtc.measure_cfg(warmup=1, repeats=2, validate=1, exact=int(exact), tol=tol))
    assert m.valid == 1, m.as_dict()
    return err
