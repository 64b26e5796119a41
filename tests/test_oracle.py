"""Pins for the CPU oracle (``-m "not gpu"``).

Each test ties ``oracle/`` to something other than itself: values printed in
SPEC/PAPER worked examples (tests/golden/), closed forms, textbook special
cases, an exactly-rounded brute force, or a library routine (numpy / torch
float64).  Chosen so a dropped term, wrong sign/index or transposed operand
fails at least one of them (see the 'mutants' test at the bottom).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from seeded_inputs import MODE_INT, MODE_UNIFORM, gen_f32

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- matmul ----

def _pin_spec_2x2_worked_example(o):
    g = _golden("spec_2x2_matmul.json")
    C, D = o.matmul(np.array(g["A"], float), np.array(g["B"], float))
    assert C.tolist() == g["C"]
    # all entries positive, so sum |a||b| equals the product itself
    assert D.tolist() == g["C"]


def _pin_identity_and_permutation_closed_forms(o):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((7, 5))
    C, _ = o.matmul(A, np.eye(5))
    assert np.array_equal(C, A)                       # A I = A
    C, _ = o.matmul(np.eye(7), A)
    assert np.array_equal(C, A)                       # I A = A
    perm = rng.permutation(5)
    Pm = np.zeros((5, 5))
    Pm[perm, np.arange(5)] = 1.0                      # column j of A P = column perm[j] of A
    C, _ = o.matmul(A, Pm)
    assert np.array_equal(C, A[:, perm])


def _pin_all_ones_and_rank1_closed_forms(o):
    M, N, K = 6, 9, 13
    C, D = o.matmul(np.ones((M, K)), np.ones((K, N)))
    assert np.all(C == K) and np.all(D == K)
    u = np.arange(1, M + 1, dtype=float) * (-1) ** np.arange(M)
    v = np.arange(2, N + 2, dtype=float)
    A = np.repeat(u[:, None], K, axis=1)              # A[i,k] = u_i
    B = np.repeat(v[None, :], K, axis=0)              # B[k,j] = v_j
    C, D = o.matmul(A, B)
    assert np.array_equal(C, K * np.outer(u, v))
    assert np.array_equal(D, K * np.outer(np.abs(u), np.abs(v)))


def _pin_brute_force_exact_on_integer_data(o):
    """Exact Python-integer brute force, non-square shapes (catches transposes)."""
    for (M, N, K) in [(1, 1, 1), (3, 4, 5), (5, 3, 7), (8, 2, 9)]:
        A = gen_f32(11, M * K, MODE_INT).reshape(M, K).astype(int)
        B = gen_f32(12, K * N, MODE_INT).reshape(K, N).astype(int)
        C, D = o.matmul(A.astype(float), B.astype(float))
        for i in range(M):
            for j in range(N):
                assert C[i, j] == sum(int(A[i, k]) * int(B[k, j]) for k in range(K))
                assert D[i, j] == sum(abs(int(A[i, k])) * abs(int(B[k, j])) for k in range(K))


def _pin_exactly_rounded_sum_on_float_data(o):
    """fp64 summation error bound: |C - exact| <= K * 2^-53 * D (summation only;
    products of fp32 inputs are exact in fp64)."""
    M, N, K = 4, 5, 257
    A = gen_f32(21, M * K).reshape(M, K).astype(np.float64)
    B = gen_f32(22, K * N).reshape(K, N).astype(np.float64)
    C, D = o.matmul(A, B)
    for i in range(M):
        for j in range(N):
            exact = sum(Fraction(A[i, k]) * Fraction(B[k, j]) for k in range(K))
            assert abs(Fraction(C[i, j]) - exact) <= Fraction(K) * Fraction(2) ** -53 * Fraction(D[i, j])
            assert D[i, j] == pytest.approx(math.fsum(abs(A[i, k] * B[k, j]) for k in range(K)), rel=1e-14)


def _pin_numpy_float64_matmul_agrees(o):
    M, N, K = 33, 47, 129
    A = gen_f32(31, M * K).reshape(M, K).astype(np.float64)
    B = gen_f32(32, K * N).reshape(K, N).astype(np.float64)
    C, D = o.matmul(A, B)
    ref = A @ B
    assert np.max(np.abs(C - ref) / D) < 1e-14
    assert np.allclose(D, np.abs(A) @ np.abs(B), rtol=1e-14, atol=0)


def _pin_paper_fig2_shape_256x258x512_integer(o):
    """The paper's running example I=256, J=258, K=512, integer data,
    checked against exact integer numpy matmul (int64 has no rounding)."""
    A = gen_f32(41, 256 * 512, MODE_INT).reshape(256, 512)
    B = gen_f32(42, 512 * 258, MODE_INT).reshape(512, 258)
    C, _ = o.matmul(A, B)
    assert np.array_equal(C.astype(np.int64), A.astype(np.int64) @ B.astype(np.int64))


# ---------------------------------------------------------------- conv2d ----

def _pin_conv_output_shapes_golden(o):  # pure shape formula (Python), no C to mutate
    g = _golden("conv_shapes.json")
    for c in g["cases"]:
        P, Q = oracle.conv_out_hw(c["H"], c["W"], c["R"], c["S"], (c["stride"],) * 2, (c["pad"],) * 2)
        assert (P, Q) == (c["P"], c["Q"])


def _pin_conv_delta_kernel_is_identity(o):
    x = gen_f32(51, 2 * 5 * 6 * 3).reshape(2, 5, 6, 3).astype(np.float64)
    w = np.zeros((3, 3, 3, 3))
    for c in range(3):
        w[1, 1, c, c] = 1.0                            # w[r,s,c,f] = [r=1][s=1][c=f]
    y, _ = o.conv2d(x, w, (1, 1), (1, 1))
    assert np.array_equal(y, x)


def _pin_conv_all_ones_padding_closed_form(o):
    """All-ones x, w, 3x3, pad 1: interior 9C, edges 6C, corners 4C."""
    N, H, W, C, F = 1, 5, 7, 4, 2
    y, D = o.conv2d(np.ones((N, H, W, C)), np.ones((3, 3, C, F)), (1, 1), (1, 1))
    expect = np.full((H, W), 9.0 * C)
    expect[0, :] = expect[-1, :] = 6.0 * C
    expect[:, 0] = expect[:, -1] = 6.0 * C
    expect[0, 0] = expect[0, -1] = expect[-1, 0] = expect[-1, -1] = 4.0 * C
    for f in range(F):
        assert np.array_equal(y[0, :, :, f], expect)
    assert np.array_equal(D, y)


def _pin_conv_1x1_equals_matmul(o):
    N, H, W, C, F = 2, 3, 4, 5, 6
    x = gen_f32(61, N * H * W * C, MODE_INT).reshape(N, H, W, C).astype(np.float64)
    w = gen_f32(62, C * F, MODE_INT).reshape(1, 1, C, F).astype(np.float64)
    y, _ = o.conv2d(x, w)
    ref = x.reshape(-1, C).astype(np.int64) @ w.reshape(C, F).astype(np.int64)
    assert np.array_equal(y.reshape(-1, F), ref)


def _im2col(x, R, S, stride, pad):
    N, H, W, C = x.shape
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    xp = np.zeros((N, H + 2 * pad, W + 2 * pad, C), x.dtype)
    xp[:, pad:pad + H, pad:pad + W, :] = x
    cols = np.zeros((N, P, Q, R, S, C), x.dtype)
    for r in range(R):
        for s in range(S):
            cols[:, :, :, r, s, :] = xp[:, r:r + stride * P:stride, s:s + stride * Q:stride, :]
    return cols.reshape(N * P * Q, R * S * C), (N, P, Q)


def _pin_conv_equals_explicit_im2col_matmul_integer(o):
    for stride, pad in [(1, 1), (2, 0), (2, 3), (1, 0)]:
        N, H, W, C, F, R, S = 2, 9, 8, 3, 4, 3, 3
        if pad == 3:
            R = S = 7
        x = gen_f32(71, N * H * W * C, MODE_INT).reshape(N, H, W, C)
        w = gen_f32(72, R * S * C * F, MODE_INT).reshape(R, S, C, F)
        y, _ = o.conv2d(x, w, (stride, stride), (pad, pad))
        cols, (n, P, Q) = _im2col(x.astype(np.int64), R, S, stride, pad)
        ref = cols @ w.reshape(R * S * C, F).astype(np.int64)
        assert np.array_equal(y.reshape(-1, F).astype(np.int64), ref), (stride, pad)


def _pin_conv_matches_torch_float64(o):
    torch = pytest.importorskip("torch")
    N, H, W, C, F = 2, 14, 14, 8, 5
    x = gen_f32(81, N * H * W * C).reshape(N, H, W, C).astype(np.float64)
    w = gen_f32(82, 3 * 3 * C * F).reshape(3, 3, C, F).astype(np.float64)
    for stride, pad in [(1, 1), (2, 1)]:
        y, D = o.conv2d(x, w, (stride, stride), (pad, pad))
        ref = torch.nn.functional.conv2d(
            torch.from_numpy(x).permute(0, 3, 1, 2),             # NHWC -> NCHW
            torch.from_numpy(w).permute(3, 2, 0, 1),             # RSCF -> FCRS
            stride=stride, padding=pad).permute(0, 2, 3, 1).numpy()
        assert y.shape == ref.shape
        assert np.max(np.abs(y - ref) / D) < 1e-14



def test_spec_2x2_worked_example():
    _pin_spec_2x2_worked_example(oracle)

def test_identity_and_permutation_closed_forms():
    _pin_identity_and_permutation_closed_forms(oracle)

def test_all_ones_and_rank1_closed_forms():
    _pin_all_ones_and_rank1_closed_forms(oracle)

def test_brute_force_exact_on_integer_data():
    _pin_brute_force_exact_on_integer_data(oracle)

def test_exactly_rounded_sum_on_float_data():
    _pin_exactly_rounded_sum_on_float_data(oracle)

def test_numpy_float64_matmul_agrees():
    _pin_numpy_float64_matmul_agrees(oracle)

def test_paper_fig2_shape_256x258x512_integer():
    _pin_paper_fig2_shape_256x258x512_integer(oracle)

def test_conv_output_shapes_golden():
    _pin_conv_output_shapes_golden(oracle)

def test_conv_delta_kernel_is_identity():
    _pin_conv_delta_kernel_is_identity(oracle)

def test_conv_all_ones_padding_closed_form():
    _pin_conv_all_ones_padding_closed_form(oracle)

def test_conv_1x1_equals_matmul():
    _pin_conv_1x1_equals_matmul(oracle)

def test_conv_equals_explicit_im2col_matmul_integer():
    _pin_conv_equals_explicit_im2col_matmul_integer(oracle)

def test_conv_matches_torch_float64():
    _pin_conv_matches_torch_float64(oracle)


PINS = [_pin_spec_2x2_worked_example, _pin_identity_and_permutation_closed_forms, _pin_all_ones_and_rank1_closed_forms, _pin_brute_force_exact_on_integer_data, _pin_exactly_rounded_sum_on_float_data, _pin_numpy_float64_matmul_agrees, _pin_paper_fig2_shape_256x258x512_integer, _pin_conv_output_shapes_golden, _pin_conv_delta_kernel_is_identity, _pin_conv_all_ones_padding_closed_form, _pin_conv_1x1_equals_matmul, _pin_conv_equals_explicit_im2col_matmul_integer, _pin_conv_matches_torch_float64]


# --------------------------------------------------------------- rounding ---

def test_round_out_bf16_matches_torch_rne():
    torch = pytest.importorskip("torch")
    vals = np.concatenate([gen_f32(91, 4096).astype(np.float64) * 300.0,
                           np.arange(-40000, 40000, 7, dtype=np.float64)])
    vals32 = vals.astype(np.float32).astype(np.float64)   # torch path: f32 -> bf16
    ours = oracle.round_out(vals32, "bf16")
    ref = torch.from_numpy(vals32.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    assert np.array_equal(oracle.round_out(vals, "f32"), vals.astype(np.float32))


# ---------------------------------------------------------------- mutants ---

class _CompiledOracle:
    """oracle.matmul / oracle.conv2d over a given C source (compiled with the oracle's own flags):
    the same marshalling as oracle/__init__.py, so a mutated copy of xtc_oracle.c can be run
    against the real pins above."""

    def __init__(self, src: str, tmpdir: str, tag: str):
        import ctypes
        import subprocess
        c_path = os.path.join(tmpdir, f"oracle_{tag}.c")
        so_path = os.path.join(tmpdir, f"liboracle_{tag}.so")
        with open(c_path, "w") as f:
            f.write(src)
        subprocess.check_call(["gcc", *oracle.CFLAGS, "-o", so_path, c_path, "-lm"])
        lib = ctypes.CDLL(so_path)
        d = ctypes.POINTER(ctypes.c_double)
        lib.oracle_matmul_f64.argtypes = [ctypes.c_int64] * 3 + [d] * 4
        lib.oracle_conv2d_f64.argtypes = [ctypes.c_int64] * 11 + [d] * 4
        self.lib, self._d = lib, d

    def _p(self, a):
        return a.ctypes.data_as(self._d)

    def matmul(self, A, B):
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        (M, K), (_, N) = A.shape, B.shape
        C, D = np.zeros((M, N)), np.zeros((M, N))
        self.lib.oracle_matmul_f64(M, N, K, self._p(A), self._p(B), self._p(C), self._p(D))
        return C, D

    def conv2d(self, x, w, stride=(1, 1), pad=(0, 0)):
        x = np.ascontiguousarray(x, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        Nb, H, W, C = x.shape
        R, S, _, F = w.shape
        P, Q = oracle.conv_out_hw(H, W, R, S, stride, pad)
        y, D = np.zeros((Nb, P, Q, F)), np.zeros((Nb, P, Q, F))
        self.lib.oracle_conv2d_f64(Nb, H, W, C, F, R, S, stride[0], stride[1], pad[0], pad[1],
                                   self._p(x), self._p(w), self._p(y), self._p(D))
        return y, D


# (name, text in xtc_oracle.c, replacement): plausible slips in the loop nests, each kept in bounds
ORACLE_MUTANTS = [
    ("matmul: B transposed", "double b = B[k * N + j];", "double b = B[j * K + k];"),
    ("matmul: A transposed", "double a = A[i * K + k];", "double a = A[k * M + i];"),
    ("matmul: last k term dropped", "for (int64_t k = 0; k < K; k++)", "for (int64_t k = 0; k < K - 1; k++)"),
    ("matmul: first k term dropped", "for (int64_t k = 0; k < K; k++)", "for (int64_t k = 1; k < K; k++)"),
    ("matmul: wrong sign", "s += a * b;", "s -= a * b;"),
    ("matmul: accumulates into a non-zero C", "double s = 0.0, d = 0.0;", "double s = 1.0, d = 0.0;"),
    ("matmul: output stored transposed", "C[i * N + j] = s;", "C[j * M + i] = s;"),
    ("matmul: D without |.|", "d += fabs(a) * fabs(b);", "d += a * b;"),
    ("conv: pad added instead of subtracted", "int64_t h = p * sh + r - ph;", "int64_t h = p * sh + r + ph;"),
    ("conv: stride dropped on q", "int64_t ww = q * sw + s - pw;", "int64_t ww = q + s - pw;"),
    ("conv: filter flipped (convolution vs correlation)", "double wv = w[((r * S + s) * C + c) * F + f];",
     "double wv = w[(((R - 1 - r) * S + (S - 1 - s)) * C + c) * F + f];"),
    ("conv: filter r/s transposed", "double wv = w[((r * S + s) * C + c) * F + f];",
     "double wv = w[((s * R + r) * C + c) * F + f];"),
    ("conv: last channel dropped", "for (int64_t c = 0; c < C; c++)", "for (int64_t c = 0; c < C - 1; c++)"),
    ("conv: output p/q transposed", "int64_t o = ((n * P + p) * Q + q) * F + f;",
     "int64_t o = ((n * Q + q) * P + p) * F + f;"),
    ("conv: zero pad as edge clamp", "double xv = 0.0;           /* the padding op's zero fill */\n"
     "                            if (h >= 0 && h < H && ww >= 0 && ww < W)\n"
     "                                xv = x[((n * H + h) * W + ww) * C + c];",
     "int64_t hc = h < 0 ? 0 : (h >= H ? H - 1 : h), wc = ww < 0 ? 0 : (ww >= W ? W - 1 : ww);\n"
     "                            double xv = x[((n * H + hc) * W + wc) * C + c];"),
]


def _failing_pins(o):
    bad = []
    for pin in PINS:
        try:
            pin(o)
        except AssertionError:
            bad.append(pin.__name__)
    return bad


def test_pins_reject_plausible_mutants(tmp_path):
    """Mutated copies of the oracle's C source (the real arithmetic, compiled) each fail at least
    one pin above, while the unmutated source -- compiled the same way -- passes them all."""
    src = open(os.path.join(os.path.dirname(oracle.__file__), "xtc_oracle.c")).read()
    assert _failing_pins(_CompiledOracle(src, str(tmp_path), "orig")) == []
    for i, (name, old, new) in enumerate(ORACLE_MUTANTS):
        assert src.count(old) == 1, f"mutant {name!r}: pattern not found once in xtc_oracle.c"
        failing = _failing_pins(_CompiledOracle(src.replace(old, new), str(tmp_path), f"m{i}"))
        assert failing, f"mutant {name!r} passes every pin"


# ---------------------------------------------------------------- widening ---
def test_to_f64_bf16_known_bit_patterns():
    """bf16 widening is the top half of an IEEE fp32 (bf16 = fp32 with 16 mantissa bits dropped):
    known patterns, including signed zero, a subnormal, the largest finite value and infinities."""
    cases = {0x0000: 0.0, 0x8000: -0.0, 0x3F80: 1.0, 0xBF80: -1.0, 0x4000: 2.0, 0x3F81: 1.0 + 2.0 ** -7,
             0x4049: 3.140625, 0x4120: 10.0, 0xC2F7: -123.5, 0x3C00: 2.0 ** -7, 0x0001: 2.0 ** -133,
             0x0080: 2.0 ** -126, 0x7F7F: (2.0 - 2.0 ** -7) * 2.0 ** 127, 0x7F80: math.inf, 0xFF80: -math.inf}
    bits = np.array(list(cases), dtype=np.uint16)
    got = oracle.to_f64(bits, "bf16")
    for b, g in zip(cases, got):
        want = cases[b]
        assert g == want and math.copysign(1.0, g) == math.copysign(1.0, want), (hex(b), g, want)
    assert np.isnan(oracle.to_f64(np.array([0x7FC0], np.uint16), "bf16")[0])
    # fp32 storage widens exactly (every fp32 is an fp64)
    f = np.array([1.0, -2.5, 2.0 ** -149, 3.4028234663852886e38, 0.1], np.float32)
    assert np.array_equal(oracle.to_f64(f, "f32"), f.astype(np.float64))
    assert oracle.to_f64(np.array([0.1], np.float32), "f32")[0] == 0.100000001490116119384765625


def test_relu_spec_worked_example():
    g = _golden("spec_relu.json")
    assert oracle.relu(np.array(g["x"], float)).tolist() == g["y"]
    # relu(matmul) closed form on a rank-1 product with mixed signs: K * max(u_i v_j, 0)
    u = np.array([1.0, -2.0, 3.0])
    v = np.array([-1.0, 2.0])
    C, _ = oracle.matmul(np.repeat(u[:, None], 4, 1), np.repeat(v[None, :], 4, 0))
    assert np.array_equal(oracle.relu(C), 4 * np.maximum(np.outer(u, v), 0))


# --------------------------------------------- consumer: bias / accumulate --
def test_consume_bias_is_an_augmented_matmul():
    """C + 1·biasᵀ = [A | 1] · [B ; biasᵀ] (block-matrix identity, computed through matmul)."""
    rng = np.random.default_rng(3)
    A = rng.integers(-2, 3, (7, 5)).astype(np.float64)
    B = rng.integers(-2, 3, (5, 6)).astype(np.float64)
    bias = rng.integers(-9, 10, 6).astype(np.float64)
    C, _ = oracle.matmul(A, B)
    aug, _ = oracle.matmul(np.hstack([A, np.ones((7, 1))]), np.vstack([B, bias[None, :]]))
    assert np.array_equal(oracle.consume(C, bias=bias), aug)


def test_consume_accumulate_is_an_augmented_matmul():
    """C_old + A·B = [A | I] · [B ; C_old] (Fig.2's C[i][j] += ...)."""
    rng = np.random.default_rng(4)
    A = rng.integers(-2, 3, (6, 4)).astype(np.float64)
    B = rng.integers(-2, 3, (4, 5)).astype(np.float64)
    Cold = rng.integers(-20, 21, (6, 5)).astype(np.float64)
    C, _ = oracle.matmul(A, B)
    aug, _ = oracle.matmul(np.hstack([A, np.eye(6)]), np.vstack([B, Cold]))
    assert np.array_equal(oracle.consume(C, c_old=Cold), aug)


def test_consume_order_hand_example():
    """relu is applied last, after C_old and bias: relu([[-3, 1]] + [[1, 0]] + [2, -5]) = [[0, 0]],
    while without relu = [[0, -4]]; and with A = 0 the output is relu(C_old + bias) broadcast."""
    O = np.array([[-3.0, 1.0]])
    assert oracle.consume(O, relu_=True, bias=[2.0, -5.0], c_old=[[1.0, 0.0]]).tolist() == [[0.0, 0.0]]
    assert oracle.consume(O, relu_=False, bias=[2.0, -5.0], c_old=[[1.0, 0.0]]).tolist() == [[0.0, -4.0]]
    assert oracle.consume(O, relu_=True, bias=[2.0, 5.0]).tolist() == [[0.0, 6.0]]
    Z, _ = oracle.matmul(np.zeros((3, 4)), np.ones((4, 2)))
    assert oracle.consume(Z, relu_=True, bias=[-1.0, 7.0]).tolist() == [[0.0, 7.0]] * 3
