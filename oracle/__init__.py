"""CPU oracle for the XTC B200 hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product package ``paper_2512_16512_b200`` never imports it (checked by
``tests/test_host.py::test_product_never_imports_oracle``), and it shares no code with the CUDA path.

The arithmetic lives in ``xtc_oracle.c`` (fp64 naive loop nests, PAPER.md
Fig.2; conv2d P:251-253/P:1152 with the zero-padding reading of
SURVEY.md §8(c) row 3).  This wrapper only marshals numpy arrays and does
the exact conversions bf16/fp32 -> fp64 on input, plus the output rounding
``round_out`` of SURVEY.md §8(c) (identity for fp32 output, RNE for bf16).

Pins (tests/test_oracle.py, all ``-m "not gpu"``): brute force on tiny
shapes, SPEC S:62's 2x2 example, identity / permutation / all-ones / rank-1
closed forms, conv delta-kernel and 4C/6C/9C padding closed forms, conv ==
explicit im2col + matmul, 1x1 conv == matmul, torch float64 conv2d.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xtc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no GPU, no nvcc involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.oracle_matmul_f64.argtypes = [i64, i64, i64, d, d, d, d]
        lib.oracle_matmul_f64.restype = None
        lib.oracle_conv2d_f64.argtypes = [i64] * 11 + [d, d, d, d]
        lib.oracle_conv2d_f64.restype = None
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def to_f64(a: np.ndarray, dtype: str) -> np.ndarray:
    """Exact widening of stored inputs: 'bf16' arrays are uint16 bit patterns."""
    if dtype == "bf16":
        f32 = (np.ascontiguousarray(a, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
        return f32.astype(np.float64)
    return np.ascontiguousarray(a, dtype=np.float32).astype(np.float64)


def matmul(A: np.ndarray, B: np.ndarray):
    """C = A @ B and D = |A| @ |B| in fp64 (Fig.2 loop nest).  A: [M,K], B: [K,N] fp64."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("inner dimensions differ")
    C = np.empty((M, N), np.float64)
    D = np.empty((M, N), np.float64)
    _load().oracle_matmul_f64(M, N, K, _p(A), _p(B), _p(C), _p(D))
    return C, D


def conv_out_hw(H, W, R, S, stride=(1, 1), pad=(0, 0)):
    """P = floor((H + 2 pad - R) / stride) + 1 (S:38 with the pad attribute)."""
    return (H + 2 * pad[0] - R) // stride[0] + 1, (W + 2 * pad[1] - S) // stride[1] + 1


def conv2d(x: np.ndarray, w: np.ndarray, stride=(1, 1), pad=(0, 0)):
    """y = conv2d(pad0(x), w): x NHWC, w RSCF, y NPQF; fp64.  Returns (y, D)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    Nb, H, W, C = x.shape
    R, S, C2, F = w.shape
    if C != C2:
        raise ValueError("channel mismatch")
    P, Q = conv_out_hw(H, W, R, S, stride, pad)
    y = np.empty((Nb, P, Q, F), np.float64)
    D = np.empty((Nb, P, Q, F), np.float64)
    _load().oracle_conv2d_f64(Nb, H, W, C, F, R, S, stride[0], stride[1], pad[0], pad[1],
                              _p(x), _p(w), _p(y), _p(D))
    return y, D


def relu(O: np.ndarray) -> np.ndarray:
    """The relu consumer op of the paper's graphs (Fig.9 matmul -> relu):
    elementwise max(x, 0) on the fp64 result, applied before round_out.
    Pinned by SPEC S:63: relu([-1, 0, 2]) = [0, 0, 2]."""
    return np.maximum(np.asarray(O, dtype=np.float64), 0.0)


def consume(O: np.ndarray, relu_: bool = False, bias=None, c_old=None) -> np.ndarray:
    """The fused consumer of the contraction (fuse), in fp64 and
    in this order: C_old + O (the accumulate flag, Fig.2's `C[i][j] +=`), + bias[n]
    broadcast over rows, then relu (above); round_out follows once.  Pinned in
    tests/test_oracle.py by [A | 1]·[B ; biasᵀ] and [A | I]·[B ; C_old] (both textbook
    block-matrix identities computed through `matmul`) and a hand example."""
    R = np.asarray(O, dtype=np.float64).copy()
    if c_old is not None:
        R = R + np.asarray(c_old, dtype=np.float64)
    if bias is not None:
        R = R + np.asarray(bias, dtype=np.float64)[None, :]
    return relu(R) if relu_ else R


def round_out(O: np.ndarray, out_dtype: str) -> np.ndarray:
    """round_out of SURVEY.md §8(c): fp32 output -> float32(O) (RN);
    bf16 output -> RNE to bf16, returned as uint16 bit patterns.
    For integer-valued O with |O| < 2^24 the fp64->fp32 step is exact, so the
    bf16 result is the single RNE rounding of O."""
    f32 = np.asarray(O, dtype=np.float64).astype(np.float32)
    if out_dtype == "f32":
        return f32
    b = f32.view(np.uint32).astype(np.uint64)
    return ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)).astype(np.uint16)


def num_threads() -> int:
    return int(_load().oracle_num_threads())
