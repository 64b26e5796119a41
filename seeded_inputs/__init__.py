"""Seeded synthetic input generator shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no contraction, no convolution,
no rounding of results).  It only turns (seed, element index) into an input
value, so that the CPU oracle (``oracle/``) and the GPU path
(``xtc_fill`` in ``include/xtc.h``) can regenerate bit-identical operands
without ever exchanging data.  The CUDA side implements the *same*
counter-based generator independently in ``paper_2512_16512_b200/csrc``;
``tests/test_gpu_parity.py::test_gpu_generator_matches_seeded_inputs`` checks the two agree bit for bit.

Generator (SURVEY.md §8(c) reading 9):

    h(seed, i)  = splitmix64(seed * 0xD1B54A32D192ED03 + i)        (mod 2^64)
    INT mode    : v = ((h >> 32) mod 5) - 2            in {-2,-1,0,1,2}
    UNIFORM mode: v = (h >> 40) * 2^-23 - 1            in [-1, 1), exact in fp32
    bf16 storage: round-to-nearest-even of the fp32 value (integers are exact)

Values are produced as fp32 (or bf16 bit patterns as uint16) in row-major
element order of the tensor they fill.
"""
from __future__ import annotations

import numpy as np

MODE_UNIFORM = 0
MODE_INT = 1

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_SEEDMUL = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def hash_u64(seed: int, start: int, count: int) -> np.ndarray:
    """Raw 64-bit hashes h(seed, i) for i in [start, start+count)."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _SEEDMUL + idx
    return _splitmix64(key)


def gen_f32(seed: int, count: int, mode: int = MODE_UNIFORM, start: int = 0) -> np.ndarray:
    """fp32 values for elements [start, start+count) of a tensor filled with ``seed``."""
    h = hash_u64(seed, start, count)
    if mode == MODE_INT:
        v = ((h >> np.uint64(32)) % np.uint64(5)).astype(np.int64) - 2
        return v.astype(np.float32)
    if mode == MODE_UNIFORM:
        u = (h >> np.uint64(40)).astype(np.float64)
        return (u * 2.0 ** -23 - 1.0).astype(np.float32)
    raise ValueError(f"unknown mode {mode}")


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round to nearest even (finite inputs only)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(u: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(u, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen_bf16_bits(seed: int, count: int, mode: int = MODE_UNIFORM, start: int = 0) -> np.ndarray:
    """bf16 bit patterns (uint16) for elements [start, start+count)."""
    return f32_to_bf16_bits(gen_f32(seed, count, mode, start))


def gen_tensor(seed: int, shape, dtype: str, mode: int = MODE_UNIFORM) -> np.ndarray:
    """A whole row-major tensor.  dtype 'f32' -> float32 array; 'bf16' -> uint16 bit array."""
    n = int(np.prod(shape)) if len(shape) else 1
    if dtype in ("f32", "tf32"):
        return gen_f32(seed, n, mode).reshape(shape)
    if dtype == "bf16":
        return gen_bf16_bits(seed, n, mode).reshape(shape)
    raise ValueError(dtype)


def gen_rows(seed: int, shape2d, rows, dtype: str, mode: int = MODE_UNIFORM) -> np.ndarray:
    """Selected rows of a row-major 2-D tensor, without generating the rest."""
    m, n = shape2d
    out = []
    for r in rows:
        if dtype == "bf16":
            out.append(gen_bf16_bits(seed, n, mode, start=int(r) * n))
        else:
            out.append(gen_f32(seed, n, mode, start=int(r) * n))
    return np.stack(out)
