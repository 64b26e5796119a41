"""The seeded generator: a pure-Python-integer restatement of its docstring
definition must agree bit for bit with the vectorised numpy version."""
import numpy as np

from seeded_inputs import (MODE_INT, MODE_UNIFORM, bf16_bits_to_f32, f32_to_bf16_bits,
                           gen_bf16_bits, gen_f32, gen_rows, hash_u64)

MASK = (1 << 64) - 1


def _splitmix(x):
    z = (x + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def _h(seed, i):
    return _splitmix((seed * 0xD1B54A32D192ED03 + i) & MASK)


def test_hash_matches_python_integers():
    for seed in (0, 1, 7, 123456789):
        h = hash_u64(seed, 1000, 64)
        assert [int(v) for v in h] == [_h(seed, 1000 + i) for i in range(64)]


def test_modes_match_definition():
    seed = 5
    f = gen_f32(seed, 256, MODE_UNIFORM)
    i = gen_f32(seed, 256, MODE_INT)
    for k in range(256):
        h = _h(seed, k)
        assert float(f[k]) == (h >> 40) * 2.0 ** -23 - 1.0
        assert float(i[k]) == ((h >> 32) % 5) - 2


def test_ranges_and_determinism():
    f = gen_f32(3, 1 << 16)
    assert f.min() >= -1.0 and f.max() < 1.0 and abs(float(f.mean())) < 0.02
    i = gen_f32(3, 1 << 16, MODE_INT)
    assert set(np.unique(i).tolist()) == {-2.0, -1.0, 0.0, 1.0, 2.0}
    assert np.array_equal(gen_f32(3, 100), gen_f32(3, 100))
    assert not np.array_equal(gen_f32(3, 100), gen_f32(4, 100))
    # offset generation equals slicing
    assert np.array_equal(gen_f32(9, 50, start=70), gen_f32(9, 120)[70:])
    rows = gen_rows(9, (10, 12), [3, 7], "f32")
    assert np.array_equal(rows, gen_f32(9, 120).reshape(10, 12)[[3, 7]])


def test_bf16_rne_and_integers_exact():
    i = gen_f32(4, 1000, MODE_INT)
    assert np.array_equal(bf16_bits_to_f32(f32_to_bf16_bits(i)), i)
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -8 + 2 ** -20], np.float32)
    # ties to even: 1+2^-8 -> 1.0 ; 1+3*2^-8 -> 1+2^-6 ; above the tie rounds up
    assert bf16_bits_to_f32(f32_to_bf16_bits(x)).tolist() == [1.0, 1.0 + 2 ** -6, 1.0 + 2 ** -7]
    b = gen_bf16_bits(4, 1000)
    assert np.array_equal(b, f32_to_bf16_bits(gen_f32(4, 1000)))
