"""256-bit regime arithmetic (csrc/wide.cuh) against Python integers, through
the library's host-side self-test export (no GPU needed)."""
from __future__ import annotations

import ctypes
import random

import numpy as np
import pytest

from paper_2601_21552_b200 import _lib

M256 = (1 << 256) - 1


def to_words(v):
    u = v & M256
    return np.array([(u >> (64 * i)) & ((1 << 64) - 1) for i in range(4)], dtype=np.uint64).view(np.int64)


def from_words(w):
    u = sum(int(x) << (64 * i) for i, x in enumerate(w.view(np.uint64)))
    return u - (1 << 256) if u >> 255 else u


def op(code, a, b):
    L = _lib.lib()
    L.oob_selftest_i256.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 3
    wa, wb, out = to_words(a), to_words(b), np.zeros(4, dtype=np.int64)
    assert L.oob_selftest_i256(code, wa.ctypes.data, wb.ctypes.data, out.ctypes.data) == 0
    return from_words(out)


def tdiv(a, b):
    q = abs(a) // abs(b)
    return q if (a < 0) == (b < 0) else -q


def samples(rng, n):
    for _ in range(n):
        bits_a = rng.choice([3, 40, 64, 65, 100, 127, 128, 129, 180, 250])
        bits_b = rng.choice([1, 3, 31, 63, 64, 65, 90, 127, 128, 200])
        a = rng.getrandbits(bits_a) * rng.choice([1, -1])
        b = rng.getrandbits(bits_b) * rng.choice([1, -1])
        yield a, b


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_i256_matches_python(seed):
    rng = random.Random(seed)
    for a, b in samples(rng, 300):
        assert op(0, a, b) == a + b
        assert op(1, a, b) == a - b
        if abs(a * b) < (1 << 254):
            assert op(2, a, b) == a * b
        if b != 0:
            assert op(3, a, b) == tdiv(a, b), (a, b)
            assert op(4, a, b) == a - b * tdiv(a, b), (a, b)
        assert op(5, a, b) == int(a < b)
        assert op(6, a, 0) == a >> 1
