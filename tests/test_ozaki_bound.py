"""CPU pin of the arithmetic the int8 fp64 engine relies on (DESIGN.md §5 "fp64 on the
integer tensor cores"; include/mpid.h id_set_fp64_engine).  Test infrastructure only: it
restates the scheme in exact Python integers and checks its claims; it shares nothing with
the CUDA path.

Claims checked on random and adversarial inputs:
  1. digit split: x = sgn(x) sum_{p<8} s_p 2^{-7(p+1)} 2^E + e with s_p in [0, 127] and
     |e| < 2^{E-56}, for E the smallest exponent with max|x| < 2^E;
  2. the kept products (p + q <= 7) of a length-K dot product differ from the exact dot
     product of the fp64 inputs by at most (8 + 1) 2^{-56} 2^{Ea+Eb} K;
  3. the int32 accumulators never overflow: |sum over K of the pairs on one diagonal|
     <= 8 * 127^2 * K < 2^31 for K <= 16384 (the TN kernel's drain interval);
  4. the int32 -> fp64 conversion trick (1.5 2^52 + 2^31 + a, minus the constant) is exact
     over the whole int32 range.
"""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

S = 8


def exp_of(mx: float) -> int:
    """Smallest E with mx < 2^E (0 for mx == 0)."""
    if mx == 0.0:
        return 0
    m, e = math.frexp(mx)      # mx = m 2^e, m in [0.5, 1)
    return e


def digits(x: float, E: int):
    X = int(Fraction(abs(x)) * Fraction(2) ** (56 - E))   # truncation toward zero
    assert 0 <= X < 2 ** 56
    d = [(X >> (49 - 7 * p)) & 127 for p in range(S)]
    sg = -1 if x < 0 else 1
    return [sg * v for v in d]


def value(ds, E):
    return sum(Fraction(v) * Fraction(2) ** (-7 * (p + 1)) for p, v in enumerate(ds)) * Fraction(2) ** E


@pytest.mark.parametrize("seed", range(4))
def test_digit_split_error_bound(seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(64) * 10.0 ** rng.uniform(-12, 12, size=64)
    x[3] = 0.0
    x[5] = -np.max(np.abs(x))          # the row max itself, negative
    E = exp_of(float(np.max(np.abs(x))))
    for v in x:
        ds = digits(float(v), E)
        assert all(-127 <= d <= 127 for d in ds)
        assert all(d == 0 or (d > 0) == (v > 0) for d in ds)
        err = abs(Fraction(float(v)) - value(ds, E))
        assert err < Fraction(2) ** (E - 56)


@pytest.mark.parametrize("seed,K", [(0, 7), (1, 100), (2, 128), (3, 33)])
def test_truncated_product_bound(seed, K):
    rng = np.random.default_rng(100 + seed)
    a = rng.standard_normal(K) * 10.0 ** rng.uniform(-3, 3, size=K)
    b = rng.standard_normal(K) * 10.0 ** rng.uniform(-3, 3, size=K)
    Ea, Eb = exp_of(float(np.max(np.abs(a)))), exp_of(float(np.max(np.abs(b))))
    da = [digits(float(v), Ea) for v in a]
    db = [digits(float(v), Eb) for v in b]
    acc = [0] * S                                     # the 8 diagonal accumulators
    for i in range(K):
        for p in range(S):
            for q in range(S - p):
                acc[p + q] += da[i][p] * db[i][q]
    approx = sum(Fraction(acc[d]) * Fraction(2) ** (-7 * d) for d in range(S)) * Fraction(2) ** (Ea + Eb - 14)
    exact = sum(Fraction(float(a[i])) * Fraction(float(b[i])) for i in range(K))
    bound = Fraction(S + 1) * Fraction(2) ** (-56) * Fraction(2) ** (Ea + Eb) * K
    assert abs(approx - exact) <= bound
    # and the relative accuracy is at the fp64 level for this (non-cancelling) data
    scale = sum(abs(Fraction(float(a[i])) * Fraction(float(b[i]))) for i in range(K))
    assert float(abs(approx - exact) / scale) < 1e-13


def test_int32_accumulators_cannot_overflow():
    # worst case: every digit 127 with equal signs, the most populated diagonal (8 pairs)
    for K in (32, 128, 16384):
        worst = 8 * 127 * 127 * K
        assert worst < 2 ** 31, K
    assert 8 * 127 * 127 * 16385 * 2 > 2 ** 31   # the drain interval is not oversized by 2x


def test_int32_to_fp64_magic_conversion_is_exact():
    base = struct.unpack("<d", struct.pack("<Q", 0x4338000000000000))[0]   # 1.5 2^52
    const = base + 2 ** 31
    for a in [0, 1, -1, 2 ** 31 - 1, -2 ** 31, 123456789, -987654321]:
        lo = (a ^ 0x80000000) & 0xFFFFFFFF if a >= 0 else ((a + 2 ** 32) ^ 0x80000000) & 0xFFFFFFFF
        bits = (0x43380000 << 32) | lo
        d = struct.unpack("<d", struct.pack("<Q", bits))[0]
        assert d - const == a
    assert const == 6755401588539392.0       # the constant in k_ozaki.cu's i2d


def test_digit_word_from_the_bit_pattern():
    """Claim 5 (k_ozaki.cu oz_digits): X = floor(|x| 2^(56-E)) equals the 53-bit significand M
    of x shifted right by 2098 - es - e, with e the biased exponent of x (1 and no hidden bit
    for subnormals) and es the biased exponent of the scale 2^(56-E); the shift is never below
    -3 because |x| < 2^E.  Exact integers against the Fraction definition above."""
    rng = np.random.default_rng(7)
    for trial in range(60):
        x = rng.standard_normal(300) * 10.0 ** int(rng.integers(-280, 280))
        x[rng.integers(0, 300, 10)] = 0.0
        x[rng.integers(0, 300, 5)] *= 2.0 ** -45
        if trial % 6 == 0:
            x = x * 2.0 ** -1000 * 2.0 ** -50            # subnormals
        if trial % 6 == 1:
            x[0] = math.ldexp(1.0 - 2.0 ** -53, 10)      # just below a power of two
        E = exp_of(float(np.abs(x).max()))
        if not (-1022 <= 56 - E <= 1023):
            continue
        es = (struct.unpack("<Q", struct.pack("<d", math.ldexp(1.0, 56 - E)))[0] >> 52) & 0x7FF
        for v in x:
            bits = struct.unpack("<Q", struct.pack("<d", float(v)))[0]
            e = (bits >> 52) & 0x7FF
            M = (bits & ((1 << 52) - 1)) | ((1 << 52) if e else 0)
            sh = 2098 - es - (e if e else 1)
            assert sh >= -3
            X = 0 if sh >= 64 else (M >> sh if sh >= 0 else M << -sh)
            assert X == int(Fraction(abs(float(v))) * Fraction(2) ** (56 - E))
            assert X < 2 ** 56
