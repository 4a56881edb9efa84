"""Pins for oracle/rounding.py (O1, O2): fl(.), u, gamma_k.

Every expected value comes from SPEC/PAPER worked examples (tests/golden), from
the IEEE encoding (exhaustive binary16 midpoints), or from independent
conversions (numpy's float16 cast, x86 cvtsd2ss via numpy's float32 cast).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle.rounding import (HALF, SINGLE, DOUBLE, gamma, gamma_printed, round_to)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _val(y):
    return math.inf if y == "inf" else float(y)


@pytest.mark.parametrize("case", GOLD["rounding_fp16"], ids=lambda c: c["cite"])
def test_spec_rounding_examples(case):
    assert round_to(case["x"], "fp16") == _val(case["y"])


def test_overflow_examples():
    for c in GOLD["overflow_fp16"]:
        assert math.isinf(round_to(c["x"], "fp16"))
    assert round_to(65519.99, "fp16") == 65504.0
    assert math.isinf(round_to(65520.0, "fp16"))           # exact tie above max -> even -> inf
    assert round_to(-1e6, "fp16") == -math.inf


def test_store_half_tiny_and_near_ties():
    g = GOLD["store_half_tiny"]
    assert round_to(g["x"], "fp16") == g["y"]                               # S:75 / A28
    assert round_to(2.0 ** -25 * (1 + 2.0 ** -30), "fp16") == 2.0 ** -24
    # single rounding from fp64 (A32): 1 + 2^-11 + 2^-40 -> 1 + 2^-10 directly
    assert round_to(1 + 2.0 ** -11 + 2.0 ** -40, "fp16") == 1 + 2.0 ** -10
    assert round_to(1 + 2.0 ** -11, "fp16") == 1.0                           # tie -> even


def test_single_add_example():
    g = GOLD["single_add"]
    s = np.float32(g["a"]) + np.float32(g["b"])
    assert float(s) == g["y"]
    assert round_to(g["a"] + g["b"], "fp32") == g["y"]


def _all_fp16_finite_positive():
    bits = np.arange(0, 0x7C00, dtype=np.uint16)        # +0 .. max finite
    return bits.view(np.float16).astype(np.float64)


def test_exhaustive_fp16_midpoints():
    """Every gap between consecutive binary16 values: midpoint -> even, +-1 fp64 ulp -> neighbour."""
    h = _all_fp16_finite_positive()
    lo, hi = h[:-1], h[1:]
    mid = (lo + hi) / 2                                  # exact in fp64
    lo_bits = np.arange(0, 0x7C00 - 1)
    even = np.where(lo_bits % 2 == 0, lo, hi)
    assert np.array_equal(round_to(mid, "fp16"), even)
    assert np.array_equal(round_to(np.nextafter(mid, np.inf), "fp16"), hi)
    assert np.array_equal(round_to(np.nextafter(mid, -np.inf), "fp16"), lo)
    assert np.array_equal(round_to(-mid, "fp16"), -even)
    assert np.array_equal(round_to(h, "fp16"), h)        # representable values are fixed points


def test_fp16_vs_numpy_cast_random():
    rng = np.random.default_rng(7)
    x = rng.standard_normal(400_000) * np.exp2(rng.uniform(-30, 18, 400_000))
    ref = x.astype(np.float16).astype(np.float64)
    assert np.array_equal(round_to(x, "fp16"), ref)


def test_fp32_vs_hardware_cast_random():
    rng = np.random.default_rng(8)
    x = rng.standard_normal(400_000) * np.exp2(rng.uniform(-160, 130, 400_000))
    with np.errstate(over="ignore"):
        ref = x.astype(np.float32).astype(np.float64)
    assert np.array_equal(round_to(x, "fp32"), ref)


def test_fp32_midpoints_sample():
    rng = np.random.default_rng(9)
    b = rng.integers(0, 0x7F7FFFFF, 200_000, dtype=np.int64).astype(np.uint32)
    lo = b.view(np.float32).astype(np.float64)
    hi = (b + 1).view(np.float32).astype(np.float64)
    mid = (lo + hi) / 2
    even = np.where(b % 2 == 0, lo, hi)
    assert np.array_equal(round_to(mid, "fp32"), even)
    assert np.array_equal(round_to(np.nextafter(mid, np.inf), "fp32"), hi)


def test_properties():
    rng = np.random.default_rng(10)
    x = np.sort(rng.standard_normal(100_000) * np.exp2(rng.uniform(-26, 15, 100_000)))
    for f in ("fp16", "fp32"):
        r = round_to(x, f)
        assert np.array_equal(round_to(r, f), r)                     # idempotent
        assert np.all(r[1:] >= r[:-1])                                # monotone
        assert np.array_equal(round_to(-x, f), -r)                    # sign symmetric
        fmt = HALF if f == "fp16" else SINGLE
        nrm = (np.abs(x) >= fmt.min_normal) & (np.abs(x) <= fmt.max_finite)
        assert np.all(np.abs(r[nrm] - x[nrm]) <= fmt.u * np.abs(x[nrm]))   # Eq. (2)
    assert np.isnan(round_to(np.nan, "fp16"))
    assert round_to(np.inf, "fp16") == np.inf
    assert round_to(5e-324, "fp16") == 0.0


def test_unit_roundoff_table1():
    t = GOLD["unit_roundoff_table1"]
    assert HALF.u == 2.0 ** -11 and SINGLE.u == 2.0 ** -24 and DOUBLE.u == 2.0 ** -53
    for f, key in ((HALF, "half"), (SINGLE, "single"), (DOUBLE, "double")):
        assert abs(f.u - t[key]) <= t["rel_tol"] * t[key]
    assert (HALF.exponent_bits, HALF.mantissa_bits) == (5, 10)
    assert (SINGLE.exponent_bits, SINGLE.mantissa_bits) == (8, 23)
    assert HALF.max_finite == 65504.0 and HALF.min_subnormal == 2.0 ** -24


def test_gamma():
    g = GOLD["gamma_printed"]
    assert abs(gamma_printed(g["k"], g["u"]) - g["y"]) <= g["rel_tol"] * g["y"]
    assert gamma_printed(2, 6e-8) == 2 * 6e-8 / (1 - 6e-8)
    assert gamma(2, 6e-8) == 2 * 6e-8 / (1 - 2 * 6e-8)
    with pytest.raises(ValueError):
        gamma(10, 0.1)
    # Lemma 3.1: prod (1+delta_i)^rho_i - 1 <= gamma_k; the worst case (1+u)^k - 1 is
    # bounded by Higham's form but NOT by the printed form at large k*u (reading R2).
    u, k = 2.0 ** -11, 1024
    worst = (1 + u) ** k - 1
    assert worst <= gamma(k, u)
    assert worst > gamma_printed(k, u)
