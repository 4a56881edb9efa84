"""O1/O2 — the floating-point model of the paper, written out bit by bit.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import anything under oracle/.  The
product path (paper_2012_00706_b200/) never imports it and the oracle never
imports the product.

Paper passages followed (PAPER.md, "P:L" = line L):
  * Eq. (1): y = +-m * b^(e-t), 0 <= m <= b^t - 1, e_min <= e <= e_max.
  * Table 1: exponent/mantissa bits 5/10, 8/23, 11/52 for
    half/single/double; u printed as 4.9e-4, 6.0e-8, 1.1e-16.
  * fl(.) and Eq. (2): fl maps a real to its closest representable
    number; u = 1/2 b^(1-t).  Ties are not specified by the paper: we use the
    IEEE-754 default round-to-nearest-even (reading R1).
  * Definition 1: gamma_k.  The printed form k*u/(1-u) is kept only as
    `gamma_printed`; bounds use Higham's Lemma 3.1 form k*u/(1-k*u), which the
    paper cites and whose precondition k*u < 1 it states (reading R2).

`round_to` is a pure integer implementation of round-to-nearest-even from an
IEEE binary64 value to binary16/binary32 (subnormals kept, overflow -> +-Inf,
NaN -> NaN).  It does not call any library float conversion, so the tests can
compare it against numpy's and x86's conversions as an independent pin.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class FloatFormat:
    """Eq. (1): precision t counts the implicit bit (t = mantissa_bits + 1)."""
    name: str
    exponent_bits: int
    mantissa_bits: int

    @property
    def t(self) -> int:
        return self.mantissa_bits + 1

    @property
    def emax(self) -> int:
        return 2 ** (self.exponent_bits - 1) - 1

    @property
    def emin(self) -> int:
        return 1 - self.emax

    @property
    def u(self) -> float:
        """Unit round-off u = 1/2 * 2^(1-t)."""
        return math.ldexp(1.0, -self.t)

    @property
    def max_finite(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, 1 - self.t), self.emax)

    @property
    def min_normal(self) -> float:
        return math.ldexp(1.0, self.emin)

    @property
    def min_subnormal(self) -> float:
        return math.ldexp(1.0, self.emin - self.t + 1)


# Table 1
HALF = FloatFormat("half", 5, 10)
SINGLE = FloatFormat("single", 8, 23)
DOUBLE = FloatFormat("double", 11, 52)
FORMATS = {"fp16": HALF, "half": HALF, "fp32": SINGLE, "single": SINGLE,
           "fp64": DOUBLE, "double": DOUBLE}


def fmt_of(name) -> FloatFormat:
    return name if isinstance(name, FloatFormat) else FORMATS[name]


def round_to(x, fmt) -> np.ndarray:
    """fl_fmt(x) for binary64 input x (array or scalar), returned as float64.

    Bit-level RNE: x = mant * 2^e2 with mant the 53-bit significand; the target
    quantum is 2^q with q = max(floor(log2|x|), e_min) - (t - 1); the integer
    mant is shifted right by (q - e2) with round-half-to-even on the dropped
    bits; results above the format's max finite value become +-Inf (P:27-31,
    Table 1).  Doubles that are themselves subnormal lie far below 2^-149 and
    round to +-0 in both low formats.
    """
    f = fmt_of(fmt)
    a = np.asarray(x, dtype=np.float64)
    scalar = a.ndim == 0
    a = np.atleast_1d(a)
    if f is DOUBLE:
        out = a.copy()
        return out[0] if scalar else out
    bits = a.view(np.uint64)
    sign = bits >> np.uint64(63)
    E = ((bits >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64)
    frac = bits & np.uint64((1 << 52) - 1)
    out = np.zeros_like(a)
    special = E == 0x7FF                      # Inf / NaN pass through
    out[special] = a[special]
    normal = (E > 0) & ~special               # binary64 subnormals -> 0
    if np.any(normal):
        En = E[normal]
        mant = frac[normal] | np.uint64(1 << 52)          # 53-bit integer
        e2 = En - 1075                                    # value = mant * 2^e2
        q = np.maximum(En - 1023, f.emin) - (f.t - 1)     # target quantum exponent
        shift = q - e2                                    # >= 29 for binary32
        big = shift >= 55                                  # all bits below half-quantum
        sh = np.where(big, 0, shift).astype(np.uint64)
        r = mant >> sh
        rem = mant & ((np.uint64(1) << sh) - np.uint64(1))
        half = np.uint64(1) << (sh - np.uint64(1))
        up = (rem > half) | ((rem == half) & ((r & np.uint64(1)) == np.uint64(1)))
        r = r + up.astype(np.uint64)
        r = np.where(big, np.uint64(0), r)
        mag = np.ldexp(r.astype(np.float64), q)           # r <= 2^t: exact
        mag = np.where(mag > f.max_finite, np.inf, mag)
        out[normal] = mag
    out = np.where(sign.astype(bool), -np.abs(out), np.abs(out))
    out[special] = a[special]
    return out[0] if scalar else out


def unit_roundoff(fmt) -> float:
    return fmt_of(fmt).u


def gamma(k: int, u: float) -> float:
    """Higham's gamma_k = k u / (1 - k u) (Lemma 3.1 of the book cited at P:34).

    Raises ValueError (SPEC's DomainError) when k u >= 1, the precondition of
    Definition 1.
    """
    if k * u >= 1.0:
        raise ValueError(f"gamma_k undefined: k*u = {k * u} >= 1 (Definition 1, P:34)")
    return k * u / (1.0 - k * u)


def gamma_printed(k: int, u: float) -> float:
    """The form printed in Definition 1, k u / (1 - u); kept to reproduce SPEC S:65."""
    if k * u >= 1.0:
        raise ValueError("k*u >= 1 (Definition 1, P:34)")
    return k * u / (1.0 - u)
