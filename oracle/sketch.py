"""O10 — sketched pivoting (second option: "a randomized sketch";
the paper's future work "matrix sketching").

TEST INFRASTRUCTURE ONLY (see oracle/rounding.py header).

Definition followed (plain, fp64):
  * Omega (l x m) with iid Rademacher entries +-1 (synth.counter_sign, the counter-based
    generator both sides implement; the random numbers are inputs, not arithmetic);
  * Y = Omega A_L  (l x n), products exact (+-1 times fp16/fp32 values), fp64 sums;
  * the pivots and R are those of the fp64 Householder QRCP of Y with exact residual
    norms recomputed every step (oracle.qrcp.qrcp_householder, fmt "fp64", acc "fp64",
    norms "recompute") — the randomized ID's column selection: with l >= rank(A) + a
    few, Y has A's column dependencies with probability 1, so an exact-rank A is
    reproduced exactly by the selected skeleton (pinned in tests/test_oracle_sketch.py).
"""
from __future__ import annotations

import numpy as np

from .qrcp import qrcp_householder


def sketch(A_L: np.ndarray, Omega: np.ndarray) -> np.ndarray:
    """Y = Omega A_L in fp64."""
    return np.asarray(Omega, dtype=np.float64) @ np.asarray(A_L, dtype=np.float64)


def sketched_qrcp(Y: np.ndarray, k_max: int, eps: float = 0.0):
    """QRCP of the sketch (fp64, exact norms each step)."""
    return qrcp_householder(np.asarray(Y, dtype=np.float64), k_max, "fp64", acc="fp64", norms="recompute",
                            eps=eps)
