"""O9 — Gram-based pivoting (the paper's future work "matrix
sketching"): the QRCP pivots and R obtained from G = A_L^T A_L by a pivoted
Cholesky factorisation instead of k streaming Householder passes.

TEST INFRASTRUCTURE ONLY (see oracle/rounding.py header).

Definition followed (plain, fp64):
  * G = A_L^T A_L.  A_L holds fp16/fp32 values, whose pairwise products are exact in
    fp64; the sums are numpy/BLAS fp64 sums (the only rounding).
  * Outer-product pivoted Cholesky, step j = 0, 1, ...:
        d_i = G_ii - sum_{l<j} R(l, i)^2                 (residual column norms^2)
        p   = argmax_{i >= j} d_i  (ties: lowest original column index, as S:216)
        swap positions j <-> p (perm, d, R(:j, :))
        R(j, j) = sqrt(d_j);  R(j, i) = (G(perm_j, perm_i) - sum_{l<j} R(l, j) R(l, i)) / R(j, j)
    In exact arithmetic d_i is ||(I - Pi_{A(:, I_j)}) a_i||^2, so p is Eq. (6)'s greedy
    pivot and R is the R factor of the pivoted Householder QR with
    R_jj >= 0: pinned against oracle.qrcp (fp64) and oracle.bruteforce.
  * Tolerance (reading R8 on the same quantity): stop before step j >= 1 when
    sum_{i >= j} d_i <= eps^2 ||A_L||_F^2.  Breakdown: d_p <= 0 -> status "underflow"
    (the Gram's resolution is exhausted; k = j).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class GramResult:
    perm: np.ndarray       # (n,) original column index at each position
    R: np.ndarray          # (k_out, n) fp64, columns in pivoted order
    k_out: int
    status: str            # "ok" | "underflow"
    top2: np.ndarray       # (k_out, 2): the two largest d_i (norms^2) at each step
    d0max: float           # max_i G_ii

    @property
    def I(self) -> np.ndarray:
        return self.perm[: self.k_out]


def gram(A_L: np.ndarray) -> np.ndarray:
    """G = A_L^T A_L in fp64."""
    A = np.asarray(A_L, dtype=np.float64)
    return A.T @ A


def pivoted_cholesky(G: np.ndarray, k_max: int, eps: float = 0.0) -> GramResult:
    G = np.asarray(G, dtype=np.float64)
    n = G.shape[0]
    if not (1 <= k_max <= n):
        raise ValueError("k out of range")
    perm = np.arange(n)
    d = np.diag(G).copy()
    R = np.zeros((k_max, n))
    top2 = np.zeros((k_max, 2))
    trace = float(np.sum(d))
    status, k_out = "ok", k_max
    for j in range(k_max):
        if eps > 0.0 and j > 0 and float(np.sum(d[j:])) <= eps * eps * trace:
            k_out = j
            break
        cand = d[j:]
        c_ = np.flatnonzero(cand == cand.max())
        p = j + int(c_[np.argmin(perm[j + c_])])
        srt = np.sort(cand)[::-1]
        top2[j] = [srt[0], srt[1] if len(srt) > 1 else -np.inf]
        if p != j:
            perm[[j, p]] = perm[[p, j]]
            d[[j, p]] = d[[p, j]]
            R[:j, [j, p]] = R[:j, [p, j]]
        if not d[j] > 0.0:
            status, k_out = "underflow", j
            break
        rjj = math.sqrt(d[j])
        R[j, j] = rjj
        rest = perm[j + 1:]
        R[j, j + 1:] = (G[perm[j], rest] - R[:j, j] @ R[:j, j + 1:]) / rjj
        d[j + 1:] -= R[j, j + 1:] ** 2
        d[j] = 0.0
    return GramResult(perm, R[:k_out], k_out, status, top2[:k_out], float(np.max(np.diag(G))))


def certified_gram_steps(res: GramResult, gamma: float, c_tie: float = 4.0) -> np.ndarray:
    """Steps whose pivot is decided beyond a perturbation of G bounded entrywise by
    gamma * sqrt(G_ii G_jj): the top-2 gap of d exceeds c_tie * gamma * max_i G_ii
    (every d_i moves by at most ~gamma * max G_ii per unit of conditioning; reading R17)."""
    gap = res.top2[:, 0] - res.top2[:, 1]
    return gap > c_tie * gamma * res.d0max
