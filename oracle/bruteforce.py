"""O8 — brute force on tiny inputs (TEST INFRASTRUCTURE ONLY).

In exact arithmetic QRCP's pivot rule is the greedy projection rule
i_{j+1} = argmax_{i not in I_j} ||(I - Pi_{A(:, I_j)}) a_i||_2 (Eq. (6)),
evaluated here in fp64 with an explicit least-squares projection per candidate.
`best_subset_error` enumerates all C(n, k) column subsets (the optimum any
column ID with |I| = k can reach).
"""
from __future__ import annotations

import itertools

import numpy as np


def greedy_pivots(A: np.ndarray, k: int) -> list:
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[1]
    I = []
    for _ in range(k):
        best, bestv = None, -1.0
        for i in range(n):
            if i in I:
                continue
            a = A[:, i]
            if I:
                B = A[:, I]
                x, *_ = np.linalg.lstsq(B, a, rcond=None)
                a = a - B @ x
            v = float(np.linalg.norm(a))
            if v > bestv:
                best, bestv = i, v
        I.append(best)
    return I


def best_subset_error(A: np.ndarray, k: int) -> float:
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[1]
    best = np.inf
    for I in itertools.combinations(range(n), k):
        B = A[:, list(I)]
        X, *_ = np.linalg.lstsq(B, A, rcond=None)
        best = min(best, float(np.linalg.norm(A - B @ X)))
    return best
