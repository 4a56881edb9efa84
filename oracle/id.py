"""O5-O8 — the fp64 ID step, its error and its bounds, written plainly.

TEST INFRASTRUCTURE ONLY (see oracle/rounding.py header).

PAPER.md passages:
  * Eq. (8), P:129-135 and Algorithm 1/2 lines 4-6:
    T = R11^+ R12, P(:, I) = [I_k T] Z^T, I = I(1:k).  Remark 1:
    pseudo-inverse because R11 may be ill-conditioned.
  * P "is computed from the R matrix and pivot indices ... via a
    least-squares problem" — `coeffs_lsq` is that least-squares problem solved
    in fp64 against A_D (reading R11, north_star's "least-squares fit of A_D
    against A_D(:,I)").
  * P:196 and Remark 2: the mixed ID is A_M = A_D(:, I_L) P_L and
    the product is evaluated in double.  `id_error` returns
    ||A_D - A_D(:, I) P||_F and its ratio to ||A_D||_F (reading R12: Frobenius,
    BASELINE.json's metric; the paper plots 2-norms).
  * Lemma 2.1: sqrt(1 + k(n-k)) and sqrt(1 + k(n-k)) sigma_{k+1}.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla


def coeffs_from_R(R: np.ndarray, perm: np.ndarray, k: int, pinv_tol: float | None = None) -> np.ndarray:
    """P = [I_k T] Z^T with T = R11^{-1} R12 in fp64 (Algorithm 2 lines 5-6).

    R (k x n, pivoted column order) is promoted to fp64.  With pinv_tol=None a
    triangular back-substitution is used (R11 upper triangular); with a
    tolerance, T = R11^+ R12 via an SVD pseudo-inverse truncating singular values
    below pinv_tol * sigma_max (Remark 1).  Column perm[j] of P is e_j (j < k);
    column perm[k + i] is T(:, i).
    """
    R = np.asarray(R, dtype=np.float64)[:k]
    n = R.shape[1]
    R11, R12 = R[:, :k], R[:, k:]
    if pinv_tol is None:
        T = sla.solve_triangular(R11, R12, lower=False) if n > k else np.zeros((k, 0))
    else:
        U, S, Vt = np.linalg.svd(R11)
        if S.size == 0 or S[0] == 0.0:
            raise ZeroDivisionError("sigma_max(R11) = 0 (DegenerateError, S:248)")
        Sinv = np.where(S > pinv_tol * S[0], 1.0 / np.where(S > 0, S, 1.0), 0.0)
        T = (Vt.T * Sinv) @ (U.T @ R12)
    P = np.zeros((k, n))
    P[:, perm[:k]] = np.eye(k)
    P[:, perm[k:]] = T
    return P


def coeffs_lsq(A_D: np.ndarray, I: np.ndarray) -> np.ndarray:
    """P(:, I) = I_k exactly; P(:, J) = argmin_X ||A_D(:, I) X - A_D(:, J)||_F.

    Solved by fp64 Householder QR of A_D(:, I) (LAPACK dgeqrf via numpy), then
    X = R^{-1} (Q^T A_D(:, J)).  Deliberately a different algorithm from the
    CUDA path's CholeskyQR2.
    """
    A_D = np.asarray(A_D, dtype=np.float64)
    I = np.asarray(I)
    n = A_D.shape[1]
    k = len(I)
    J = np.setdiff1d(np.arange(n), I, assume_unique=False)
    AI = A_D[:, I]
    Q, R = np.linalg.qr(AI, mode="reduced")
    X = sla.solve_triangular(R, Q.T @ A_D[:, J], lower=False)
    P = np.zeros((k, n))
    P[:, I] = np.eye(k)
    P[:, J] = X
    return P


def id_error(A_D: np.ndarray, I: np.ndarray, P: np.ndarray):
    """(||A_D - A_D(:, I) P||_F, same / ||A_D||_F), products in fp64 (Remark 2).

    Column sums of squares are accumulated with math.fsum (correctly rounded)
    so the value is independent of summation order.
    """
    A_D = np.asarray(A_D, dtype=np.float64)
    E = A_D - A_D[:, np.asarray(I)] @ P
    abs2 = math.fsum(math.fsum(col) for col in (E * E).T)
    nrm2 = math.fsum(math.fsum(col) for col in (A_D * A_D).T)
    return math.sqrt(abs2), math.sqrt(abs2) / math.sqrt(nrm2) if nrm2 > 0 else float("nan")


def id_error_blocked(A_D: np.ndarray, I: np.ndarray, P: np.ndarray, cols: int = 64):
    """id_error for large matrices: the same definition (Remark 2: residual formed
    and squared in fp64), evaluated 64 columns at a time; each column's sum of
    squares is numpy's fp64 pairwise sum and the column sums are added with
    math.fsum.  Pinned against id_error (tests/test_oracle_id.py)."""
    A_D = np.asarray(A_D)
    I = np.asarray(I)
    AI = np.ascontiguousarray(A_D[:, I])
    n = A_D.shape[1]
    parts, nrm = [], []
    for c0 in range(0, n, cols):
        c1 = min(n, c0 + cols)
        blk = np.asarray(A_D[:, c0:c1], dtype=np.float64)
        E = blk - AI @ P[:, c0:c1]
        parts.extend(np.einsum("ij,ij->j", E, E).tolist())
        nrm.extend(np.einsum("ij,ij->j", blk, blk).tolist())
    abs2, nrm2 = math.fsum(parts), math.fsum(nrm)
    return math.sqrt(abs2), math.sqrt(abs2) / math.sqrt(nrm2) if nrm2 > 0 else float("nan")


def low_skeleton(A_D: np.ndarray, I: np.ndarray, fmt: str, s: float) -> np.ndarray:
    """A_L(:, I) in A_D's units: fl_L(s A_D(:, I)) / s (the low-precision ID's
    skeleton; Algorithm 2 line 8 with A_L instead of A_D)."""
    from .rounding import round_to
    AI = np.asarray(A_D, dtype=np.float64)[:, np.asarray(I)]
    return round_to(AI * s, fmt).reshape(AI.shape) / s


def id_error_skeleton(A_D: np.ndarray, X: np.ndarray, P: np.ndarray):
    """(||A_D - X P||_F, same / ||A_D||_F) for an arbitrary skeleton X (m x k), fp64,
    column sums of squares added with math.fsum (the Â_L variant of P:196)."""
    A_D = np.asarray(A_D, dtype=np.float64)
    E = A_D - X @ P
    abs2 = math.fsum(math.fsum(col) for col in (E * E).T)
    nrm2 = math.fsum(math.fsum(col) for col in (A_D * A_D).T)
    return math.sqrt(abs2), math.sqrt(abs2) / math.sqrt(nrm2) if nrm2 > 0 else float("nan")


def spectral_error(A_D: np.ndarray, X: np.ndarray, P: np.ndarray):
    """(||A_D - X P||_2, same / ||A_D||_2) by LAPACK SVD — the paper's metric."""
    A_D = np.asarray(A_D, dtype=np.float64)
    e = float(np.linalg.norm(A_D - X @ P, 2))
    a = float(np.linalg.norm(A_D, 2))
    return e, e / a if a > 0 else float("nan")


def lemma_bound(k: int, n: int, sigma_k1: float):
    """Lemma 2.1: (sqrt(1 + k(n-k)), sqrt(1 + k(n-k)) sigma_{k+1})."""
    c = math.sqrt(1.0 + k * (n - k))
    return c, c * sigma_k1


def eckart_young_fro(sigma: np.ndarray, k: int) -> float:
    """Lower bound on any rank-k approximation error in Frobenius norm: sqrt(sum_{j>k} sigma_j^2)."""
    s = np.asarray(sigma, dtype=np.float64)
    return math.sqrt(float(np.sum(s[k:] ** 2)))


def post_bound(resid_k: float, s: float, T_norm2: float, normAD_F: float, u_L: float,
               k: int, nb: int, m: int, u_acc: float) -> float:
    """B_post (reading R13): a-posteriori Frobenius bound on the mixed-ID error.

    err_F <= rho_k + (1 + ||T||_2) (u_L + eta_QR) ||A_D||_F, with rho_k = the
    QR's remaining column-norm mass / s (undoing range scaling) and
    eta_QR = (ceil(k/nb) + 2 sqrt(k)) u_L + 4 k gamma_d(u_acc), d = 8 + ceil(log2(m)).
    """
    from .rounding import gamma
    d = 8 + math.ceil(math.log2(max(m, 2)))
    eta = (math.ceil(k / max(nb, 1)) + 2.0 * math.sqrt(k)) * u_L + 4 * k * gamma(d, u_acc)
    return resid_k / s + (1.0 + T_norm2) * (u_L + eta) * normAD_F
