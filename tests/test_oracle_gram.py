"""Pins for oracle/gram.py (O9, NEXT-4): Gram-based pivoting by pivoted Cholesky.

Pins (none retypes the oracle's own loop):
  * brute-force greedy projection pivots (oracle/bruteforce.py, Eq. (6)) on tiny inputs;
  * LAPACK dgeqp3 (scipy) pivots and |diag R| in fp64 on well-separated inputs;
  * the fp64 Householder QRCP oracle: same pivots, same R (R_jj >= 0) to 1e-9;
  * closed form: orthogonal columns -> pivots sorted by norm, R = diag(norms);
  * the Cholesky identity R11^T R11 = G(I, I), R11^T R12 = G(I, J) (LAPACK-free check by
    explicit products);
  * exact-rank input -> breakdown (status underflow) at the rank; tolerance stop at the
    Eckart-Young-style crossing of the exact residual.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle.bruteforce import greedy_pivots
from oracle.gram import certified_gram_steps, gram, pivoted_cholesky
from oracle.qrcp import qrcp_householder


def _sep(m, n, seed, decay=8.0):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    return U @ np.diag(np.exp(-np.arange(n) / decay)) @ V.T


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_greedy_bruteforce(seed):
    A = _sep(12, 8, seed, decay=2.0)
    r = pivoted_cholesky(gram(A), 6)
    assert list(r.perm[:6]) == greedy_pivots(A, 6)


def test_lapack_dgeqp3_and_householder_oracle():
    A = _sep(300, 80, 5, decay=12.0)
    k = 60
    r = pivoted_cholesky(gram(A), k)
    _, Rl, pl = sla.qr(A, mode="economic", pivoting=True)
    q = qrcp_householder(A, k, "fp64", acc="fp64")
    cert = certified_gram_steps(r, gamma=1e-14)
    first = int(np.argmin(cert)) if not cert.all() else k
    assert first > 40
    assert np.array_equal(r.perm[:first], pl[:first])
    assert np.array_equal(r.perm[:first], q.perm[:first])
    d = np.abs(np.diag(Rl))[:first]
    assert np.max(np.abs(np.diag(r.R)[:first] - d) / d) < 1e-9
    # R rows equal the Householder R (both sign-normalised, R_jj >= 0) on the agreed prefix
    assert np.max(np.abs(r.R[:first, :first] - q.R[:first, :first])) < 1e-9 * np.abs(q.R[0, 0])


def test_orthogonal_columns_closed_form():
    rng = np.random.default_rng(7)
    Q = np.linalg.qr(rng.standard_normal((40, 10)))[0]
    norms = np.array([3.0, 7.0, 1.0, 5.0, 2.0, 9.0, 4.0, 6.0, 8.0, 0.5])
    A = Q * norms
    r = pivoted_cholesky(gram(A), 10)
    assert list(r.perm) == list(np.argsort(-norms))
    assert np.allclose(r.R, np.diag(np.sort(norms)[::-1]), atol=1e-12)


def test_cholesky_identity():
    A = _sep(100, 30, 11, decay=5.0)
    k = 12
    G = gram(A)
    r = pivoted_cholesky(G, k)
    I, J = r.perm[:k], r.perm[k:]
    R11, R12 = r.R[:, :k], r.R[:, k:]
    assert np.allclose(R11.T @ R11, G[np.ix_(I, I)], rtol=0, atol=1e-12 * G.max())
    assert np.allclose(R11.T @ R12, G[np.ix_(I, J)], rtol=0, atol=1e-12 * G.max())
    assert np.all(np.diff(np.diag(R11)) <= 1e-12)            # |R_jj| non-increasing (greedy)


def test_exact_rank_breakdown_and_tolerance():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((50, 5)) @ rng.standard_normal((5, 20))
    r = pivoted_cholesky(gram(A), 10)
    assert r.status == "underflow" or r.k_out == 10
    if r.status == "underflow":
        assert r.k_out >= 5
    # tolerance: k_eps is the first j whose exact residual mass is <= eps ||A||_F
    A = _sep(200, 40, 3, decay=4.0)
    G = gram(A)
    eps = 1e-2
    r = pivoted_cholesky(G, 40, eps=eps)
    k = r.k_out
    I = r.perm[:k]
    X, *_ = np.linalg.lstsq(A[:, I], A, rcond=None)
    res = np.linalg.norm(A - A[:, I] @ X)
    assert res <= eps * np.linalg.norm(A) * (1 + 1e-9)
    Ip = r.perm[:k - 1]
    Xp, *_ = np.linalg.lstsq(A[:, Ip], A, rcond=None)
    assert np.linalg.norm(A - A[:, Ip] @ Xp) > eps * np.linalg.norm(A)


def test_ties_lowest_original_index():
    G = np.eye(6) * 2.0
    r = pivoted_cholesky(G, 6)
    assert list(r.perm) == list(range(6))
