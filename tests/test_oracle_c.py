"""Pins for oracle/cqrcp.c (oracle/fast.py): the C restatement of the oracle's QRCP.

It must give the numpy oracle's (oracle/qrcp.py, formation "fma") result BIT FOR BIT —
permutation, R, residual masses, norms — for every format, both arithmetic models,
several store intervals, tolerance stops, ragged row counts, ties and underflow; and
it must not depend on the number of threads.  The numpy oracle is itself pinned by
tests/test_oracle_qrcp.py (LAPACK dgeqp3, MGS, brute force, planted skeletons, hand
examples); the fp64 C run is also checked against LAPACK dgeqp3 directly.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle.fast import qrcp_c
from oracle.qrcp import certified_steps, make_AL, qrcp_householder
from oracle.rounding import round_to
from synth import gen_config, gen_exact_rank, gen_planted


def same(a, b):
    assert a.k_out == b.k_out and a.status == b.status
    assert np.array_equal(a.perm, b.perm)
    assert np.array_equal(a.R, b.R)
    assert a.resid == b.resid
    assert a.normAL == b.normAL and a.maxnorm0 == b.maxnorm0
    assert np.array_equal(a.top2, b.top2)


@pytest.mark.parametrize("fmt,sc", [("fp16", "pow2"), ("fp32", "none"), ("fp64", "none")])
@pytest.mark.parametrize("model", ["paper", "kernel"])
@pytest.mark.parametrize("nb", [1, 4, 32])
def test_C1_bit_identical(fmt, sc, model, nb):
    AL, _ = make_AL(gen_config("C1", 2), fmt, sc)
    same(qrcp_householder(AL, 32, fmt, nb=nb, model=model), qrcp_c(AL, 32, fmt, nb=nb, model=model))


@pytest.mark.parametrize("fmt,sc,eps", [("fp16", "maxabs", 0.0), ("fp32", "none", 1e-3), ("fp16", "pow2", 1e-2)])
def test_C2_slice_bit_identical(fmt, sc, eps):
    A = np.asfortranarray(gen_config("C2", 1)[:, :256])
    AL, _ = make_AL(A, fmt, sc)
    for model in ("paper", "kernel"):
        same(qrcp_householder(AL, 64, fmt, nb=4, eps=eps, model=model),
             qrcp_c(AL, 64, fmt, nb=4, eps=eps, model=model))


def test_ragged_rows_planted_exact_rank_ties_underflow():
    A, skel, _ = gen_planted(250, 90, 20, rho=1.1, eta=1e-9, seed=3)      # m % 8 != 0
    for fmt, sc in (("fp16", "pow2"), ("fp32", "none")):
        AL, _ = make_AL(A, fmt, sc)
        r = qrcp_c(AL, 20, fmt, nb=8)
        same(qrcp_householder(AL, 20, fmt, nb=8, model="paper"), r)
        assert np.array_equal(r.perm[:20], skel)
    X = gen_exact_rank(203, 40, 7, seed=1)
    same(qrcp_householder(X, 30, "fp64", eps=1e-10, model="paper"), qrcp_c(X, 30, "fp64", eps=1e-10))
    assert qrcp_c(X, 30, "fp64", eps=1e-10).k_out == 7
    E = np.eye(9)                                                          # exact ties
    assert list(qrcp_c(E, 4, "fp64").perm[:4]) == [0, 1, 2, 3]
    Z = round_to(np.full((12, 3), 1e-20), "fp16").reshape(12, 3)          # underflow
    r = qrcp_c(Z, 1, "fp16")
    assert r.status == "underflow" and r.k_out == 0


def test_thread_count_independent():
    AL, _ = make_AL(gen_config("C2", 0)[:, :300], "fp16", "maxabs")
    same(qrcp_c(AL, 48, "fp16", nb=4, threads=1), qrcp_c(AL, 48, "fp16", nb=4, threads=7))


def test_fp64_against_lapack_dgeqp3():
    rng = np.random.default_rng(11)
    A = rng.standard_normal((300, 70)) @ np.diag(np.exp(-np.arange(70) / 12.0)) @ sla.qr(rng.standard_normal((70, 70)))[0]
    r = qrcp_c(A, 70, "fp64")
    Q, R, P = sla.qr(A, pivoting=True, mode="economic")
    cert = certified_steps(r, c_tie=64, u_acc=2.0 ** -52)
    fu = int(np.argmin(cert)) if not cert.all() else 70
    assert fu > 50
    assert np.array_equal(P[:fu], r.perm[:fu])
    assert np.allclose(np.abs(np.diag(R)), np.diag(r.R), rtol=1e-10, atol=1e-13 * abs(R[0, 0]))
