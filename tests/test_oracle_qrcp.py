"""Pins for oracle/qrcp.py (O4): pivoted Householder QR in the simulated low precision.

Pins (none retypes the oracle's own formulas):
  * SPEC hand examples S:195-196;
  * LAPACK dgeqp3 (scipy.linalg.qr(pivoting=True)) in fp64;
  * the paper-literal MGS variant (different algorithm, same exact-arithmetic result);
  * brute-force greedy projection pivots (oracle/bruteforce.py) on tiny inputs;
  * planted-skeleton inputs whose pivots are known in closed form;
  * exact-rank inputs; QR invariants (A Z = Q R, Q^T Q = I, |R_jj| non-increasing);
  * a hand-computed store-point example (reading R4).
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.bruteforce import greedy_pivots
from oracle.qrcp import (certified_steps, form_Q, make_AL, qrcp_householder, qrcp_mgs)
from oracle.rounding import HALF, SINGLE, round_to
from synth import gen_config, gen_exact_rank, gen_planted

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("fmt", ["fp64", "fp32", "fp16"])
def test_hand_example_S196(fmt):
    g = GOLD["qr_hand"]
    A = np.array(g["A"], dtype=np.float64)
    r = qrcp_householder(A, g["k"], fmt)
    assert list(r.perm[:1]) == g["piv"][:1]
    tol = 0 if fmt == "fp64" else SINGLE.u
    assert abs(r.R[0, 0] - 5.0) <= 5 * tol + 1e-15
    assert abs(r.R[0, 1] - 1.4) <= 1.4 * 2 * SINGLE.u + 1e-15
    Q = form_Q(r.V, r.tau)
    s = np.sign(Q[0, 0])
    assert np.allclose(s * Q[:, 0], g["Q"], atol=1e-7)
    pm, Rm, Qm = qrcp_mgs(A, 1, fmt)
    tolm = HALF.u if fmt == "fp16" else SINGLE.u       # MGS stores r_ji in the low format (S:192e)
    assert list(pm[:1]) == g["piv"][:1] and abs(Rm[0, 1] - 1.4) <= 1.4 * 3 * tolm


def test_identity_ties_S195():
    g = GOLD["qr_identity"]
    r = qrcp_householder(np.eye(g["n"]), g["k"], "fp64")
    assert list(r.perm[: g["k"]]) == g["piv"]
    assert np.allclose(np.abs(r.R), np.array(g["R"], dtype=float))


def test_fp64_matches_lapack_dgeqp3():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((200, 60)) @ np.diag(np.exp(-np.arange(60) / 10.0)) @ sla.qr(rng.standard_normal((60, 60)))[0]
    r = qrcp_householder(A, 60, "fp64")
    Q, R, P = sla.qr(A, pivoting=True, mode="economic")
    cert = certified_steps(r, c_tie=64, u_acc=2.0 ** -52)
    first_unc = int(np.argmin(cert)) if not cert.all() else 60
    assert first_unc > 40
    assert np.array_equal(P[:first_unc], r.perm[:first_unc])
    assert np.allclose(np.abs(np.diag(R)), np.diag(r.R), rtol=1e-10, atol=1e-13 * abs(R[0, 0]))
    assert np.allclose(np.abs(R[:first_unc]), np.abs(r.R[:first_unc]), rtol=1e-9, atol=1e-12 * abs(R[0, 0]))


def test_fp64_householder_equals_mgs():
    A = gen_config("C1")
    r = qrcp_householder(A, 32, "fp64")
    pm, Rm, Qm = qrcp_mgs(A, 32, "fp64")
    assert np.array_equal(pm[:32], r.perm[:32])
    assert np.allclose(np.abs(Rm), np.abs(r.R), atol=1e-12 * abs(r.R[0, 0]))


@pytest.mark.parametrize("seed", range(6))
def test_bruteforce_greedy_pivots(seed):
    rng = np.random.default_rng(seed)
    m, n, k = 9, 8, 4
    A = rng.standard_normal((m, n)) * np.exp(rng.uniform(-2, 1, n))[None, :]
    ref = greedy_pivots(A, k)
    assert list(qrcp_householder(A, k, "fp64").perm[:k]) == ref
    AL = round_to(A, "fp32").reshape(A.shape)
    r32 = qrcp_householder(AL, k, "fp32")
    if certified_steps(r32).all():
        assert list(r32.perm[:k]) == greedy_pivots(AL, k)


def test_first_pivot_is_max_norm_column():
    A = gen_config("C2")
    for fmt, sc in (("fp32", "none"), ("fp16", "maxabs")):
        AL, _ = make_AL(A, fmt, sc)
        r = qrcp_householder(AL[:, :300], 1, fmt)
        assert r.perm[0] == int(np.argmax(np.linalg.norm(AL[:, :300], axis=0)))


@pytest.mark.parametrize("fmt,nb", [("fp64", 1), ("fp32", 8), ("fp16", 1), ("fp16", 8), ("fp16", 32)])
def test_planted_skeleton(fmt, nb):
    A, skel, C = gen_planted(256, 128, 32, rho=1.1, eta=1e-9, seed=1)
    AL, _ = make_AL(A, fmt, "pow2" if fmt == "fp16" else "none")
    r = qrcp_householder(AL, 32, fmt, nb=nb)
    assert r.status == "ok"
    assert sorted(r.perm[:32]) == sorted(skel)
    assert np.array_equal(r.perm[:32], skel)          # planted order: decreasing rho^-(j-1)


@pytest.mark.parametrize("fmt", ["fp64", "fp32", "fp16"])
def test_qr_invariants(fmt):
    A = gen_config("C1")
    AL, _ = make_AL(A, fmt, "pow2" if fmt == "fp16" else "none")
    k, nb = 32, 8
    r = qrcp_householder(AL, k, fmt, nb=nb)
    Q = form_Q(r.V, r.tau)
    u_L = {"fp64": 2.0 ** -53, "fp32": SINGLE.u, "fp16": HALF.u}[fmt]
    u_acc = 2.0 ** -53 if fmt == "fp64" else SINGLE.u
    assert np.linalg.norm(Q.T @ Q - np.eye(k)) <= 10 * k * u_acc
    # residual of the first k pivoted columns (A35): || A_L Z(:,1:k) - Q R(:,1:k) ||
    D = np.diag(np.sign(np.diag(Q.T @ AL[:, r.perm[:k]])))   # row signs removed by R_jj >= 0
    res = np.linalg.norm(AL[:, r.perm[:k]] - (Q @ D) @ np.triu(r.R[:, :k]))
    eta = (math.ceil(k / nb) + 2 * math.sqrt(k)) * u_L + 4 * k * 300 * u_acc
    assert res <= (eta + u_acc) * np.linalg.norm(AL)
    d = np.diag(r.R)
    assert np.all(d >= 0)
    mx = r.maxnorm0
    assert np.all(d[1:] <= d[:-1] * (1 + 4 * u_L) + 64 * u_acc * mx)        # A36


def test_exact_rank_stops_on_tolerance():
    A = gen_exact_rank(300, 80, 12, seed=2)
    r = qrcp_householder(A, 40, "fp64", eps=1e-10)
    assert r.k_out == 12
    r32 = qrcp_householder(round_to(A, "fp32").reshape(A.shape), 40, "fp32", eps=1e-5)
    assert r32.k_out == 12


def test_store_point_hand_example():
    """A = [[3,1],[4,1],[0,0]]: after step 0, W(1,1) = 1 - 0.5*2.4 = -0.2 (fp32); with
    nb = 1 it is stored as fl16(-0.2) = -0.199951171875 before the step-1 norm, so
    R(1,1) = 0.199951171875; with nb = 2 no store happens and R(1,1) = fl32(0.2)."""
    A = np.array([[3.0, 1.0], [4.0, 1.0], [0.0, 0.0]])
    r1 = qrcp_householder(A, 2, "fp16", nb=1)
    r2 = qrcp_householder(A, 2, "fp16", nb=2)
    assert r1.R[1, 1] == 0.199951171875
    assert abs(r2.R[1, 1] - 0.2) <= 4 * SINGLE.u
    assert r2.R[1, 1] != 0.199951171875


def test_underflow_status():
    A = np.full((4, 3), 1e-20)
    AL = round_to(A, "fp16").reshape(A.shape)          # 1e-20 -> 0 in binary16
    r = qrcp_householder(AL, 1, "fp16")
    assert r.status == "underflow" and r.k_out == 0


def test_fp32_pivots_match_fp64_on_gapped_input():
    A, skel, C = gen_planted(1024, 256, 48, rho=1.05, eta=1e-8, seed=4)
    r64 = qrcp_householder(A, 48, "fp64")
    r32 = qrcp_householder(round_to(A, "fp32").reshape(A.shape), 48, "fp32", nb=16)
    assert np.array_equal(r64.perm[:48], r32.perm[:48])


@pytest.mark.parametrize("fmt,nb", [("fp16", 4), ("fp32", 4), ("fp64", 1)])
def test_norm_and_accumulation_variants_agree_on_certified_steps(fmt, nb):
    """Reading R5/R6 cross-check: the one-step downdate vs recomputing the norms every
    step, and the 8-row fp32 chains vs fp64 accumulation, give the same
    pivots on every certified step."""
    A = gen_config("C1")
    AL, _ = make_AL(A, fmt, "pow2" if fmt == "fp16" else "none")
    base = qrcp_householder(AL, 32, fmt, nb=nb)
    cert = certified_steps(base)
    fu = int(np.argmin(cert)) if not cert.all() else 32
    assert fu >= 20
    for kw in ({"norms": "recompute"}, {"acc": "fp64"}, {"norms": "recompute", "acc": "fp64"}):
        alt = qrcp_householder(AL, 32, fmt, nb=nb, **kw)
        assert np.array_equal(alt.perm[:fu], base.perm[:fu]), kw


def test_chain8_is_an_accurate_sum():
    """The blocked order stays within a few fp32 ulps of the exact (fsum) column sums."""
    from oracle.qrcp import chain8
    rng = np.random.default_rng(1)
    X = rng.standard_normal((4096, 5)).astype(np.float32)
    got = chain8(X, X, np.float32)
    ref = np.array([math.fsum(float(v) ** 2 for v in X[:, c]) for c in range(5)])
    assert np.all(np.abs(got - ref) <= 8 * SINGLE.u * ref)


# ---- formation "tc" (the D-OTF form the tensor-core pass follows) and model "paper" ----
# Pins: LAPACK dgeqp3 / the fp64 Householder QR of the same A_L (an exact-arithmetic
# identity: every formation computes the same R), the right-looking formation (a
# different order of the same operations), planted skeletons, and the QR invariants
# A35 (factorisation residual) / A36 (|diag R| non-increasing).

@pytest.mark.parametrize("nb", [8, 32])
def test_tc_formation_R_matches_fp64_householder(nb):
    """fp32 storage, no store inside the run (nb >= k) or every 8 steps: the D-OTF
    formation's R equals the fp64 QR of the same A_L to a few fp32 units."""
    A = gen_config("C1", 1)
    AL, _ = make_AL(A, "fp32", "none")
    k = 32
    r = qrcp_householder(AL, k, "fp32", nb=nb, formation="tc")
    r64 = qrcp_householder(AL, k, "fp64")
    Q, R, P = sla.qr(AL, pivoting=True, mode="economic")
    cert = certified_steps(r)
    fu = int(np.argmin(cert)) if not cert.all() else k
    assert fu >= 24
    assert np.array_equal(r.perm[:fu], P[:fu]) and np.array_equal(r.perm[:fu], r64.perm[:fu])
    mx = r.maxnorm0
    assert np.max(np.abs(r.R[:fu, :] - r64.R[:fu, :])) <= 64 * k * SINGLE.u * mx


@pytest.mark.parametrize("fmt,nb", [("fp16", 32), ("fp16", 8), ("fp32", 32)])
def test_tc_formation_planted_and_invariants(fmt, nb):
    A, skel, C = gen_planted(512, 128, 32, rho=1.1, eta=1e-9, seed=2)
    AL, _ = make_AL(A, fmt, "pow2" if fmt == "fp16" else "none")
    r = qrcp_householder(AL, 32, fmt, nb=nb, formation="tc")
    assert np.array_equal(r.perm[:32], skel)
    k = 32
    u_L = HALF.u if fmt == "fp16" else SINGLE.u
    u_acc = SINGLE.u
    Q = form_Q(r.V, r.tau)
    D = np.diag(np.sign(np.diag(Q.T @ AL[:, r.perm[:k]])))
    res = np.linalg.norm(AL[:, r.perm[:k]] - (Q @ D) @ np.triu(r.R[:, :k]))
    eta = (math.ceil(k / nb) + 2 * math.sqrt(k)) * u_L + 4 * k * 300 * u_acc
    assert res <= (eta + u_acc) * np.linalg.norm(AL)                     # A35
    d = np.diag(r.R)
    assert np.all(d >= 0) and np.all(d[1:] <= d[:-1] * (1 + 4 * u_L) + 64 * u_acc * r.maxnorm0)   # A36


@pytest.mark.parametrize("fmt,nb", [("fp16", 32), ("fp16", 4), ("fp32", 16)])
def test_tc_and_paper_models_agree_with_kernel_model_on_certified_steps(fmt, nb):
    """Three faithful orders of the same precision model — D-OTF formation with fp64
    sums, right-looking with per-op rounding + fp64 sums ("paper"), right-looking with
    one-rounding updates + 8-row fp32 chains ("kernel") — pick the same pivots on every
    certified step and reach the same residual mass to a few storage units."""
    A = gen_config("C1", 3)
    AL, _ = make_AL(A, fmt, "pow2" if fmt == "fp16" else "none")
    runs = [qrcp_householder(AL, 32, fmt, nb=nb, formation="tc"),
            qrcp_householder(AL, 32, fmt, nb=nb, model="paper"),
            qrcp_householder(AL, 32, fmt, nb=nb, model="kernel")]
    cert = certified_steps(runs[1], c_tie=64)
    fu = int(np.argmin(cert)) if not cert.all() else 32
    assert fu >= 20
    for r in runs[1:]:
        assert np.array_equal(r.perm[:fu], runs[0].perm[:fu])
    u_L = HALF.u if fmt == "fp16" else SINGLE.u
    for r in runs[1:]:
        assert abs(r.resid[fu] - runs[0].resid[fu]) <= 64 * u_L * runs[0].resid[0]
