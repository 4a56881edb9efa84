"""Pins for oracle/id.py (O5-O7): coefficients, error, bounds.

Pins: SPEC S:250-252 coefficient examples; numpy's lstsq; exact-rank and
planted inputs (P(:,J) = C, zero error); Eckart-Young; the Pythagorean identity
of an orthogonal projection; Lemma 2.1 numbers;
Table 3 singular-value ratios.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle.id import (coeffs_from_R, coeffs_lsq, eckart_young_fro, id_error, lemma_bound,
                       post_bound)
from oracle.qrcp import make_AL, qrcp_householder
from oracle.rounding import HALF, SINGLE
from synth import gen_config, gen_decay, gen_exact_rank, gen_planted

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("c", GOLD["coef_examples"], ids=lambda c: c["cite"])
def test_spec_coefficient_examples(c):
    R = np.array(c["R"], dtype=float)
    P = coeffs_from_R(R, np.array(c["piv"]), c["k"], pinv_tol=1e-12 if c.get("pinv") else None)
    assert np.allclose(P, np.array(c["P"]), atol=1e-15)


def test_lsq_matches_numpy_lstsq():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((120, 40))
    I = np.array([3, 17, 5, 30, 11])
    P = coeffs_lsq(A, I)
    X, *_ = np.linalg.lstsq(A[:, I], A, rcond=None)
    assert np.allclose(P, X, atol=1e-12)
    assert np.array_equal(P[:, I], np.eye(5))


def test_exact_rank_zero_error_and_planted_C():
    A = gen_exact_rank(200, 60, 7, seed=1)
    r = qrcp_householder(A, 7, "fp64")
    P = coeffs_lsq(A, r.I)
    assert id_error(A, r.I, P)[1] <= 1e-12
    A2, skel, C = gen_planted(256, 128, 32, rho=1.1, eta=0.0, seed=2)
    P2 = coeffs_lsq(A2, skel)
    J = np.setdiff1d(np.arange(128), skel)
    assert id_error(A2, skel, P2)[1] <= 1e-12
    # P(:, J) reproduces C up to the generator's column permutation
    assert np.abs(np.sort(P2[:, J].ravel()) - np.sort(C.ravel())).max() <= 1e-10


def test_R_mode_equals_lsq_in_fp64():
    A = gen_config("C1")
    r = qrcp_householder(A, 32, "fp64")
    PR = coeffs_from_R(r.R, r.perm, 32)
    PL = coeffs_lsq(A, r.I)
    kappa = np.linalg.cond(A[:, r.I])
    assert np.linalg.norm(PR - PL) / np.linalg.norm(PL) <= 1e-15 * kappa ** 2 + 1e-12


def test_error_properties():
    A = gen_config("C1")
    sigma = 10.0 ** (-np.arange(128) / 8.0)
    AL, s = make_AL(A, "fp16", "pow2")
    r = qrcp_householder(AL, 32, "fp16", nb=32)
    P = coeffs_lsq(A, r.I)
    E = A - A[:, r.I] @ P
    assert np.all(E[:, r.I] == 0.0)                                  # skeleton columns exact
    ab, rel = id_error(A, r.I, P)
    ey = eckart_young_fro(sigma, 32)
    assert ey <= ab                                                   # Eckart-Young lower bound
    Q, _ = np.linalg.qr(A[:, r.I])
    pyth = math.sqrt(max(np.linalg.norm(A) ** 2 - np.linalg.norm(Q.T @ A) ** 2, 0.0))
    assert abs(pyth - ab) <= 1e-6 * ab                               # orthogonal projection
    T2 = np.linalg.norm(coeffs_from_R(r.R, r.perm, 32), 2)
    Bp = post_bound(r.resid[32], s, T2, np.linalg.norm(A),
                    HALF.u, 32, 32, 256, SINGLE.u)
    assert ab <= Bp


def test_lemma_numbers():
    g = GOLD["lemma"]
    c, b = lemma_bound(g["k"], g["n"], g["sigma"])
    assert abs(c - g["c"]) <= g["abs_tol"] and abs(b - g["bound"]) <= g["abs_tol"]
    f = GOLD["paper_bound_fast"]
    k = f["k"]
    # P:241's 3.3e-5 is reproduced with sigma_k (reading R14); with sigma_{k+1} it is 3.0e-5
    assert abs(lemma_bound(k, f["n"], k ** -4.0)[1] - f["value"]) <= f["rel_tol"] * f["value"]
    assert lemma_bound(k, f["n"], (k + 1) ** -4.0)[1] < 0.95 * f["value"]
    o = GOLD["optimal_rank20"]
    assert abs(21.0 ** -1 - o["slow"]) < 1e-15 and abs(21.0 ** -2 - o["medium"]) < 1e-15
    assert 0.5 * o["fast_approx"] <= 21.0 ** -4 <= 2 * o["fast_approx"]


@pytest.mark.parametrize("t", GOLD["table3_ratios"], ids=lambda t: t["cite"])
def test_table3_ratios_and_generator_spectrum(t):
    p = t["p"]
    assert abs(50.0 ** -p - t["s50_s1"]) <= 0.05 * t["s50_s1"]
    assert abs(1000.0 ** -p - t["sn_s1"]) <= 1e-3 * t["sn_s1"]
    A, sigma = gen_decay(p, 300, 200, seed=0)
    s = np.linalg.svd(A, compute_uv=False)
    big = sigma > 1e-13
    assert np.allclose(s[big], sigma[big], rtol=1e-10, atol=1e-15)


def test_blocked_error_equals_definition():
    """id_error_blocked (used at full size) against the fsum definition id_error."""
    from oracle.id import id_error_blocked
    A = gen_config("C2", 0)[:, :300]
    I = np.array([5, 17, 2, 250, 99, 64, 130])
    P = coeffs_lsq(A, I)
    a = id_error(A, I, P)
    b = id_error_blocked(A, I, P, cols=37)
    assert abs(a[0] - b[0]) <= 1e-13 * a[0] and abs(a[1] - b[1]) <= 1e-13 * a[1]


def test_low_skeleton_and_spectral_error_pins():
    """Â_L skeleton = RNE rounding of the scaled columns (pinned by numpy's fp16/fp32
    casts, which round once from fp64); the 2-norm error equals the largest singular
    value of the residual and is >= the Eckart-Young 2-norm bound sigma_{k+1}."""
    from oracle.id import id_error_skeleton, low_skeleton, spectral_error
    A, sigma = gen_decay(2, 120, 80, seed=4)
    I = np.array([0, 5, 9, 17, 33])
    for fmt, dt in (("fp16", np.float16), ("fp32", np.float32)):
        X = low_skeleton(A, I, fmt, 8.0)
        assert np.array_equal(X, (A[:, I] * 8.0).astype(dt).astype(np.float64) / 8.0)
    P = coeffs_lsq(A, I)
    e2, r2 = spectral_error(A, A[:, I], P)
    assert e2 >= sigma[len(I)] * (1 - 1e-12)
    assert abs(r2 - e2 / sigma[0]) <= 1e-12 * r2
    ef, _ = id_error_skeleton(A, A[:, I], P)
    assert abs(ef - id_error(A, I, P)[0]) <= 1e-12 * ef and e2 <= ef * (1 + 1e-12)


def test_post_bound_reduces_to_the_exact_error_and_holds():
    """B_post (reading R13) pins: (i) with u_L = u_acc = 0 it is rho_k / s, the QR's
    residual mass, which in exact arithmetic IS the LSQ-ID error ||(I - Q Q^T) A||_F —
    checked on fp64 QRCPs (no storage rounding, s = 1) to 1e-9; (ii) it is monotone in
    u_L; (iii) it holds (err <= B_post) and is not vacuous (B_post < ||A||_F / 4) on
    fp16 / fp32 runs of C1 (3 seeds), a C2 slice and a planted input."""
    from oracle.rounding import SINGLE as S32
    for seed in range(3):
        A = gen_config("C1", seed)
        r = qrcp_householder(A, 32, "fp64")
        e = id_error(A, r.I, coeffs_lsq(A, r.I))[0]
        B0 = post_bound(r.resid[32], 1.0, 5.0, np.linalg.norm(A), 0.0, 32, 32, 256, 0.0)
        assert abs(B0 - e) <= 1e-9 * e
    cases = [(gen_config("C1", s), "fp16", "pow2", 32, 32) for s in range(3)]
    cases += [(gen_config("C1", 0), "fp32", "none", 32, 4)]
    cases += [(np.asfortranarray(gen_config("C2", 0)[:, :256]), "fp16", "maxabs", 64, 4)]
    A, _, _ = gen_planted(512, 128, 32, rho=1.1, eta=1e-9, seed=5)
    cases += [(A, "fp16", "pow2", 32, 8)]
    for A, fmt, sc, k, nb in cases:
        AL, s = make_AL(A, fmt, sc)
        r = qrcp_householder(AL, k, fmt, nb=nb)
        P = coeffs_lsq(A, r.I)
        ab, _ = id_error(A, r.I, P)
        T2 = np.linalg.norm(coeffs_from_R(r.R, r.perm, k), 2)
        uL = HALF.u if fmt == "fp16" else S32.u
        B = post_bound(r.resid[k], s, T2, np.linalg.norm(A), uL, k, nb, A.shape[0], S32.u)
        B2 = post_bound(r.resid[k], s, T2, np.linalg.norm(A), 2 * uL, k, nb, A.shape[0], S32.u)
        assert ab <= B < B2
        assert B < 0.25 * np.linalg.norm(A)
