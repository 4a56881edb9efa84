"""Pins for oracle/sketch.py (O10, NEXT-4 second option) and synth.counter_sign.

  * the generator: entries +-1, balanced, independent of the row split (counter-based),
    E[Omega^T Omega] = l I checked through the Johnson-Lindenstrauss norm ratio;
  * exact-rank input: the sketched skeleton reproduces A exactly (LSQ error ~ 0);
  * planted skeleton: the sketch recovers the planted columns;
  * orthogonal columns with well separated norms: the pivots follow the norm order;
  * l >= m with Omega = identity rows is the unsketched QRCP (pivots equal).
"""
import numpy as np

from oracle.id import coeffs_lsq, id_error
from oracle.qrcp import qrcp_householder
from oracle.sketch import sketch, sketched_qrcp
from synth import SKETCH_STREAM, counter_sign, gen_planted


def test_counter_sign_properties():
    S = counter_sign(3, SKETCH_STREAM, np.arange(20000), np.arange(64))
    assert S.shape == (64, 20000) and set(np.unique(S)) == {-1, 1}
    assert abs(S.mean()) < 0.01
    # counter-based: a row block drawn alone equals the same rows of the full draw
    assert np.array_equal(counter_sign(3, SKETCH_STREAM, np.arange(5000, 6000), np.arange(64)), S[:, 5000:6000])
    # columns are (nearly) orthogonal: Omega Omega^T / m ~ I
    C = S.astype(np.float64) @ S.T.astype(np.float64) / S.shape[1]
    assert np.max(np.abs(C - np.eye(64))) < 0.05


def test_jl_norm_preservation():
    rng = np.random.default_rng(0)
    m, l = 4000, 256
    Om = counter_sign(1, SKETCH_STREAM, np.arange(m), np.arange(l)).astype(np.float64)
    X = rng.standard_normal((m, 50))
    ratio = np.sum((Om @ X) ** 2, axis=0) / (l * np.sum(X ** 2, axis=0))
    assert np.all(np.abs(ratio - 1.0) < 5 * np.sqrt(2.0 / l))


def test_exact_rank_is_reproduced():
    rng = np.random.default_rng(4)
    m, n, r = 3000, 200, 12
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    Om = counter_sign(0, SKETCH_STREAM, np.arange(m), np.arange(r + 8))
    res = sketched_qrcp(sketch(A, Om), r)
    I = res.perm[:r]
    P = coeffs_lsq(A, I)
    assert id_error(A, I, P)[1] < 1e-10


def test_planted_skeleton_recovered():
    A, skel, _ = gen_planted(4096, 300, 24, rho=1.05, eta=1e-9, seed=3)
    Om = counter_sign(0, SKETCH_STREAM, np.arange(4096), np.arange(40))
    res = sketched_qrcp(sketch(A, Om), 24)
    assert set(res.perm[:24]) == set(skel)


def test_orthogonal_columns_norm_order():
    rng = np.random.default_rng(7)
    Q = np.linalg.qr(rng.standard_normal((2000, 8)))[0]
    norms = np.array([3.0, 7.0, 1.0, 5.0, 2.0, 11.0, 4.0, 8.0]) ** 1.5
    A = Q * norms
    Om = counter_sign(2, SKETCH_STREAM, np.arange(2000), np.arange(512))
    res = sketched_qrcp(sketch(A, Om), 8)
    assert list(res.perm) == list(np.argsort(-norms))


def test_identity_sketch_is_plain_qrcp():
    rng = np.random.default_rng(9)
    A = rng.standard_normal((60, 40)) @ np.diag(np.exp(-np.arange(40) / 6.0))
    res = sketched_qrcp(sketch(A, np.eye(60)), 20)
    ref = qrcp_householder(A, 20, "fp64", acc="fp64")
    assert np.array_equal(res.perm[:20], ref.perm[:20])
