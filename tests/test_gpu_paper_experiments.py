"""NEXT-3: the paper's §3 experiments through the GPU path, against the
oracle's double-precision ID.

Datasets Slow / Medium / Fast (sigma_i = i^-p, p = 1, 2, 4; 1000 x 1000, P:207,
synth.gen_decay).  The double ID (Â_D = A_D(:, I_D) P_D, fp64 QRCP + P_D = R11^-1 R12)
comes from the oracle; the mixed ID (Â_M = A_D(:, I_L) P_L) from the GPU with the
paper's coefficients P_L = R11^-1 R12 of the low-precision R (Algorithm 2 lines 5-6).
Metrics: relative 2-norm distance to the double ID, ||Â_M - Â_D||_2 / ||Â_D||_2
(§3.1), and relative 2-norm error against the ground truth A_D (§3.2).

What is asserted is what the text states for single precision, in its own terms:
  * P:233 (Fast / Medium): "almost all spectral errors are smaller than single precision
    unit round-off (6e-8)" -> at least 3/4 of the ranks below 6e-8; Slow: "good
    accuracy ... larger than unit round-off" -> below 1e-5 (P:253 bounds the slow
    single-ID discrepancy by 1e-6; the mixed one is no worse, we allow 10x).
  * the low-rank error dominates -> the mixed ID's ground-truth error is
    within 1e-6 absolute of the double ID's and below the Lemma 2.1 envelope
    sqrt(1 + k(n-k)) sigma_{k+1}.
  * P:243 (column sweep, k = 20): "mixed single precision ID achieves error around
    1e-8" vs the double ID -> below 1e-6 for every n.
Half precision, every dataset, scaling none and pow2: "within 1-2
digits of accuracy of the double precision approximation in almost all cases" ->
||Â_M - Â_D||_2 / ||Â_D||_2 <= 1e-2 everywhere; and the ground-truth error stays under
the Lemma 2.1 envelope plus the half unit round-off u16 = 4.9e-4 — on Fast the
fp16 error floors near 5e-5 once sigma_{k+1} drops below it (k >= 41 exceeds the bare
envelope).  The paper's simulated-half "break" for k > 21 on Fast is not
reproduced (R15): every run completes with status ok.
"""
import math

import numpy as np
import pytest

from oracle.id import coeffs_from_R, lemma_bound
from oracle.qrcp import qrcp_householder
from synth import gen_decay

pytestmark = pytest.mark.gpu

DATASETS = {"slow": 1.0, "medium": 2.0, "fast": 4.0}
RANKS = [5, 11, 15, 21, 25, 31, 41, 51]
_DOUBLE = {}


def _double_id(name, A, kmax=51):
    """Oracle fp64 Householder QRCP (exact fp64 sums), cached per dataset; the first k
    steps of a rank-kmax run are the rank-k run."""
    if name not in _DOUBLE:
        _DOUBLE[name] = qrcp_householder(A, kmax, "fp64", acc="fp64")
    return _DOUBLE[name]


def _gpu_mixed(A, fmt, scaling, k):
    from paper_2012_00706_b200.mpid import IDError, MPID
    from tests.gpu_helpers import to_dev
    h = MPID(to_dev(A), k_max=k, fp64=fmt == "fp64")
    try:
        q = h.qrcp(fmt, scaling, k=k, allow_underflow=True)
        out = {"k_out": q.k, "status": q.status, "I": q.piv[:q.k]}
        if q.k:
            out["P"] = h.coeffs("R").cpu().numpy()
            out["rel2"] = h.error_ex("AD", 2, iters=250)[1]
            out["rel2_low"] = h.error_ex("AL", 2, iters=250)[1]
        return out
    except IDError as e:
        return {"k_out": 0, "status": e.name}
    finally:
        h.close()


def _dist_to_double(A, g, dres, k):
    PD = coeffs_from_R(dres.R, dres.perm, k)
    AD_hat = A[:, dres.perm[:k]] @ PD
    AM_hat = A[:, g["I"]] @ g["P"]
    return float(np.linalg.norm(AM_hat - AD_hat, 2) / np.linalg.norm(AD_hat, 2)), \
        float(np.linalg.norm(A - AD_hat, 2) / np.linalg.norm(A, 2))


@pytest.mark.parametrize("name", list(DATASETS))
def test_rank_sweep_single(name):
    A, sigma = gen_decay(DATASETS[name], 1000, 1000, seed=0)
    dres = _double_id(name, A)
    rows, below_u = [], 0
    for k in RANKS:
        g = _gpu_mixed(A, "fp32", "none", k)
        assert g["status"] == 0 and g["k_out"] == k
        dist, rel2_D = _dist_to_double(A, g, dres, k)
        env = lemma_bound(k, 1000, float(sigma[k]))[1]
        rows.append((k, dist, g["rel2"], rel2_D, g["rel2_low"], env))
        below_u += dist < 6e-8
        assert g["rel2"] <= env, (name, k, g["rel2"], env)
        assert abs(g["rel2"] - rel2_D) <= 1e-6, (name, k, g["rel2"], rel2_D)
        # the GPU's own double ID (ID_FP64) is the oracle's to rounding
        gd = _gpu_mixed(A, "fp64", "none", k)
        dist_D, _ = _dist_to_double(A, gd, dres, k)
        assert dist_D <= 1e-12, (name, k, dist_D)
        if name == "slow":
            assert dist < 1e-5, (k, dist)
    for r in rows:
        print(f"{name:6s} k={r[0]:2d} |M-D|/|D|={r[1]:.2e} err_M={r[2]:.3e} err_D={r[3]:.3e} "
              f"err_L={r[4]:.3e} lemma={r[5]:.2e}")
    if name != "slow":
        assert below_u >= math.ceil(0.75 * len(RANKS)), rows


def test_column_sweep_single():
    for name, p in DATASETS.items():
        A, _ = gen_decay(p, 1000, 1000, seed=0)
        for n in (100, 300, 600, 1000):
            An = np.asfortranarray(A[:, :n])
            dres = qrcp_householder(An, 20, "fp64", acc="fp64")
            g = _gpu_mixed(An, "fp32", "none", 20)
            dist, rel2_D = _dist_to_double(An, g, dres, 20)
            print(f"{name:6s} n={n:4d} |M-D|/|D|={dist:.2e} err_M={g['rel2']:.3e} err_D={rel2_D:.3e}")
            assert dist < 1e-6, (name, n, dist)


@pytest.mark.parametrize("name", list(DATASETS))
def test_rank_sweep_half(name):
    A, sigma = gen_decay(DATASETS[name], 1000, 1000, seed=0)
    dres = _double_id(name, A)
    for scaling in ("none", "pow2"):
        for k in RANKS:
            g = _gpu_mixed(A, "fp16", scaling, k)
            if g["k_out"] < k or g["status"] != 0:
                print(f"{name:6s} fp16/{scaling} k={k:2d} break: status={g['status']} k_out={g['k_out']}")
                continue
            dist, rel2_D = _dist_to_double(A, g, dres, k)
            env = lemma_bound(k, 1000, float(sigma[k]))[1]
            print(f"{name:6s} fp16/{scaling} k={k:2d} |M-D|/|D|={dist:.2e} err_M={g['rel2']:.3e} "
                  f"err_D={rel2_D:.3e} err_L={g['rel2_low']:.3e} lemma={env:.2e}")
            assert dist <= 1e-2, (name, scaling, k, dist)
            assert g["rel2"] <= env + 4.9e-4, (name, scaling, k, g["rel2"], env)
