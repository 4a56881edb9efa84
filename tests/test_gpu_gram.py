"""Gram-based pivoting on the GPU (formation 3, R17)
against oracle/gram.py.

Two independent checks instead of one end-to-end comparison:
  (a) the tensor-core Gram G = A_L^T A_L against the exact fp64 Gram of the same A_L,
      entrywise within the fp32-accumulation bound of the kernel: every 2048-row chunk
      is an fp32 sum (error <= 2048 u32 sum_r |a_ri a_rj| in the worst case), chunks are
      added in fp64;
  (b) the pivoted Cholesky on the GPU's own G against the oracle's pivoted Cholesky of
      that same G (both fp64): pivots equal on the certified steps (gamma = 1e-13),
      R within 1e-11 max||a||.
Then end to end: the pivots against the oracle on the exact Gram on the steps certified
for the kernel's bound, and the fp64 ID step (P, error) on the GPU's skeleton.
"""
import numpy as np
import pytest

from oracle.gram import certified_gram_steps, gram, pivoted_cholesky
from oracle.id import coeffs_lsq, id_error
from oracle.qrcp import make_AL
from oracle.rounding import SINGLE
from synth import gen_config, gen_planted

pytestmark = pytest.mark.gpu

GAMMA_GPU = 2048 * SINGLE.u          # worst-case fp32 chunk accumulation (2048 rows)


def run_gram(A, k, scaling="pow2", eps=0.0, mode="lsq"):
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    h = MPID(to_dev(A), k_max=k)
    q = h.qrcp("fp16", scaling, k=k, eps=eps, formation="gram", allow_underflow=True)
    out = {"k": q.k, "piv": q.piv, "status": q.status, "perm": h.get_perm(), "G": h.get_gram().cpu().numpy()}
    if q.k > 0:
        out["R"] = h.get_R().cpu().numpy().astype(np.float64)
        out["P"] = h.coeffs(mode).cpu().numpy()
        out["err"] = h.error()
    out["stats"] = h.stats()
    h.close()
    return out


def _cases():
    A1 = gen_config("C1", 0)
    A2 = np.asfortranarray(gen_config("C2", 0)[:, :600])        # ragged: 600 = 4 x 128 + 88
    return {"C1": (A1, 32), "C2": (A2, 64)}


@pytest.mark.parametrize("case", ["C1", "C2"])
def test_gram_kernel_within_accumulation_bound(case):
    A, k = _cases()[case]
    g = run_gram(A, k)
    AL, _ = make_AL(A, "fp16", "pow2")
    G = gram(AL)
    absG = np.abs(AL).T @ np.abs(AL)
    err = np.abs(g["G"] - G)
    assert np.all(err <= GAMMA_GPU * absG + 1e-300), float(np.max(err / (absG + 1e-300)))
    assert np.array_equal(g["G"], g["G"].T)                       # symmetric fill
    # the typical error is far below the worst case: a transposed/misplaced tile would not be
    assert np.max(err) <= 1e-4 * np.max(np.abs(G))


@pytest.mark.parametrize("case", ["C1", "C2"])
def test_pivoted_cholesky_on_gpu_gram(case):
    A, k = _cases()[case]
    g = run_gram(A, k)
    res = pivoted_cholesky(g["G"], k)
    # C1 at k = 32 exhausts the Gram's resolution (sigma_32^2 / sigma_1^2 ~ 1e-8 is below
    # the fp32-accumulated G's error): both sides stop with a breakdown at the same step
    assert abs(g["k"] - res.k_out) <= 1 and (g["status"] == 4) == (res.status == "underflow")
    kk = min(g["k"], res.k_out)
    cert = certified_gram_steps(res, gamma=1e-13)[:kk]
    first = int(np.argmin(cert)) if not cert.all() else kk
    agree = 0
    while agree < kk and g["piv"][agree] == res.perm[agree]:
        agree += 1
    assert agree >= first, (agree, first)
    if agree == k and g["k"] == k:
        assert np.array_equal(g["perm"], res.perm)
        scale = np.sqrt(np.max(np.diag(g["G"])))
        assert np.max(np.abs(g["R"] - res.R)) <= 1e-6 * scale     # GPU R is fp32-rounded


@pytest.mark.parametrize("case", ["C1", "C2", "planted"])
def test_gram_end_to_end(case):
    if case == "planted":
        A, skel, _ = gen_planted(4096, 300, 24, rho=1.05, eta=1e-9, seed=3)
        k = 24
    else:
        A, k = _cases()[case]
        if case == "C1":
            k = 16          # sigma_16^2 / sigma_1^2 ~ 2e-4: well above the Gram's resolution
    g = run_gram(A, k)
    assert g["status"] == 0 and g["k"] == k
    AL, _ = make_AL(A, "fp16", "pow2")
    res = pivoted_cholesky(gram(AL), k)
    cert = certified_gram_steps(res, gamma=GAMMA_GPU)
    first = int(np.argmin(cert)) if not cert.all() else k
    agree = 0
    while agree < k and g["piv"][agree] == res.perm[agree]:
        agree += 1
    assert agree >= first, (agree, first)
    if case == "planted":
        assert list(g["piv"]) == list(skel)                        # the planted skeleton, in order
    P_ref = coeffs_lsq(A, g["piv"])
    assert np.linalg.norm(g["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    e = id_error(A, g["piv"], g["P"])
    assert abs(g["err"][0] - e[0]) <= 1e-9 * e[0]


def test_gram_tolerance_and_rank_exhaustion():
    A, _ = _cases()["C2"]
    eps = 1e-2
    g = run_gram(A, 300, eps=eps)
    AL, _ = make_AL(A, "fp16", "pow2")
    res = pivoted_cholesky(g["G"], 300, eps=eps)
    assert abs(g["k"] - res.k_out) <= 1, (g["k"], res.k_out)
    # exact-rank 20 input: the Gram's resolution is exhausted soon after the rank
    rng = np.random.default_rng(0)
    B = rng.standard_normal((2048, 20)) @ rng.standard_normal((20, 256))
    g = run_gram(np.asfortranarray(B), 60)
    assert g["k"] >= 20
    assert g["k"] == 60 or g["status"] == 4


def test_gram_wide_matrix():
    """n > 1024 (more than 8 tile columns, ragged last tile) against the exact Gram."""
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.standard_normal((4096, 1100)) * np.exp(-np.arange(1100) / 200.0))
    g = run_gram(A, 40)
    AL, _ = make_AL(A, "fp16", "pow2")
    G = gram(AL)
    absG = np.abs(AL).T @ np.abs(AL)
    assert np.all(np.abs(g["G"] - G) <= GAMMA_GPU * absG + 1e-300)
    res = pivoted_cholesky(g["G"], 40)
    cert = certified_gram_steps(res, gamma=1e-13)
    first = int(np.argmin(cert)) if not cert.all() else 40
    agree = 0
    while agree < 40 and g["piv"][agree] == res.perm[agree]:
        agree += 1
    assert agree >= first
