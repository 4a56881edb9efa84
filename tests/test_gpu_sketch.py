"""Sketched pivoting on the GPU (formation 4; SURVEY §8(f) NEXT-4 second option, DESIGN.md
R18) against oracle/sketch.py.

  (a) the sketch Y = Omega A_L: Omega is regenerated on the host from the same
      counter-based generator (synth.counter_sign); the tcgen05 product must lie within
      the kernel's fp32 chunk-accumulation bound of the exact fp64 product, entrywise
      (|dY_ic| <= 2048 u32 sum_r |a_rc|);
  (b) the one-CTA fp64 QRCP of Y against the oracle's QRCP of the GPU's own Y: pivots on
      the certified steps (u_acc = 2^-53), R within fp32 rounding;
  (c) end to end: planted skeleton, exact-rank reproduction, and the fp64 ID step on the
      GPU's skeleton (P to 1e-10, error to 1e-9).
"""
import numpy as np
import pytest

from oracle.id import coeffs_from_R, coeffs_lsq, id_error
from oracle.qrcp import certified_steps, make_AL
from oracle.rounding import DOUBLE, SINGLE
from oracle.sketch import sketch, sketched_qrcp
from synth import SKETCH_STREAM, counter_sign, gen_config, gen_planted

pytestmark = pytest.mark.gpu

GAMMA_GPU = 2048 * SINGLE.u


def run_sketch(A, k, oversample=10, seed=0, mode="lsq", scaling="pow2"):
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    h = MPID(to_dev(A), k_max=k)
    q = h.qrcp("fp16", scaling, k=k, formation="sketch", oversample=oversample, seed=seed, allow_underflow=True)
    Y, l = h.get_sketch()
    out = {"k": q.k, "piv": q.piv, "status": q.status, "perm": h.get_perm(), "Y": Y.cpu().numpy(), "l": l}
    if q.k > 0:
        out["R"] = h.get_R().cpu().numpy().astype(np.float64)
        out["P"] = h.coeffs(mode).cpu().numpy()
        out["err"] = h.error()
    h.close()
    return out


def _omega(seed, m, l):
    return counter_sign(seed, SKETCH_STREAM, np.arange(m), np.arange(l)).astype(np.float64)


@pytest.mark.parametrize("case,seed", [("C1", 0), ("C2", 5)])
def test_sketch_within_accumulation_bound(case, seed):
    A = gen_config(case, 0)
    if case == "C2":
        A = np.asfortranarray(A[:, :600])
    k = 20
    g = run_sketch(A, k, seed=seed)
    assert g["l"] == k + 10
    AL, _ = make_AL(A, "fp16", "pow2")
    Om = _omega(seed, A.shape[0], g["l"])
    Y = sketch(AL, Om)
    bound = GAMMA_GPU * (np.abs(Om) @ np.abs(AL))
    assert np.all(np.abs(g["Y"] - Y) <= bound + 1e-300), float(np.max(np.abs(g["Y"] - Y) / (bound + 1e-300)))
    assert np.max(np.abs(g["Y"] - Y)) <= 1e-4 * np.max(np.abs(Y))     # a misplaced tile would be O(1)


@pytest.mark.parametrize("case", ["C1", "C2"])
def test_small_qrcp_on_gpu_sketch(case):
    A = gen_config(case, 0)
    if case == "C2":
        A = np.asfortranarray(A[:, :600])
    k = 20
    g = run_sketch(A, k)
    res = sketched_qrcp(g["Y"], k)
    cert = certified_steps(res, c_tie=64.0, u_acc=DOUBLE.u)
    first = int(np.argmin(cert)) if not cert.all() else k
    agree = 0
    while agree < k and g["piv"][agree] == res.perm[agree]:
        agree += 1
    assert agree >= first, (agree, first)
    if agree == k:
        assert np.array_equal(g["perm"], res.perm)
        assert np.max(np.abs(g["R"] - res.R)) <= 4 * SINGLE.u * np.max(np.abs(res.R))


def test_sketch_planted_and_exact_rank():
    A, skel, _ = gen_planted(4096, 300, 24, rho=1.05, eta=1e-9, seed=3)
    g = run_sketch(A, 24)
    assert set(g["piv"]) == set(skel)
    rng = np.random.default_rng(4)
    B = np.asfortranarray(rng.standard_normal((3000, 12)) @ rng.standard_normal((12, 200)))
    g = run_sketch(B, 12, scaling="none")
    P = coeffs_lsq(B, g["piv"])
    assert id_error(B, g["piv"], P)[1] < 1e-6        # fp16 A_L picks an independent skeleton


@pytest.mark.parametrize("mode", ["lsq", "R"])
def test_sketch_fp64_id_step(mode):
    A = np.asfortranarray(gen_config("C2", 0)[:, :600])
    k = 32
    g = run_sketch(A, k, mode=mode, seed=2, oversample=16)
    P_ref = coeffs_lsq(A, g["piv"]) if mode == "lsq" else coeffs_from_R(g["R"], g["perm"], k)
    assert np.linalg.norm(g["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    e = id_error(A, g["piv"], g["P"])
    assert abs(g["err"][0] - e[0]) <= 1e-9 * e[0]
    # a sketched skeleton is a good one: within 2x of the Householder QRCP's error here
    from tests.gpu_helpers import run_gpu
    h = run_gpu(A, "fp16", "pow2", k)
    assert e[1] <= 2.0 * h["err"][1] + 1e-12
