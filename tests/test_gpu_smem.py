"""The one-launch shared-memory QRCP (formation 5, k_qrcp_smem.cu; the default for C1):
it implements the oracle's paper model operation for operation, so pivots, R and the
residual mass must equal oracle/cqrcp.c (model "paper") BIT FOR BIT — C1 (BASELINE configs[0])
in fp16 and fp32 over 5 seeds and four store intervals, tolerance stops, ragged shapes,
planted skeletons and underflow."""
import numpy as np
import pytest

from oracle.fast import qrcp_c
from oracle.id import coeffs_lsq, id_error
from oracle.qrcp import make_AL
from oracle.rounding import round_to
from synth import gen_config, gen_planted

pytestmark = pytest.mark.gpu


def _run(A, fmt, sc, k, nb=0, eps=0.0, allow_underflow=False):
    import torch
    from paper_2012_00706_b200.mpid import MPID
    h = MPID(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), k_max=k)
    q = h.qrcp(fmt, sc, k=k, nb=nb, eps=eps, formation="smem", allow_underflow=allow_underflow)
    out = {"k": q.k, "piv": q.piv, "status": q.status, "stats": h.stats()}
    if q.k > 0 and q.status == 0:
        out["R"] = h.get_R().cpu().numpy().astype(np.float64)
        out["perm"] = h.get_perm()
        out["P"] = h.coeffs("lsq").cpu().numpy()
        out["err"] = h.error()
    h.close()
    return out


def _same(out, r, k):
    assert out["k"] == r.k_out
    assert np.array_equal(out["perm"], r.perm)
    assert np.array_equal(out["R"][:, :], r.R[: out["k"], :])
    assert out["stats"]["resid_est"] == r.resid[-1]          # the same fp64 bits


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("fmt,sc", [("fp16", "pow2"), ("fp32", "none")])
@pytest.mark.parametrize("nb", [1, 4, 16, 32])
def test_C1_bit_identical_to_paper_oracle(seed, fmt, sc, nb):
    A = gen_config("C1", seed)
    out = _run(A, fmt, sc, 32, nb=nb)
    assert out["stats"]["formation"] == 5
    AL, _ = make_AL(A, fmt, sc)
    r = qrcp_c(AL, 32, fmt, nb=nb, model="paper")
    _same(out, r, 32)
    P_ref = coeffs_lsq(A, out["piv"])
    assert np.linalg.norm(out["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)


def test_default_formation_for_C1_and_tolerance_stop():
    A = gen_config("C1", 3)
    import torch
    from paper_2012_00706_b200.mpid import MPID
    h = MPID(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), k_max=100)
    q = h.qrcp("fp16", "pow2", k=100, eps=1e-3)
    st = h.stats()
    h.close()
    assert st["formation"] == 5 and st["nb"] == 16
    AL, _ = make_AL(A, "fp16", "pow2")
    r = qrcp_c(AL, 100, "fp16", nb=16, eps=1e-3, model="paper")
    assert q.k == r.k_out and np.array_equal(q.piv, r.perm[: r.k_out])


@pytest.mark.parametrize("m,n,k", [(200, 90, 30), (97, 61, 61), (8, 5, 5), (280, 150, 24)])
def test_ragged_shapes_bit_identical(m, n, k):
    rng = np.random.default_rng(m * n + k)
    A = np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 11.0)[None, :])
    for fmt, sc in (("fp16", "pow2"), ("fp32", "none")):
        out = _run(A, fmt, sc, k, nb=8)
        AL, _ = make_AL(A, fmt, sc)
        _same(out, qrcp_c(AL, k, fmt, nb=8, model="paper"), k)
        e = id_error(A, out["piv"], out["P"])
        assert abs(out["err"][1] - e[1]) <= 1e-9 * e[1]


def test_planted_and_underflow():
    A, skel, C = gen_planted(256, 128, 32, rho=1.1, eta=1e-9, seed=4)
    out = _run(A, "fp16", "pow2", 32)
    assert np.array_equal(out["piv"], skel)
    Z = np.full((40, 6), 1e-20)
    o = _run(Z, "fp16", "none", 1, allow_underflow=True)
    assert o["status"] == 4 and o["k"] == 0
