"""The double ID on the GPU (ID_FP64; Â_D of P:196, Algorithm 1
P:143-155) against the oracle's fp64 QRCP and against LAPACK's dgeqp3.

Reading R16: in fp64 both sides round every product and every sum
separately (the oracle cannot fuse an fp64 multiply-add), so the formed trailing
matrix is the oracle's element for element; the 8-row group partials are added in a
different order (numpy pairwise vs. the kernel's per-warp order), so R agrees to a few
ulps, not bit for bit, and pivots are compared on the certified steps (R10 with
u_acc = 2^-53).
"""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle.id import coeffs_from_R, coeffs_lsq, id_error
from oracle.qrcp import certified_steps, make_AL, qrcp_householder
from oracle.rounding import DOUBLE
from synth import gen_config, gen_decay

pytestmark = pytest.mark.gpu


def run64(A, k, nb=4, scaling="none", eps=0.0, mode="lsq"):
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    h = MPID(to_dev(A), k_max=k, fp64=True)
    q = h.qrcp("fp64", scaling, k=k, nb=nb, eps=eps)
    out = {"k": q.k, "piv": q.piv, "perm": h.get_perm(), "R": h.get_R64().cpu().numpy(),
           "R32": h.get_R().cpu().numpy()}
    out["P"] = h.coeffs(mode).cpu().numpy()
    out["err"] = h.error()
    out["stats"] = h.stats()
    h.close()
    return out


def _prefix(piv, res):
    cert = certified_steps(res, u_acc=DOUBLE.u)
    k = min(len(piv), res.k_out)
    first_unc = next((i for i in range(k) if not cert[i]), k)
    agree = 0
    while agree < k and piv[agree] == res.perm[agree]:
        agree += 1
    return agree, first_unc


def test_fp64_round_is_the_scaled_copy():
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    A = gen_config("C1", 0)
    for scaling in ("none", "maxabs", "pow2"):
        h = MPID(to_dev(A), k_max=8, fp64=True)
        h.round_only("fp64", scaling)
        AL = h.get_AL().cpu().numpy()
        ref, _ = make_AL(A, "fp64", scaling)
        assert np.array_equal(AL.view(np.uint64), np.asarray(ref).view(np.uint64)), scaling
        h.close()


@pytest.mark.parametrize("case", ["C1", "C2", "fast", "medium"])
def test_fp64_parity_with_oracle(case):
    if case in ("C1", "C2"):
        A = gen_config(case, 0)
        if case == "C2":
            A = np.asfortranarray(A[:2048, :512])
        k = 32
    else:
        A, _ = gen_decay({"fast": 4.0, "medium": 2.0}[case], 1000, 1000, seed=0)
        k = 51
    lsq = case in ("C1", "C2")          # A(:, I) of the decay sets is too ill-conditioned for CholQR
    g = run64(A, k, mode="lsq" if lsq else "R")
    AL, _ = make_AL(A, "fp64", "none")
    res = qrcp_householder(AL, k, "fp64", nb=4)
    agree, first_unc = _prefix(g["piv"], res)
    assert agree >= first_unc, (agree, first_unc)
    scale = res.maxnorm0
    if agree == k:
        assert np.array_equal(g["perm"], res.perm)
        assert np.max(np.abs(g["R"] - res.R)) <= 1e-12 * scale
    else:
        assert np.max(np.abs(g["R"][:agree, :agree] - res.R[:agree, :agree])) <= 1e-12 * scale
    # the fp64 ID step on the GPU's I: P within 1e-10 of the oracle's, error within 1e-9
    P_ref = coeffs_lsq(A, g["piv"]) if lsq else coeffs_from_R(g["R"], g["perm"], k)
    assert np.linalg.norm(g["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    e_ref = id_error(A, g["piv"], g["P"])
    assert abs(g["err"][0] - e_ref[0]) <= 1e-9 * e_ref[0]


def test_fp64_matches_lapack_dgeqp3():
    """External pin: LAPACK's column-pivoted QR (dgeqp3) picks the same columns on the
    certified steps, and |diag R| agrees to 1e-12 relative."""
    A, _ = gen_decay(2.0, 600, 300, seed=3)
    k = 60
    g = run64(A, k)
    _, Rl, pl = sla.qr(A, mode="economic", pivoting=True)
    res = qrcp_householder(A, k, "fp64", nb=4)
    cert = certified_steps(res, u_acc=DOUBLE.u)
    first_unc = next((i for i in range(k) if not cert[i]), k)
    lap_agree = 0
    while lap_agree < k and g["piv"][lap_agree] == pl[lap_agree]:
        lap_agree += 1
    assert lap_agree >= first_unc, (lap_agree, first_unc)
    d_gpu = np.abs(np.diag(g["R"][:, :k]))[:lap_agree]
    d_lap = np.abs(np.diag(Rl))[:lap_agree]
    assert np.max(np.abs(d_gpu - d_lap) / d_lap) <= 1e-12
    assert np.all(np.diag(g["R"][:, :k]) >= 0)          # sign-normalised R_jj = |beta|


def test_fp64_R_mode_coefficients_and_fp32_export():
    A = np.asfortranarray(gen_config("C2", 0)[:1024, :256])
    k = 24
    g = run64(A, k, mode="R")
    P_ref = coeffs_from_R(g["R"], g["perm"], k)
    assert np.linalg.norm(g["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    assert np.array_equal(g["R32"], g["R"].astype(np.float32))


def test_fp64_nb_and_tolerance():
    """nb changes only when the formed block is written back (exact in fp64): pivots equal
    for nb = 1, 2, 8; the tolerance stop matches the oracle's k_eps (reading R8)."""
    A = np.asfortranarray(gen_config("C2", 0)[:2048, :384])
    ref = run64(A, 40, nb=4)
    for nb in (1, 2, 8):
        g = run64(A, 40, nb=nb)
        assert np.array_equal(g["piv"], ref["piv"]), nb
        assert np.max(np.abs(g["R"] - ref["R"])) <= 1e-13 * np.max(np.abs(ref["R"]))
    eps = 1e-3
    g = run64(A, 200, eps=eps)
    res = qrcp_householder(A, 200, "fp64", nb=4, eps=eps)
    assert abs(g["k"] - res.k_out) <= 1, (g["k"], res.k_out)


def test_fp64_column_split_matches_oracle():
    """n > 1024: the fp64 pass splits the columns over two CTA columns (and re-stores)."""
    rng = np.random.default_rng(11)
    m, n, k = 1536, 1100, 20
    A = np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 300.0))
    g = run64(A, k, nb=4)
    res = qrcp_householder(A, k, "fp64", nb=4)
    agree, first_unc = _prefix(g["piv"], res)
    assert agree >= first_unc, (agree, first_unc)
    if agree == k:
        assert np.max(np.abs(g["R"] - res.R)) <= 1e-12 * res.maxnorm0
