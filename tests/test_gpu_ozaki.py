"""The int8 engine of the fp64 ID step (include/mpid.h id_set_fp64_engine; k_ozaki.cu;
DESIGN.md §5): G2 = Q1^T Q1, W = Q1^T A_D(:, J) and the error's A_D(:, I) T on the int8
tensor cores by the Ozaki scheme.  On one handle and one QRCP (so one skeleton I), the
coefficients and the error are computed with the DMMA engine and with the int8 engine and
compared with each other and with the oracle's fp64 LSQ (Householder QR of A_D(:, I),
P:178) and error (fsum of the fp64 residual, Remark 2 P:199-201).

Acceptance (north_star): P within 1e-10 relative of the oracle given the same I; the error
within 1e-9 relative of the oracle's on the same (I, P) inputs.  Shapes: ragged m (not a
multiple of the 32-row K-step or the 128-row tile), ragged J (not a multiple of the 32- and
64-column tiles), k across the K-step boundaries (1, 31, 32, 33, 100, 128), columns and
rows spread over 12 decades, exact zero rows and columns, and sign changes.
"""
import numpy as np
import pytest

from oracle.id import coeffs_lsq, id_error, id_error_blocked
from synth import gen_config
from synth.generators import fourier_params, gen_fourier

pytestmark = pytest.mark.gpu


def _both(At, A, k, fmt="fp32", scaling="none"):
    from paper_2012_00706_b200.mpid import MPID
    h = MPID(At, k_max=k)
    q = h.qrcp(fmt, scaling, k=k)
    out = {"piv": q.piv.copy(), "k": q.k}
    for eng in ("dmma", "int8"):
        h.set_fp64_engine(eng)
        out["P_" + eng] = h.coeffs("lsq").cpu().numpy()
        out["err_" + eng] = h.error()
        out["st_" + eng] = h.stats()
    h.close()
    return out


def _check(A, out, err_fn=id_error):
    I = out["piv"]
    assert out["st_int8"]["fp64_engine"] == 2 and out["st_int8"]["fp64_engine_err"] == 2
    assert out["st_dmma"]["fp64_engine"] == 1 and out["st_dmma"]["fp64_engine_err"] == 1
    P_ref = coeffs_lsq(A, I)
    nP = np.linalg.norm(P_ref)
    d_or = np.linalg.norm(out["P_int8"] - P_ref) / nP
    d_eng = np.linalg.norm(out["P_int8"] - out["P_dmma"]) / nP
    assert d_or <= 1e-10, f"int8 P vs oracle {d_or:.3e}"
    assert d_eng <= 1e-10, f"int8 P vs DMMA P {d_eng:.3e}"
    # the error of each engine's own P against the oracle's residual of that P
    for eng in ("dmma", "int8"):
        a_ref, r_ref = err_fn(A, I, out["P_" + eng])
        a, r = out["err_" + eng]
        assert abs(a - a_ref) <= 1e-9 * a_ref, f"{eng} error {a} vs oracle {a_ref}"
    return d_or, d_eng


@pytest.mark.parametrize("k", [1, 31, 32, 33, 100, 128])
def test_int8_engine_ragged_C2(k):
    """C2's generator cut to 4059 x 1019 rows / columns (ragged K-steps, row tiles, J tiles)."""
    from tests.gpu_helpers import to_dev
    A = np.asfortranarray(gen_config("C2", 0)[:4059, :1019])
    out = _both(to_dev(A), A, k)
    _check(A, out)


def test_int8_engine_wide_dynamic_range():
    """Columns scaled over 12 decades, rows over 6, a zero column and zero rows: the per-
    column (A_D, Q1, T) and per-row (A_I) exponents of the slicing."""
    from tests.gpu_helpers import to_dev
    rng = np.random.default_rng(7)
    m, n, k = 3001, 333, 40
    A = gen_config("C2", 3)[:m, :n].copy()
    A *= 10.0 ** rng.uniform(-6, 6, size=(1, n))
    A *= 10.0 ** rng.uniform(-3, 3, size=(m, 1))
    A[:, 17] = 0.0
    A[100:140, :] = 0.0
    A = np.asfortranarray(A)
    out = _both(to_dev(A), A, k, fmt="fp32", scaling="none")
    _check(A, out)


def test_int8_engine_on_the_C4_analogue():
    """The 32^3-row C4 analogue (k = 100): the int8 engine's P and error match the oracle and
    the DMMA engine, and are bitwise reproducible across handles."""
    import torch
    from paper_2012_00706_b200.mpid import MPID
    fp = fourier_params(32, 64, 1024, 0)
    At = gen_fourier(fp, 0, device="cuda")
    A = np.asfortranarray(At.cpu().numpy().T)
    h = MPID(At, k_max=100)
    h.set_fp64_engine("int8")
    q = h.qrcp("fp16", "pow2", k=100)
    P = h.coeffs("lsq").cpu().numpy()
    e = h.error()
    st = h.stats()
    h.close()
    assert st["fp64_engine"] == 2 and st["fp64_engine_err"] == 2
    out = _both(At, A, 100, fmt="fp16", scaling="pow2")
    assert np.array_equal(out["piv"], q.piv)
    assert np.array_equal(out["P_int8"], P) and out["err_int8"] == e   # deterministic
    _check(A, out, err_fn=id_error_blocked)
    del At
    torch.cuda.empty_cache()


def test_int8_engine_refused_where_it_does_not_apply():
    """k > 128 (the K of the error GEMM must fit one 128-row operand): ID_ERR_ARG."""
    from paper_2012_00706_b200.mpid import MPID, IDError
    from tests.gpu_helpers import to_dev
    A = np.asfortranarray(gen_config("C2", 0)[:2048, :512])
    h = MPID(to_dev(A), k_max=160)
    h.qrcp("fp32", "none", k=160)
    h.set_fp64_engine("int8")
    with pytest.raises(IDError):
        h.coeffs("lsq")
    h.set_fp64_engine("auto")
    h.coeffs("lsq")
    assert h.stats()["fp64_engine"] == 1
    h.close()


def test_auto_engine_choice():
    """Auto: the int8 engine from 32768 rows per shard with k <= 128, else DMMA."""
    import torch
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    A = np.asfortranarray(gen_config("C2", 0)[:4096, :256])
    h = MPID(to_dev(A), k_max=16)
    h.qrcp("fp32", "none", k=16)
    h.coeffs("lsq")
    h.error()
    st = h.stats()
    assert st["fp64_engine"] == 1 and st["fp64_engine_err"] == 1
    h.close()
    fp = fourier_params(32, 64, 1024, 0)
    At = gen_fourier(fp, 0, device="cuda")
    h = MPID(At, k_max=100)
    h.qrcp("fp16", "pow2", k=100)
    h.coeffs("lsq")
    h.error()
    st = h.stats()
    assert st["fp64_engine"] == 2 and st["fp64_engine_err"] == 2
    h.close()
    del At
    torch.cuda.empty_cache()


def test_engine_limits_fall_back_to_dmma():
    """n beyond 64 x SMs (the TN kernel's one-CTA-per-(row group, tile) grid): the automatic
    engine is DMMA, a forced int8 engine is refused, and P still matches the oracle."""
    import torch
    from paper_2012_00706_b200.mpid import MPID, IDError
    from tests.gpu_helpers import to_dev
    rng = np.random.default_rng(5)
    m, n, k = 32768, 9600, 16
    A = np.asfortranarray(rng.standard_normal((m, 40)) @ rng.standard_normal((40, n))
                          + 1e-3 * rng.standard_normal((m, n)))
    h = MPID(to_dev(A), k_max=k)
    q = h.qrcp("fp32", "none", k=k)
    P = h.coeffs("lsq").cpu().numpy()
    h.error()
    st = h.stats()
    assert st["fp64_engine"] == 1 and st["fp64_engine_err"] == 1
    h.set_fp64_engine("int8")
    with pytest.raises(IDError):
        h.coeffs("lsq")
    h.close()
    P_ref = coeffs_lsq(A, q.piv)
    assert np.linalg.norm(P - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    torch.cuda.empty_cache()
