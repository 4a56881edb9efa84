"""The one-launch cooperative QRCP (formation 6, k_qrcp_coop.cu; include/mpid.h) against the
oracle's paper model (oracle/cqrcp.c, update = rne, fp64 row-order sums; R4b/R5):
the kernel keeps the whole matrix in the shared memory of all SMs and forms each column's
fp64 sums per row slab, adding the slab partials in slab order — an association of the same
fp64 sum, so pivots must agree on every step the oracle certifies (reading R10) and R to
working precision.  Shapes: C2 (4096 x 1024), ragged m (the last slab shorter than the
others), k = 16 / 64 / 128, fp16 (store interval 16) and fp32, a tolerance stop, and C2's
acceptance checks (P, error) on top."""
import numpy as np
import pytest

from oracle.fast import qrcp_c
from oracle.id import coeffs_lsq, id_error
from oracle.qrcp import make_AL
from synth import gen_config

pytestmark = pytest.mark.gpu


def _run(A, fmt, sc, k, eps=0.0, formation="coop"):
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    h = MPID(to_dev(A), k_max=k)
    q = h.qrcp(fmt, sc, k=k, eps=eps, formation=formation)
    st = h.stats()
    out = {"k": q.k, "piv": q.piv.copy(), "stats": st, "R": h.get_R().cpu().numpy().astype(np.float64),
           "perm": h.get_perm()}
    out["P"] = h.coeffs("lsq").cpu().numpy()
    out["err"] = h.error()
    h.close()
    return out


def _compare(A, out, fmt, sc, k, eps=0.0):
    from tests.gpu_helpers import C_TIE, prefix_match
    AL, _ = make_AL(A, fmt, sc)
    r = qrcp_c(AL, k, fmt, nb=out["stats"]["nb"], eps=eps, model="paper")
    agree, fu = prefix_match(out["piv"], r, c_tie=C_TIE)
    assert agree >= fu, (agree, fu)
    if agree == r.k_out == out["k"]:
        scale = float(np.max(np.sqrt(np.sum(np.asarray(AL, dtype=np.float64) ** 2, axis=0))))
        assert np.max(np.abs(out["R"][:k] - r.R[:k])) <= 1e-5 * scale
    P_ref = coeffs_lsq(A, out["piv"])
    assert np.linalg.norm(out["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    e = id_error(A, out["piv"], out["P"])
    assert abs(out["err"][0] - e[0]) <= 1e-9 * e[0]
    return r, agree, fu


@pytest.mark.parametrize("k", [16, 64, 128])
@pytest.mark.parametrize("fmt,sc", [("fp16", "maxabs"), ("fp32", "none")])
def test_coop_C2(k, fmt, sc):
    A = gen_config("C2", 0)
    out = _run(A, fmt, sc, k)
    assert out["stats"]["formation"] == 6 and out["k"] == k
    _compare(A, out, fmt, sc, k)


def test_coop_refused_when_it_does_not_fit():
    """A shard larger than all SMs' shared memory: ID_ERR_ARG, not a silent fallback."""
    from paper_2012_00706_b200.mpid import MPID, IDError
    from tests.gpu_helpers import to_dev
    A = np.asfortranarray(np.tile(gen_config("C2", 1), (4, 1)))    # 16384 x 1024: 64 MB in fp32
    h = MPID(to_dev(A), k_max=8)
    with pytest.raises(IDError):
        h.qrcp("fp16", "maxabs", k=8, formation="coop")
    h.close()


@pytest.mark.parametrize("m,n", [(4001, 1000), (1500, 777), (6000, 512)])
def test_coop_ragged(m, n):
    A = np.asfortranarray(gen_config("C2", 2)[:m, :n])
    out = _run(A, "fp16", "maxabs", 40)
    _compare(A, out, "fp16", "maxabs", 40)


def test_coop_tolerance_stop():
    A = gen_config("C2", 3)
    out = _run(A, "fp32", "none", 200, eps=1e-3)
    r, agree, fu = _compare(A, out, "fp32", "none", 200, eps=1e-3)
    assert abs(out["k"] - r.k_out) <= 1
