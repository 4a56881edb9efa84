"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Acceptance (BASELINE.json north_star):
  * A_L bit-identical to the oracle's fl_L(s A_D);
  * first pivot = max-norm column of A_L;
  * pivots: ordered prefix equal up to the first uncertified oracle step; the
    whole set equal on gapped (planted) inputs;
  * relative Frobenius error within 5 % of the oracle's (same fmt, nb, LSQ);
  * P within 1e-10 relative of the oracle's LSQ P computed from the GPU's I;
  * R mode: P within 1e-10 of the oracle's R11^{-1} R12 fed the GPU's R.
"""
import math

import numpy as np
import pytest

from oracle.id import coeffs_from_R, coeffs_lsq, id_error
from oracle.qrcp import make_AL, qrcp_householder
from oracle.rounding import round_to
from synth import gen_config, gen_exact_rank, gen_planted
from oracle.fast import qrcp_c
from tests.gpu_helpers import C_TIE, oracle_qrcp, prefix_match, run_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2012_00706_b200 import mpid
    mpid.lib()


_CACHE = {}


def cfg(name, seed=0):
    key = (name, seed)
    if key not in _CACHE:
        _CACHE[key] = gen_config(name, seed)
    return _CACHE[key]


def _al_bits(AL, fmt):
    return AL.astype(np.float16).view(np.uint16) if fmt == "fp16" else AL.astype(np.float32).view(np.uint32)


@pytest.mark.parametrize("name,fmt,scaling", [("C1", "fp16", "pow2"), ("C1", "fp32", "none"),
                                              ("C2", "fp16", "maxabs"), ("C2", "fp32", "none"),
                                              ("C2", "fp16", "pow2")])
def test_AL_bit_identical(name, fmt, scaling):
    from paper_2012_00706_b200.mpid import MPID
    A = cfg(name)
    h = MPID(to_dev(A), k_max=8)
    h.round_only(fmt, scaling)
    g = h.get_AL().cpu().numpy()
    AL, s = make_AL(A, fmt, scaling)
    assert h.stats()["scale"] == s
    assert np.array_equal(_al_bits(g.astype(np.float64), fmt), _al_bits(AL, fmt))


def test_AL_near_ties_and_specials():
    """cvt.rn.f16.f64 single rounding on targeted near-ties (reading R1, A32), subnormals."""
    from paper_2012_00706_b200.mpid import MPID
    vals = [1 + 2.0 ** -11 + 2.0 ** -40, 1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 2.0 ** -25,
            2.0 ** -25 * (1 + 2.0 ** -30), 3 * 2.0 ** -26, 6.1e-5, 65504.0, -0.1, 0.1,
            2.0 ** -24, 1.5 * 2.0 ** -24, 5e-324, 0.0, -0.0, 65519.99]
    A = np.array(vals * 16, dtype=np.float64).reshape(64, 4, order="F")
    h = MPID(to_dev(A), k_max=1)
    for fmt in ("fp16", "fp32"):
        h.round_only(fmt, "none")
        g = h.get_AL().cpu().numpy().astype(np.float64)
        ref = round_to(A, fmt).reshape(A.shape)
        assert np.array_equal(_al_bits(g, fmt), _al_bits(ref, fmt)), fmt


def test_overflow_status():
    from paper_2012_00706_b200.mpid import MPID, IDError
    A = np.ones((64, 8))
    A[5, 3] = 1e6
    h = MPID(to_dev(A), k_max=2)
    with pytest.raises(IDError) as e:
        h.qrcp("fp16", "none", k=2)
    assert e.value.name == "OVERFLOW"


def test_underflow_status():
    A = np.full((40, 6), 1e-20)
    out = run_gpu(A, "fp16", "none", 1, allow_underflow=True)
    assert out["status"] == 4 and out["k"] == 0


def _compare(A, fmt, scaling, k, nb, min_prefix_frac=0.0, eps=0.0, key=None, formation="ffma"):
    """GPU run vs two oracles on the same A_L: the formation's own model (FFMA pass: the
    one-rounding update + 8-row fp32 chains, "kernel"; tcgen05 pass: the D-OTF block
    rounded once, fp64 row-order sums, "tc") and the independent paper model (per-op RNE
    update, fp64 row-order sums; oracle/cqrcp.c).  Pivots: ordered prefix up to the first
    step either oracle does not certify (reading R10, c_tie calibrated); error within 5 %
    of both; P within 1e-10 of the oracle's LSQ from the GPU's I; the GPU's error equal to
    the oracle's evaluation of the GPU's (I, P) to 1e-9."""
    out = run_gpu(A, fmt, scaling, k, nb=nb, eps=eps, formation=formation)
    AL, s = make_AL(A, fmt, scaling)
    oform = "tc" if formation == "tc" else "fma"
    r = (oracle_qrcp(key, A, fmt, scaling, k, nb, eps, formation=oform) if key
         else qrcp_householder(AL, k, fmt, nb=nb, eps=eps, formation=oform))
    rp = qrcp_c(AL, k, fmt, nb=nb, eps=eps, model="paper")
    assert out["piv"][0] == int(np.argmax(np.linalg.norm(AL, axis=0)))
    for ref, own in ((r, True), (rp, False)):
        agree, first_unc = prefix_match(out["piv"], ref, c_tie=C_TIE)
        assert agree >= first_unc, (agree, first_unc, out["piv"][:10], ref.perm[:10])
        # error parity (same fmt, nb, LSQ mode): GPU error vs oracle pipeline error — within
        # 5 % of the formation's own model always; of the paper model when the comparison
        # covers every pivot (with a store after every step, nb = 1, two faithful fp16
        # models part at the uncertified steps and their errors differ by up to ~15 %,
        # SURVEY App. A)
        err_or = id_error(A, ref.I, coeffs_lsq(A, ref.I))[1]
        err_gpu = out["err"][1]
        tol = 0.05 if (own or first_unc >= k or nb > 1) else 0.20
        assert abs(err_gpu - err_or) <= tol * err_or, (err_gpu, err_or, own)
    agree, first_unc = prefix_match(out["piv"], r, c_tie=C_TIE)
    # P parity given the same I: oracle LSQ from the GPU's I
    I = out["piv"]
    P_ref = coeffs_lsq(A, I)
    relP = np.linalg.norm(out["P"] - P_ref) / np.linalg.norm(P_ref)
    assert relP <= 1e-10, relP
    assert np.array_equal(out["P"][:, I], np.eye(len(I)))
    # error of the GPU's own (I, P) recomputed by the oracle
    e_re = id_error(A, I, out["P"])
    assert abs(e_re[1] - out["err"][1]) <= 1e-9 * max(e_re[1], 1e-300) + 1e-14
    return out, r, agree, first_unc


@pytest.mark.parametrize("fmt,scaling,nb", [("fp16", "pow2", 4), ("fp32", "none", 4), ("fp16", "pow2", 1),
                                            ("fp16", "pow2", 16), ("fp32", "none", 32 // 2)])
def test_C1_parity(fmt, scaling, nb):
    _compare(cfg("C1"), fmt, scaling, 32, nb)


@pytest.mark.parametrize("k,fmt,scaling", [(128, "fp32", "none"), (64, "fp32", "none"), (16, "fp32", "none"),
                                           (128, "fp16", "maxabs"), (64, "fp16", "maxabs"),
                                           (16, "fp16", "maxabs")])
def test_C2_parity(k, fmt, scaling):
    _compare(cfg("C2"), fmt, scaling, k, 4, key="C2")


@pytest.mark.parametrize("fmt,nb", [("fp16", 4), ("fp32", 8), ("fp16", 1)])
def test_planted_pivot_set(fmt, nb):
    A, skel, C = gen_planted(4096, 512, 64, rho=1.05, eta=1e-9, seed=3)
    out, r, agree, fu = _compare(A, fmt, "pow2" if fmt == "fp16" else "none", 64, nb)
    assert sorted(out["piv"]) == sorted(skel)
    assert np.array_equal(out["piv"], skel)


# ---- the tcgen05 pass (R14; the default for fp16 with range scaling): S^T I +
# (-F) V^T in hi / lo fp16 pairs, fp32 accumulation in TMEM ----------------------------
@pytest.mark.parametrize("nb", [4, 8, 16, 32])
def test_C1_parity_tcgen05(nb):
    out, r, agree, fu = _compare(cfg("C1"), "fp16", "pow2", 32, nb, formation="tc")
    assert out["stats"]["formation"] == 2 and out["stats"]["nb"] == nb


@pytest.mark.parametrize("k", [128, 64, 16])
def test_C2_parity_tcgen05(k):
    _compare(cfg("C2"), "fp16", "maxabs", k, 16, key="C2tc", formation="tc")


@pytest.mark.parametrize("nb", [16, 4])
def test_planted_pivot_set_tcgen05(nb):
    A, skel, C = gen_planted(4096, 512, 64, rho=1.05, eta=1e-9, seed=3)
    out, r, agree, fu = _compare(A, "fp16", "pow2", 64, nb, formation="tc")
    assert np.array_equal(out["piv"], skel)


def test_tcgen05_R_close_to_oracle():
    """R rows agree with the oracle's D-OTF model (the exact block rounded once) to the
    accuracy of the hi / lo fp16 product and the fp32 chains (<= 1e-5 max ||a_i||)."""
    A = cfg("C1")
    out = run_gpu(A, "fp16", "pow2", 32, nb=16, formation="tc")
    AL, _ = make_AL(A, "fp16", "pow2")
    r = qrcp_householder(AL, 32, "fp16", nb=16, formation="tc")
    assert np.array_equal(out["piv"], r.perm[:32])
    assert np.abs(out["R"][:, :32] - r.R[:, :32]).max() <= 1e-5 * r.maxnorm0


@pytest.mark.parametrize("m,n,k,nb", [(1000, 77, 20, 16), (4099, 290, 70, 8), (65536, 300, 40, 16),
                                      (20000, 2048, 24, 16), (3000, 1030, 33, 4), (256, 129, 32, 32),
                                      (40, 10, 10, 16)])
def test_tcgen05_ragged_and_wide_shapes(m, n, k, nb):
    """Ragged row blocks (m % 128 != 0), ragged column tiles (n - j % 128 != 0), one to
    sixteen column tiles (two epilogue groups, up to 8 tiles each), many row blocks per
    CTA (the smem ring, the accumulator ring and the V / u double buffers wrap), store
    steps every nb, against the oracle's tc model and the paper model."""
    rng = np.random.default_rng(m + n + k)
    A = np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 9.0)[None, :])
    _compare(A, "fp16", "pow2", k, nb, formation="tc")


def test_tcgen05_tolerance_rank():
    A = np.asfortranarray(gen_config("C2", 1)[:, :512])
    out = run_gpu(A, "fp16", "maxabs", 200, nb=16, eps=1e-2, formation="tc")
    AL, _ = make_AL(A, "fp16", "maxabs")
    r = qrcp_householder(AL, 200, "fp16", nb=16, eps=1e-2, formation="tc")
    assert abs(out["k"] - r.k_out) <= 1
    if out["k"] != r.k_out:
        kk = min(out["k"], r.k_out)
        assert abs(r.resid[kk] - 1e-2 * r.normAL) <= 1e-3 * r.normAL


@pytest.mark.parametrize("n,fmt,nb", [(1030, "fp32", 2), (1030, "fp16", 4), (2048, "fp32", 4)])
def test_column_split_store_steps_bit_identical(n, fmt, nb):
    """n > 1024: the pass splits the columns over two CTAs; on store steps no lane may
    write another column's chunk (regression: invalid lanes aliased a CTA's first column)."""
    rng = np.random.default_rng(5)
    from synth.generators import haar
    U = haar(rng, 4096, 300)
    V = haar(rng, n, 300)
    A = np.asfortranarray((U * np.exp(-np.arange(1, 301) / 30.0)) @ V.T)
    sc = "pow2" if fmt == "fp16" else "none"
    out = run_gpu(A, fmt, sc, 40, nb=nb)
    AL, _ = make_AL(A, fmt, sc)
    r = qrcp_householder(AL, 40, fmt, nb=nb)
    assert np.array_equal(out["piv"], r.perm[:40])
    assert np.array_equal(out["perm"], r.perm)
    assert np.array_equal(out["R"], r.R)                 # same operation order: bit-identical


def test_exact_rank_zero_error():
    A = gen_exact_rank(2000, 300, 24, seed=5)
    out = run_gpu(A, "fp32", "none", 24)
    assert out["err"][1] <= 1e-12


def test_R_mode_trsm_parity():
    """R mode: the GPU's fp64 triangular solve fed the GPU's R vs the oracle's solve of the same R."""
    A = cfg("C1")
    for fmt, sc in (("fp16", "pow2"), ("fp32", "none")):
        out = run_gpu(A, fmt, sc, 32, mode="R")
        Rg, perm = out["R"], out["perm"]
        assert np.array_equal(perm[:32], out["piv"])
        P_ref = coeffs_from_R(Rg, perm, 32)
        relP = np.linalg.norm(out["P"] - P_ref) / np.linalg.norm(P_ref)
        assert relP <= 1e-10, relP
        assert np.all(np.diag(Rg[:, :32]) >= 0)


def test_R_close_to_oracle_when_pivots_agree():
    A = cfg("C1")
    out = run_gpu(A, "fp32", "none", 32, nb=4)
    AL, _ = make_AL(A, "fp32", "none")
    r = qrcp_householder(AL, 32, "fp32", nb=4)
    if np.array_equal(out["piv"], r.perm[:32]):
        # R rows agree to fp32 accumulation level relative to ||A_L||
        assert np.abs(out["R"][:, :32] - r.R[:, :32]).max() <= 1e-5 * r.maxnorm0


@pytest.mark.parametrize("m,n,k", [(1000, 77, 20), (20, 10, 10), (300, 33, 33), (513, 64, 1),
                                   (257, 1, 1), (4099, 290, 70)])
def test_ragged_and_edge_shapes(m, n, k):
    rng = np.random.default_rng(m + n + k)
    A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 7.0)[None, :]
    A = np.asfortranarray(A)
    for fmt, sc in (("fp32", "none"), ("fp16", "pow2")):
        out = run_gpu(A, fmt, sc, k, nb=4)
        AL, s = make_AL(A, fmt, sc)
        r = qrcp_householder(AL, k, fmt, nb=4)
        agree, fu = prefix_match(out["piv"], r)
        assert agree >= fu
        assert out["k"] == k
        I = out["piv"]
        P_ref = coeffs_lsq(A, I)
        assert np.linalg.norm(out["P"] - P_ref) <= 1e-10 * max(np.linalg.norm(P_ref), 1e-300)
        e = id_error(A, I, out["P"])                 # the fused error on the GPU's own P
        assert abs(out["err"][0] - e[0]) <= 1e-9 * e[0] + 1e-300


# The fused error kernels (Remark 2) and the LSQ refit's TN GEMMs: the warp-specialised one needs an even row
# count (odd m takes the register-staged kernel); k spans < 1 k-stage, a ragged last stage
# (k % 8 != 0), whole stages; m x n spans one tile, ragged tiles and > 148 tiles (several
# tiles per CTA, i.e. the ring and the A_D buffer wrap across tiles).
@pytest.mark.parametrize("m,n,k", [(130, 50, 1), (1024, 140, 3), (1023, 140, 3), (2000, 300, 8),
                                   (4098, 261, 13), (4097, 261, 13), (40000, 400, 100), (39999, 257, 64),
                                   (6000, 200, 70), (8192, 300, 86), (12000, 260, 120),
                                   (5000, 180, 52)])
def test_error_kernel_shapes(m, n, k):
    rng = np.random.default_rng(m * 7 + n + k)
    A = np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 9.0)[None, :])
    out = run_gpu(A, "fp32", "none", k, nb=4)
    I = out["piv"]
    # the LSQ products (Q1^T Q1, Q1^T A_J): even m takes the mbarrier-pipelined TN GEMM
    # (8-row M tiles when that pads less: k = 52 / 70 / 86 / 100 / 120 -> MR = 7 / 9 / 11 / 13 / 15), odd m the register-staged one
    P_ref = coeffs_lsq(A, I)
    assert np.linalg.norm(out["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    e = id_error(A, I, out["P"])
    assert abs(out["err"][0] - e[0]) <= 1e-9 * e[0]
    assert abs(out["err"][1] - e[1]) <= 1e-9 * e[1]


def test_tolerance_rank_matches_oracle():
    A = gen_config("C2", 1)[:, :512]
    A = np.asfortranarray(A)
    out = run_gpu(A, "fp32", "none", 200, eps=1e-3)
    AL, _ = make_AL(A, "fp32", "none")
    r = qrcp_householder(AL, 200, "fp32", nb=4, eps=1e-3)
    assert abs(out["k"] - r.k_out) <= 1
    resid = r.resid
    if out["k"] != r.k_out:  # only when the crossing step is within rounding of the threshold
        kk = min(out["k"], r.k_out)
        assert abs(resid[kk] - 1e-3 * r.normAL) <= 1e-4 * r.normAL


def test_tolerance_rank_fp16_matches_oracle():
    """fp16 storage, re-store every nb = 4 steps: the storage noise is part of the
    residual both sides measure (reading R8), so k_eps is compared with the oracle."""
    A = np.asfortranarray(gen_config("C2", 1)[:, :512])
    out = run_gpu(A, "fp16", "maxabs", 200, eps=1e-2)
    AL, _ = make_AL(A, "fp16", "maxabs")
    r = qrcp_householder(AL, 200, "fp16", nb=4, eps=1e-2)
    assert abs(out["k"] - r.k_out) <= 1
    if out["k"] != r.k_out:
        kk = min(out["k"], r.k_out)
        assert abs(r.resid[kk] - 1e-2 * r.normAL) <= 1e-3 * r.normAL


def test_graph_and_stream_paths_identical_and_deterministic():
    A = cfg("C1")
    a = run_gpu(A, "fp16", "pow2", 32, use_graph=True)
    b = run_gpu(A, "fp16", "pow2", 32, use_graph=False)
    c = run_gpu(A, "fp16", "pow2", 32, use_graph=True)
    assert np.array_equal(a["piv"], b["piv"]) and np.array_equal(a["piv"], c["piv"])
    assert np.array_equal(a["P"], b["P"]) and np.array_equal(a["P"], c["P"])
    assert a["err"] == b["err"] == c["err"]


def test_host_buffer_path_equals_device_path():
    A = cfg("C1")
    a = run_gpu(A, "fp16", "pow2", 32)
    b = run_gpu(A, "fp16", "pow2", 32, host=True)
    assert np.array_equal(a["piv"], b["piv"]) and np.array_equal(a["P"], b["P"])


# ---- NEXT-1 / NEXT-2: the low-precision skeleton and the paper's 2-norm metric ----------
@pytest.mark.parametrize("fmt,scaling", [("fp16", "pow2"), ("fp32", "none")])
def test_error_variants_and_spectral_norm(fmt, scaling):
    from oracle.id import id_error_skeleton, low_skeleton, spectral_error
    from oracle.qrcp import scale_factor
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    A = np.asfortranarray(gen_config("C2", 0)[:, :400])
    k = 24
    h = MPID(to_dev(A), k_max=k)
    q = h.qrcp(fmt, scaling, k=k)
    I = q.piv
    for mode in ("lsq", "R"):
        P = h.coeffs(mode).cpu().numpy()
        s = scale_factor(A, scaling)
        XL = low_skeleton(A, I, fmt, s)
        # Frobenius, both skeletons, against the oracle given the GPU's (I, P)
        ef = h.error_ex("AD", "fro")
        assert abs(ef[0] - id_error_skeleton(A, A[:, I], P)[0]) <= 1e-9 * ef[0]
        el = h.error_ex("AL", "fro")
        ref = id_error_skeleton(A, XL, P)
        assert abs(el[0] - ref[0]) <= 1e-9 * ref[0] and abs(el[1] - ref[1]) <= 1e-9 * ref[1]
        # 2-norm by power iteration: converges from below to LAPACK's value
        for sk, X in (("AD", A[:, I]), ("AL", XL)):
            e2 = h.error_ex(sk, 2, iters=200)
            ex = spectral_error(A, X, P)
            assert e2[0] <= ex[0] * (1 + 1e-9) and e2[0] >= ex[0] * (1 - 1e-3), (sk, e2, ex)
            assert abs(e2[1] - ex[1]) <= 1e-3 * ex[1]
    h.close()


@pytest.mark.parametrize("m,n,k", [(8192, 700, 300), (4096, 300, 140)])
def test_lsq_large_k_blocked_cholesky(m, n, k):
    """k > 143: the Gram matrix no longer fits shared memory and the blocked
    left-looking Cholesky runs; P must still match the oracle's Householder LSQ."""
    rng = np.random.default_rng(m + k)
    A = np.asfortranarray(rng.standard_normal((m, n)) @ np.diag(np.exp(-np.arange(n) / 200.0)))
    out = run_gpu(A, "fp32", "none", k)
    P_ref = coeffs_lsq(A, out["piv"])
    assert np.linalg.norm(out["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)


def test_lsq_fallback_to_cholqr2():
    """When the fp16 R11 no longer preconditions A_I (true residuals far below the fp16
    noise), R2's diagonal spread exceeds 1e3 and the call reruns as CholQR2
    (id_stats.lsq_path = 2); the well-conditioned default stays on path 1."""
    from paper_2012_00706_b200.mpid import MPID
    from tests.gpu_helpers import to_dev
    rng = np.random.default_rng(21)
    m, n, r = 4096, 120, 40
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) + 3e-7 * rng.standard_normal((m, n))
    A = np.asfortranarray(A)
    h = MPID(to_dev(A), k_max=48)
    q = h.qrcp("fp16", "pow2", k=48)
    P = h.coeffs("lsq").cpu().numpy()
    assert h.stats()["lsq_path"] == 2
    P_ref = coeffs_lsq(A, q.piv)
    assert np.linalg.norm(P - P_ref) <= 1e-7 * np.linalg.norm(P_ref)
    h.close()
    B = cfg("C1")
    h = MPID(to_dev(B), k_max=24)
    h.qrcp("fp16", "pow2", k=24)
    h.coeffs("lsq")
    assert h.stats()["lsq_path"] == 1
    h.close()


@pytest.mark.parametrize("fmt", ["fp16", "fp32", "fp64"])
def test_degenerate_inputs(fmt):
    """Edge cases: a NaN or Inf in A_D -> OVERFLOW; an all-zero matrix -> UNDERFLOW at
    step 0 (no pivot); k > min(m, n) -> DIM; a single column; fewer rows than a group."""
    from paper_2012_00706_b200.mpid import MPID, IDError
    scaling = "pow2" if fmt == "fp16" else "none"
    for bad in (np.nan, np.inf):
        A = np.ones((64, 8))
        A[7, 2] = bad
        h = MPID(to_dev(A), k_max=2, fp64=fmt == "fp64")
        with pytest.raises(IDError) as e:
            h.qrcp(fmt, scaling, k=2)
        assert e.value.name == "OVERFLOW"
        h.close()
    h = MPID(to_dev(np.zeros((64, 8))), k_max=3, fp64=fmt == "fp64")
    q = h.qrcp(fmt, scaling, k=3, allow_underflow=True)
    assert q.status == 4 and q.k == 0
    h.close()
    h = MPID(to_dev(np.ones((16, 4))), k_max=4, fp64=fmt == "fp64")
    with pytest.raises(IDError) as e:
        h.qrcp(fmt, scaling, k=5)
    assert e.value.name == "DIM"
    h.close()
    rng = np.random.default_rng(1)
    for (m, n, k) in [(100, 1, 1), (5, 3, 3), (7, 20, 4)]:
        A = rng.standard_normal((m, n))
        out = run_gpu(A, fmt, scaling, k, nb=1)
        assert out["k"] == k
        P_ref = coeffs_lsq(A, out["piv"])
        assert np.linalg.norm(out["P"] - P_ref) <= 1e-10 * max(1.0, np.linalg.norm(P_ref))
