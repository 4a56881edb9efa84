"""Generator checks (synth/): structure of the synthetic workloads (DESIGN.md input recipe)."""
import math

import numpy as np

from synth import (config_spec, counter_normal, fourier_params, gen_config, gen_fourier,
                   gen_planted, haar)


def test_haar_orthonormal():
    Q = haar(np.random.default_rng(0), 500, 120)
    assert np.linalg.norm(Q.T @ Q - np.eye(120)) <= 1e-12


def test_c1_spectrum_and_layout():
    A = gen_config("C1", seed=0)
    assert A.shape == (256, 128) and A.flags.f_contiguous
    s = np.linalg.svd(A, compute_uv=False)
    sig = 10.0 ** (-np.arange(128) / 8.0)
    big = sig > 1e-12
    assert np.allclose(s[big], sig[big], rtol=1e-9, atol=1e-15)


def test_counter_normal_shard_invariance_and_backends():
    full = counter_normal(4, 9, np.arange(1000), np.arange(5))
    part = counter_normal(4, 9, np.arange(600, 1000), np.arange(5))
    assert np.array_equal(full[:, 600:], part)
    t = counter_normal(4, 9, np.arange(1000), np.arange(5), device="cpu").numpy()
    assert np.allclose(full, t, rtol=0, atol=1e-14)
    assert abs(full.mean()) < 0.1 and abs(full.std() - 1) < 0.05


def test_fourier_closed_forms():
    fp = fourier_params(16, 24, 96, seed=5)
    A = gen_fourier(fp, 5, noise=False)
    # equal column norms sqrt(m/2 sum a^2) and ||A||_F^2 = (m/2) n sum a^2 (discrete orthogonality)
    cn = np.linalg.norm(A, axis=0)
    ref = math.sqrt(fp.m / 2 * np.sum(fp.amp ** 2))
    assert np.allclose(cn, ref, rtol=1e-9)
    assert abs(np.linalg.norm(A) ** 2 / fp.clean_fro2 - 1) < 1e-9
    assert np.linalg.matrix_rank(A) <= 2 * fp.L
    sh = gen_fourier(fp, 5, row0=1000, m_loc=500, noise=True)
    An = gen_fourier(fp, 5, noise=True)
    assert np.array_equal(sh, An[1000:1500])
    t = gen_fourier(fp, 5, device="cpu").numpy().T
    assert np.allclose(t, An, atol=1e-10)


def test_planted_structure():
    A, skel, C = gen_planted(128, 40, 8, rho=1.2, eta=0.0, seed=3)
    S = A[:, skel]
    J = np.setdiff1d(np.arange(40), skel)
    X, *_ = np.linalg.lstsq(S, A[:, J], rcond=None)
    assert np.linalg.norm(S @ X - A[:, J]) <= 1e-12 * np.linalg.norm(A)
    assert np.abs(C).max() <= 0.5 * math.sqrt(1 - 1.2 ** -2)


def test_config_specs():
    assert config_spec("C4").m == 128 ** 3 and config_spec("C5").n == 2048
    assert config_spec("C2").scaling["fp16"] == "maxabs"
