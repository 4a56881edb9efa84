"""Debug: R rows of the first steps, GPU vs oracle, n > 1024."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.generators import haar
from oracle.qrcp import make_AL, qrcp_householder
from tests.gpu_helpers import run_gpu
m, n, r = 4096, int(os.environ.get("N", "1030")), 300
rng = np.random.default_rng(5)
U = haar(rng, m, r); V = haar(rng, n, r)
A = np.asfortranarray((U * np.exp(-np.arange(1, r + 1) / 30.0)) @ V.T)
for k in (1, 2, 3):
    out = run_gpu(A, "fp32", "none", k, nb=4)
    AL, s = make_AL(A, "fp32", "none")
    res = qrcp_householder(AL, k, "fp32", nb=4)
    perm_g = out["perm"]
    print("k", k, "piv", out["piv"], res.perm[:k], "perm equal", np.array_equal(perm_g, res.perm))
    d = np.abs(out["R"] - res.R)
    bad = np.argwhere(d > 1e-6 * np.abs(res.R).max())
    print("  R maxdiff", d.max(), "nbad", len(bad), "bad cols", bad[:10].tolist())
