"""Debug: first step whose R row differs (GPU vs oracle), n > 1024."""
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
k = int(os.environ.get("K", "48"))
for nb in (4, 1, 2):
    out = run_gpu(A, "fp32", "none", k, nb=nb)
    AL, s = make_AL(A, "fp32", "none")
    res = qrcp_householder(AL, k, "fp32", nb=nb)
    print("nb", nb, "piv equal", np.array_equal(out["piv"], res.perm[:k]), "perm equal", np.array_equal(out["perm"], res.perm))
    d = np.abs(out["R"] - res.R)
    rows = np.flatnonzero(d.max(axis=1) > 0)
    print("  first differing R row", rows[:5], "max", d.max())
    if len(rows):
        i = rows[0]
        cols = np.flatnonzero(d[i] > 0)
        print("  row", i, "cols", cols[:20], "ncols", len(cols), "n", n)
