"""Debug: GPU vs oracle on a wide matrix (n > 1024 -> two column splits in the pass)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.generators import haar
from oracle.qrcp import make_AL, qrcp_householder
from tests.gpu_helpers import run_gpu, prefix_match
m, n, r = int(os.environ.get("M", "4096")), int(os.environ.get("N", "2048")), 300
rng = np.random.default_rng(5)
U = haar(rng, m, r); V = haar(rng, n, r)
A = np.asfortranarray((U * np.exp(-np.arange(1, r + 1) / 30.0)) @ V.T)
A += 1e-6 * np.linalg.norm(A) / np.sqrt(m * n) * rng.standard_normal((m, n))
k = int(os.environ.get("K", "64"))
for fmt in ("fp32", "fp16"):
    sc = "none" if fmt == "fp32" else "pow2"
    out = run_gpu(A, fmt, sc, k, nb=4)
    AL, s = make_AL(A, fmt, sc)
    res = qrcp_householder(AL, k, fmt, nb=4)
    agree, fu = prefix_match(out["piv"], res)
    nAL = np.linalg.norm(AL)
    print(fmt, "agree", agree, "first_unc", fu, "gpu resid_est", out["stats"]["resid_est"] / out["stats"]["normAL_fro"],
          "oracle resid", res.resid[k] / nAL, flush=True)
    print("  first R rows diff", [float(np.abs(out["R"][i, i:i + 50] - res.R[i, i:i + 50]).max()) for i in range(min(agree, 6))])
