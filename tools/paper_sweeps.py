"""NEXT-3: the paper's §3 experiments on the GPU path.

Datasets: Slow / Medium / Fast decay, A = U diag(i^-p) V^T, 1000 x 1000, p = 1, 2, 4
(Table 3; synth.gen_decay).  For each low precision (fp32 = the paper's
single, fp16 = its simulated half) and each target rank of the rank sweep
k = 5, 7, ..., 51, and for the column sweep n = 100, 200, ..., 1000 at
m = 1000, k = 20, one mixed-precision ID through the C ABI with the
paper's coefficients P_L = R11^-1 R12 from the low-precision R (Algorithm 2 lines 5-6),
and the relative 2-norm errors against the ground truth A_D of both variants of
P:196: the mixed ID (skeleton A_D(:, I)) and the low-precision ID (skeleton A_L(:, I)).
Also recorded: sigma_{k+1} and the Lemma 2.1 envelope sqrt(1 + k(n-k)) sigma_{k+1}
(P:190-191).  The double ID Â_D = A_D(:, I_D) P_D (Algorithm 1) runs on the GPU too
(ID_FP64), and every low-precision point records its §3.1 distance to it,
||Â - Â_D||_2 / ||Â_D||_2; tests/test_gpu_paper_experiments.py checks the paper's claims
against the oracle's double ID.

    python tools/paper_sweeps.py > profiles/r01_paper_sweeps.jsonl
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_00706_b200.mpid import IDError, MPID  # noqa: E402
from synth import gen_decay  # noqa: E402

DATASETS = {"slow": 1.0, "medium": 2.0, "fast": 4.0}


def run(A, fmt, k, scaling, double=None):
    """One ID through the C ABI; with `double` = (I_D, P_D) of the GPU's fp64 ID also the
    §3.1 distance ||Â - Â_D||_2 / ||Â_D||_2 (products on the host in fp64)."""
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    h = MPID(At, k_max=k, fp64=fmt == "fp64")
    out = {"k": k, "fmt": fmt, "scaling": scaling}
    try:
        q = h.qrcp(fmt, scaling, k=k, allow_underflow=True)
        out["k_out"] = q.k
        out["status"] = {0: "ok", 4: "underflow"}.get(q.status, q.status)
        if q.k == 0:
            return out
        P = h.coeffs("R").cpu().numpy()                     # P_L from the low-precision R
        out["I"], out["P"] = q.piv[:q.k].tolist(), P
        if double is not None:
            ID, PD = double
            AD_hat = A[:, ID] @ PD
            out["dist_to_double"] = float(np.linalg.norm(A[:, q.piv[:q.k]] @ P - AD_hat, 2) /
                                          np.linalg.norm(AD_hat, 2))
        out["rel2_mixed"] = h.error_ex("AD", 2, iters=250)[1]
        out["rel2_low"] = h.error_ex("AL", 2, iters=250)[1]
        out["relF_mixed"] = h.error_ex("AD", "fro")[1]
    except IDError as e:
        out["status"] = e.name
    finally:
        h.close()
    return out


def emit(r, **kw):
    r.pop("P", None)
    r.pop("I", None)
    r.update(kw)
    print(json.dumps(r), flush=True)


def main():
    for name, p in DATASETS.items():
        A, sigma = gen_decay(p, 1000, 1000, seed=0)
        dbl_rank, dbl_cols = {}, {}
        for k in range(5, 52, 2):                  # the double ID (GPU, ID_FP64) first
            r = run(A, "fp64", k, "none")
            dbl_rank[k] = (r["I"], r["P"])
            emit(r, sweep="rank", dataset=name, m=1000, n=1000, sigma_k1=float(sigma[k]),
                 lemma_bound=math.sqrt(1 + k * (1000 - k)) * float(sigma[k]))
        for n in range(100, 1001, 100):
            r = run(np.asfortranarray(A[:, :n]), "fp64", 20, "none")
            dbl_cols[n] = (r["I"], r["P"])
            emit(r, sweep="columns", dataset=name, m=1000, n=n)
        for fmt, scaling in (("fp32", "none"), ("fp16", "none"), ("fp16", "pow2")):
            for k in range(5, 52, 2):
                r = run(A, fmt, k, scaling, dbl_rank[k])
                emit(r, sweep="rank", dataset=name, m=1000, n=1000, sigma_k1=float(sigma[k]),
                     lemma_bound=math.sqrt(1 + k * (1000 - k)) * float(sigma[k]))
            for n in range(100, 1001, 100):
                r = run(np.asfortranarray(A[:, :n]), fmt, 20, scaling, dbl_cols[n])
                emit(r, sweep="columns", dataset=name, m=1000, n=n)


if __name__ == "__main__":
    main()
