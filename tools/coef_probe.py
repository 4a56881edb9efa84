"""Coefficient-stage probe on C4: t_coef_ms and the LSQ path after each pivoting variant,
and the coefficient stage repeated on the same skeleton (no QRCP in between).
    python tools/coef_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2012_00706_b200 import mpid  # noqa: E402
from tools.bench_configs import device_matrix  # noqa: E402

At, spec = device_matrix("C4")
n, m = At.shape
for formation in ("auto", "gram", "auto"):
    h = mpid.MPID(At, k_max=100, m_global=m)
    for rep in range(3):
        h.qrcp("fp16", "pow2", k=100, formation=formation)
        h.coeffs("lsq")
        s1 = h.stats()
        h.coeffs("lsq")
        s2 = h.stats()
        print(formation, rep, "coef after qrcp %.2f ms (path %d), repeated %.2f ms (path %d)" %
              (s1["t_coef_ms"], s1["lsq_path"], s2["t_coef_ms"], s2["lsq_path"]), flush=True)
    h.close()
