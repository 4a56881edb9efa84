"""Profiling driver for the tcgen05 pass: C4 rows, fp16, formation=tc, few steps."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=1 << 21)
ap.add_argument("--k", type=int, default=12)
ap.add_argument("--nb", type=int, default=16)
ap.add_argument("--form", default="tc")
a = ap.parse_args()
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, a.rows, device="cuda")
h = mpid.MPID(A, k_max=a.k, m_global=a.rows)
q = h.qrcp("fp16", "pow2", k=a.k, nb=a.nb, use_graph=False, formation=a.form)
torch.cuda.synchronize()
print(q.k, h.stats())
