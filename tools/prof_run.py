"""Small profiling driver: one C4-shaped ID (reduced rows) through the C ABI."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=1 << 19)
ap.add_argument("--k", type=int, default=24)
ap.add_argument("--fmt", default="fp16")
ap.add_argument("--nb", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--graph", type=int, default=1)
a = ap.parse_args()
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, a.rows, device="cuda")
h = mpid.MPID(A, k_max=a.k, m_global=a.rows)
for _ in range(a.reps):
    q = h.qrcp(a.fmt, "pow2" if a.fmt == "fp16" else "none", k=a.k, nb=a.nb, use_graph=bool(a.graph))
    P = h.coeffs("lsq")
    e = h.error()
torch.cuda.synchronize()
print(q.k, e, h.stats())
