"""One ID of the C5 per-GPU shard (2^21 x 2048, k = 512, fp16) for profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C5")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m // 8, device="cuda")
h = mpid.MPID(A, k_max=512, m_global=spec.m // 8)
q = h.qrcp("fp16", "pow2", k=512, use_graph=False)
P = h.coeffs("lsq")
e = h.error()
torch.cuda.synchronize()
print(q.k, e, h.stats())
