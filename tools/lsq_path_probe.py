import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m, device="cuda")
h = mpid.MPID(A, k_max=100)
for form in ("ffma", "gram", "sketch", "ffma"):
    for rep in range(3):
        q = h.qrcp("fp16", "pow2", k=100, formation=form)
        h.coeffs("lsq"); e = h.error()
        st = h.stats()
    print(form, st["lsq_path"], round(st["t_coef_ms"], 2), e[1])
