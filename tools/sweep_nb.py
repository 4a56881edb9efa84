"""Sweep the store interval nb on the C4 workload: QRCP time and panel-pass bandwidth."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m, device="cuda")
k = 100
h = mpid.MPID(A, k_max=k)
m, n = spec.m, spec.n
for arg in sys.argv[1:] or ["fp16"]:
    fmt, form = (arg.split(":") + ["ffma"])[:2]
    nbs = (4, 8, 12, 16, 24, 32) if form == "tc" else (2, 3, 4, 5, 6, 8, 12, 16)
    for nb in nbs:
        ts = []
        for rep in range(3):
            q = h.qrcp(fmt, "pow2" if fmt == "fp16" else "none", k=k, nb=nb, profile=True, formation=form)
            st = h.stats()
            ts.append((st["t_qrcp_ms"], st["t_pass_ms"]))
        tq, tp = min(ts)
        s = 2 if fmt == "fp16" else 4
        byt = sum((m - j) * (n - j) * s * (2 if (j > 0 and j % nb == 0) else 1) for j in range(k))
        print(f"{fmt} {form} nb={nb:2d} qrcp {tq:7.2f} ms  pass {tp:7.2f} ms  {byt / tp / 1e6:7.0f} GB/s  read-only-equiv {sum((m-j)*(n-j)*s for j in range(k))/tp/1e6:7.0f} GB/s", flush=True)
