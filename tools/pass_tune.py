"""QRCP time on C4 (fp16, k = 100) for a given store interval nb; run with
MPID_PASS_STAGE_KB=<kb> to vary the pass's stage size.  Min of 5 after a warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m, device="cuda")
h = mpid.MPID(A, k_max=100)
for nb in [int(x) for x in sys.argv[1:]] or [4]:
    ts = []
    for rep in range(6):
        q = h.qrcp("fp16", "pow2", k=100, nb=nb)
        if rep:
            ts.append(h.stats()["t_qrcp_ms"])
    print(f"stage_kb={os.environ.get('MPID_PASS_STAGE_KB', '48')} nb={nb} qrcp min {min(ts):.2f} ms  median {sorted(ts)[len(ts)//2]:.2f}", flush=True)
