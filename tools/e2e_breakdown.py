"""Where the end-to-end (host-buffer) time of one C4 ID goes: H2D copy in id_create, the
first QRCP call of a handle (graph capture + instantiate + run), coefficients + P to host,
error.  Wall clock with device syncs between phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m, device="cuda")
Ah = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
Ah.copy_(A)
del A
torch.cuda.empty_cache()
for it in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    h = mpid.MPID(Ah, k_max=100)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    q = h.qrcp("fp16", "pow2", k=100)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    q = h.qrcp("fp16", "pow2", k=100)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    P = h.coeffs("lsq").cpu()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    e = h.error()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    h.close()
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"create+H2D {d[0]:.1f} ms  qrcp#1 (capture) {d[1]:.1f}  qrcp#2 {d[2]:.1f}  coeffs+D2H {d[3]:.1f}  error {d[4]:.1f}")
