"""Where does the host time between the three C-ABI calls go? (C4 workload)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m, device="cuda")
h = mpid.MPID(A, k_max=100)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); q = h.qrcp("fp16", "pow2", k=100, nb=4); t1 = time.perf_counter()
    P = h.coeffs("lsq"); t2 = time.perf_counter()
    e = h.error(); t3 = time.perf_counter()
    st = h.stats()
    print(f"host: qrcp {1e3*(t1-t0):.2f} coef {1e3*(t2-t1):.2f} err {1e3*(t3-t2):.2f} total {1e3*(t3-t0):.2f} | "
          f"events: qrcp {st['t_qrcp_ms']:.2f} coef {st['t_coef_ms']:.2f} err {st['t_err_ms']:.2f} "
          f"launch(host) {st['t_host_launch_ms']:.2f} call(gpu) {st['t_call_gpu_ms']:.2f}", flush=True)
