"""C4 (bench workload): one QRCP, then the fp64 stage with the int8 engine and with DMMA
(for an ncu launch list: python tools/oz_prof.py under ncu -k regex:... )."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200.mpid import MPID
from synth import config_spec
from synth.generators import fourier_params, gen_fourier
spec = config_spec("C4")
rows = int(sys.argv[1]) if len(sys.argv) > 1 else spec.m
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, row0=0, m_loc=rows, device="cuda")
h = MPID(A, k_max=100)
h.qrcp("fp16", "pow2", k=100)
for eng in ("int8", "dmma", "int8"):
    h.set_fp64_engine(eng)
    try:
        h.coeffs("lsq")
        e = h.error()
    except Exception as ex:   # measurement knobs (MPID_OZ_DBG) produce garbage coefficients
        e = str(ex)[:60]
    st = h.stats()
    print(eng, st["fp64_engine"], st["fp64_engine_err"], "coef", st["t_coef_ms"], "err", st["t_err_ms"], e)
