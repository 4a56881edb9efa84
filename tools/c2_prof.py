"""C2 (4096 x 1024, k = 128, fp16): one QRCP + coefficients + error, for an ncu launch list."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2012_00706_b200.mpid import MPID
from synth import gen_config
A = torch.from_numpy(np.ascontiguousarray(gen_config("C2", 0).T)).cuda()
h = MPID(A, k_max=128)
for i in range(3):
    h.qrcp("fp16", "maxabs", k=128)
    h.coeffs("lsq")
    h.error()
print(h.stats())
