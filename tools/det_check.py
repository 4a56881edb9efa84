import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2012_00706_b200.mpid import MPID
from synth.generators import fourier_params, gen_fourier
fp = fourier_params(32, 64, 1024, 0)
At = gen_fourier(fp, 0, device="cuda")
res = []
for rep in range(2):
    h = MPID(At, k_max=100)
    q = h.qrcp("fp16", "pow2", k=100)
    R = h.get_R().cpu().numpy()
    outs = []
    for eng in ("int8", "int8", "dmma", "int8"):
        h.set_fp64_engine(eng)
        P = h.coeffs("lsq").cpu().numpy(); e = h.error()
        outs.append((P, e))
    res.append((q.piv.copy(), R, outs))
    h.close()
print("piv equal", np.array_equal(res[0][0], res[1][0]))
print("R equal", np.array_equal(res[0][1], res[1][1]), np.abs(res[0][1]-res[1][1]).max())
for i in range(4):
    print("call", i, "P equal across handles", np.array_equal(res[0][2][i][0], res[1][2][i][0]), res[0][2][i][1], res[1][2][i][1])
print("int8 within handle", np.array_equal(res[0][2][0][0], res[0][2][1][0]), np.array_equal(res[0][2][0][0], res[0][2][3][0]))
