"""Quick GPU probe of the tcgen05 pass against the FFMA pass and the oracle (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2012_00706_b200.mpid import MPID
from oracle.qrcp import make_AL, qrcp_householder
from oracle.fast import qrcp_c
from oracle.id import coeffs_lsq, id_error
from synth import gen_config, gen_planted
from synth.generators import fourier_params, gen_fourier
from tests.gpu_helpers import prefix_match, C_TIE


def run(A, fmt, sc, k, nb, formation, eps=0.0):
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    h = MPID(At, k_max=k)
    q = h.qrcp(fmt, sc, k=k, nb=nb, formation=formation, eps=eps)
    R = h.get_R().cpu().numpy().astype(np.float64)
    P = h.coeffs("lsq").cpu().numpy()
    e = h.error()
    st = h.stats()
    h.close()
    return q, R, P, e, st


cases = [("C1", gen_config("C1", 0), "fp16", "pow2", 32),
         ("C2", gen_config("C2", 1), "fp16", "maxabs", 128),
         ("planted", gen_planted(4096, 512, 64, rho=1.05, eta=1e-9, seed=2)[0], "fp16", "pow2", 64),
         ("C4a", gen_fourier(fourier_params(32, 64, 1024, 0), 0), "fp16", "pow2", 100)]
for name, A, fmt, sc, k in cases:
    AL, s = make_AL(A, fmt, sc)
    for nb in (32, 8):
        r = qrcp_householder(AL, k, fmt, nb=nb, formation="tc") if A.shape[0] <= 4096 else qrcp_c(AL, k, fmt, nb=nb)
        rp = qrcp_c(AL, k, fmt, nb=nb, model="paper")
        try:
            q, R, P, e, st = run(A, fmt, sc, k, nb, "tc")
        except Exception as ex:
            print(name, nb, "tc FAILED", ex, flush=True)
            continue
        ag, fu = prefix_match(q.piv, r, c_tie=C_TIE)
        ag2, fu2 = prefix_match(q.piv, rp, c_tie=C_TIE)
        kk = min(ag, k)
        dR = np.max(np.abs(R[:kk] - r.R[:kk])) / r.maxnorm0 / 2 ** -24 if kk else -1
        e_or = id_error(A, r.I, coeffs_lsq(A, r.I))[1]
        Pref = coeffs_lsq(A, q.piv)
        print(f"{name} nb={nb} k={q.k} agree tc-oracle {ag}/{fu} paper {ag2}/{fu2} dR/u32max {dR:.1f} "
              f"err {e[1]:.5e} oracle {e_or:.5e} ratio {e[1]/e_or:.4f} dP {np.linalg.norm(P-Pref)/np.linalg.norm(Pref):.1e} "
              f"form {st['formation']} nb {st['nb']}", flush=True)

# C4 full timing: tc vs ffma
fp = fourier_params(128, 64, 1024, 0)
At = gen_fourier(fp, 0, device="cuda")
h = MPID(At, k_max=100)
for form, nb in (("ffma", 4), ("tc", 32), ("tc", 16)):
    for it in range(3):
        q = h.qrcp("fp16", "pow2", k=100, nb=nb, formation=form, profile=True)
        st = h.stats()
    P = h.coeffs("lsq"); e = h.error()
    print(f"C4 {form} nb={nb}: qrcp {st['t_qrcp_ms']:.2f} ms pass {st['t_pass_ms']:.2f} ms err {e[1]:.6e} piv[:8] {q.piv[:8]}", flush=True)
