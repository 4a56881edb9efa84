"""C4 fp16 QRCP through the tcgen05 pass (for ncu captures of k_pass_tc)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2012_00706_b200.mpid import MPID
from synth.generators import fourier_params, gen_fourier

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
form = sys.argv[2] if len(sys.argv) > 2 else "tc"
fp = fourier_params(128, 64, 1024, 0)
At = gen_fourier(fp, 0, device="cuda")
h = MPID(At, k_max=100)
for it in range(2):
    q = h.qrcp("fp16", "pow2", k=100, nb=nb, formation=form, profile=True)
    st = h.stats()
    print(f"{form} nb={nb} qrcp {st['t_qrcp_ms']:.2f} ms pass {st['t_pass_ms']:.2f} ms", flush=True)
