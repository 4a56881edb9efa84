"""One QRCP of C5's per-GPU share at 8 GPUs (2,097,152 x 2048 Fourier snapshots, 256 modes,
k = 512, fp16): the tcgen05 panel pass at the C5 shard shape (for ncu: the trailing update's
tensor-pipe utilisation; SURVEY H3's standalone K7 evidence)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_00706_b200.mpid import MPID
from synth import config_spec
from synth.generators import fourier_params, gen_fourier
spec = config_spec("C5")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, row0=0, m_loc=spec.m // 8, device="cuda")
h = MPID(A, k_max=512, m_global=spec.m // 8)
q = h.qrcp("fp16", "pow2", k=int(sys.argv[1]) if len(sys.argv) > 1 else 512, profile=True)
st = h.stats()
print({k: st[k] for k in ("t_qrcp_ms", "t_pass_ms", "formation", "nb", "k_out")})
