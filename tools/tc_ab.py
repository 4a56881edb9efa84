"""A/B of the tcgen05 pass variants on C4 (fp16, k = 100, nb = 16): one subprocess per
environment setting (the knobs are read once per process), QRCP time min / median of 5."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys
sys.path.insert(0, %r)
import torch
from paper_2012_00706_b200 import mpid
from synth import config_spec, fourier_params, gen_fourier
spec = config_spec("C4")
fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
A = gen_fourier(fp, 0, 0, spec.m, device="cuda")
h = mpid.MPID(A, k_max=100)
ts = []
for rep in range(6):
    q = h.qrcp("fp16", "pow2", k=100)
    if rep: ts.append(h.stats()["t_qrcp_ms"])
ts.sort()
print("%%s qrcp min %%.2f median %%.2f ms piv[:6]=%%s" %% (os.environ.get("TAG"), ts[0], ts[len(ts)//2], list(q.piv[:6])), flush=True)
''' % ROOT
# (libmpid_base.so: a build of the previous commit, copied beside libmpid.so by hand)
combos = [("nvb2", {"MPID_TC_NVB": "2"}), ("nvb3", {})]
for tag, env in combos * int(sys.argv[1] if len(sys.argv) > 1 else 1):
    e = dict(os.environ, TAG=tag, **env)
    r = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or ("FAILED " + tag + ": " + r.stderr[-800:]), flush=True)
