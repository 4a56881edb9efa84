"""Debug: GPU vs oracle pivots/R rows on C1 for given (fmt, nb, graph) cases.
usage: debug_parity.py fmt:nb:graph [...]   e.g. fp32:1:0 fp16:4:1"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import gen_config
from oracle.qrcp import make_AL, qrcp_householder
from tests.gpu_helpers import run_gpu, prefix_match
A = gen_config(os.environ.get("CFG", "C1"), 0)
k = int(os.environ.get("K", "32"))
for case in sys.argv[1:]:
    fmt, nb, g = case.split(":")
    nb, g = int(nb), bool(int(g))
    sc = "pow2" if fmt == "fp16" else "none"
    print("case", fmt, nb, g, flush=True)
    out = run_gpu(A, fmt, sc, k, nb=nb, use_graph=g)
    AL, s = make_AL(A, fmt, sc)
    r = qrcp_householder(AL, k, fmt, nb=nb)
    agree, fu = prefix_match(out["piv"], r)
    Rg = out["R"]
    d = [float(np.abs(Rg[i, i:] - r.R[i, i:]).max()) for i in range(min(agree + 1, k))]
    print(fmt, nb, g, "agree", agree, "first_unc", fu, "Rdiff", ["%.1e" % x for x in d[:6]], flush=True)
