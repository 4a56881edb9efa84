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
    parts = case.split(":")
    fmt, nb, g = parts[:3]
    form = parts[3] if len(parts) > 3 else "ffma"
    nb, g = int(nb), bool(int(g))
    sc = "pow2" if fmt == "fp16" else "none"
    print("case", fmt, nb, g, form, flush=True)
    out = run_gpu(A, fmt, sc, k, nb=nb, use_graph=g, formation=form)
    AL, s = make_AL(A, fmt, sc)
    r = qrcp_householder(AL, k, fmt, nb=nb, formation="tc" if form == "tc" else "fma")
    agree, fu = prefix_match(out["piv"], r)
    Rg = out["R"]
    d = [float(np.abs(Rg[i, i:] - r.R[i, i:]).max()) for i in range(min(agree + 1, k))]
    print(fmt, nb, g, form, "stats", out["stats"]["formation"], "err", out["err"][1], "agree", agree, "first_unc", fu, "Rdiff", ["%.1e" % x for x in d[:6]], flush=True)
