#!/usr/bin/env python
"""SURVEY A33 calibration of the tie-certification constant c_tie (reading R10).

Runs the oracle against itself in two faithful orders — model "paper" (per-operation
RNE update, fp64 sums in row order) and model "kernel" (one-rounding update, 8-row fp32
chains) — over >= 20 seeds of C1 and C2 (and 5 seeds of the 32^3-row C4 analogue) in
fp16 and fp32 at nb = 4 and nb = 32, records every first pivot divergence and the
paper-model top-2 margin at that step in units of u32 * max_i ||a_i||, and sets
c_tie = max(8, 4 x the largest such margin).  Calls only oracle/ (and the seeded input
generators); writes tests/golden/ctie_calibration.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.fast import qrcp_c  # noqa: E402
from oracle.qrcp import make_AL  # noqa: E402
from synth import gen_config  # noqa: E402
from synth.generators import fourier_params, gen_fourier  # noqa: E402

U32 = 2.0 ** -24


def runs():
    for seed in range(20):
        A = gen_config("C1", seed)
        for fmt, sc in (("fp16", "pow2"), ("fp32", "none")):
            yield "C1", seed, fmt, sc, A, 32
    for seed in range(20):
        A = gen_config("C2", seed)
        for fmt, sc in (("fp16", "maxabs"), ("fp32", "none")):
            yield "C2", seed, fmt, sc, A, 128
    for seed in range(5):
        fp = fourier_params(32, 64, 1024, seed)
        A = gen_fourier(fp, seed)
        yield "C4a", seed, "fp16", "pow2", A, 100


def main():
    out = {"what": __doc__.strip().splitlines()[0], "unit": "u32 * max_i ||a_i||", "runs": 0,
           "divergences": [], "min_certified_margin_seen": None}
    t0 = time.time()
    min_margin = np.inf
    for name, seed, fmt, sc, A, k in runs():
        AL, _ = make_AL(A, fmt, sc)
        for nb in (4, 32):
            a = qrcp_c(AL, k, fmt, nb=nb, model="paper")
            b = qrcp_c(AL, k, fmt, nb=nb, model="kernel")
            out["runs"] += 1
            unit = U32 * a.maxnorm0
            margins = (a.top2[:, 0] - a.top2[:, 1]) / unit
            kk = min(a.k_out, b.k_out)
            d = next((j for j in range(kk) if a.perm[j] != b.perm[j]), None)
            upto = kk if d is None else d
            if upto:
                min_margin = min(min_margin, float(np.min(margins[:upto])))
            if d is not None:
                out["divergences"].append({"config": name, "seed": seed, "fmt": fmt, "nb": nb, "step": int(d),
                                           "margin": float(margins[d]),
                                           "set_equal": bool(set(a.perm[:kk]) == set(b.perm[:kk]))})
            print(name, seed, fmt, nb, "diverge at", d, "margin %.3g" % (margins[d] if d is not None else -1),
                  flush=True)
    mx = max([d["margin"] for d in out["divergences"]], default=0.0)
    out["max_margin_at_divergence"] = mx
    out["min_certified_margin_seen"] = float(min_margin)
    out["c_tie"] = max(8.0, 4.0 * mx)
    out["seconds"] = time.time() - t0
    p = os.path.join(ROOT, "tests", "golden", "ctie_calibration.json")
    json.dump(out, open(p, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "divergences"}))


if __name__ == "__main__":
    main()
