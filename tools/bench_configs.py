"""Time the full ID (scale/round + QRCP + LSQ coefficients + fused error) through the C ABI
on every BASELINE.json config that fits one GPU, plus the per-GPU workload of C5 at
8 GPUs (one 2^21-row shard; the allreduces it would add are ~k x 10-30 us).

    python tools/bench_configs.py > profiles/r01_configs.jsonl

One JSON line per (config, fmt, k): device time per ID (median of reps after a warm-up),
stage times, TFLOP/s of the algorithmic flops (bench.flops), the pass's HBM fraction
and the relative Frobenius error.  Inputs are generated on the device (C4/C5) or on
the host (C1-C3) — never timed.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import alg_qrcp_bytes, design_pass_bytes, flops, load_peaks  # noqa: E402
from paper_2012_00706_b200 import mpid  # noqa: E402
from synth import config_spec, fourier_params, gen_config, gen_fourier  # noqa: E402

CASES = [("C1", "fp16", 32, 0.0), ("C1", "fp32", 32, 0.0),
         ("C2", "fp32", 16, 0.0), ("C2", "fp32", 64, 0.0), ("C2", "fp32", 128, 0.0),
         ("C2", "fp16", 16, 0.0), ("C2", "fp16", 64, 0.0), ("C2", "fp16", 128, 0.0),
         ("C3", "fp16", 256, 0.0), ("C3", "fp16", 512, 1e-3),
         ("C3", "fp64", 256, 0.0),
         ("C4", "fp16", 100, 0.0), ("C4", "fp32", 100, 0.0), ("C4", "fp64", 100, 0.0),
         ("C5/8", "fp16", 512, 0.0),
         # C5's per-GPU shard at P = 4 from pinned HOST memory, streamed in row blocks (64 GiB)
         ("C5/4-host", "fp16", 512, 0.0),
         # NEXT-4: Gram pivoting (formation 3)
         ("C3", "fp16", 256, 0.0, "gram"), ("C4", "fp16", 100, 0.0, "gram"), ("C5/8", "fp16", 512, 0.0, "gram"),
         # NEXT-4 second option: sketched pivoting (formation 4)
         ("C3", "fp16", 256, 0.0, "sketch"), ("C4", "fp16", 100, 0.0, "sketch"), ("C5/8", "fp16", 512, 0.0, "sketch")]


def device_matrix(name):
    if name == "C5/4-host":
        spec = config_spec("C5")
        fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
        rows = spec.m // 4
        Ah = torch.empty((spec.n, rows), dtype=torch.float64, pin_memory=True)
        for c0 in range(0, rows, 1 << 21):          # generated on the device in row slabs
            Ah[:, c0:c0 + (1 << 21)].copy_(gen_fourier(fp, 0, c0, 1 << 21, device="cuda"))
        return Ah, spec
    if name in ("C4", "C5/8"):
        spec = config_spec("C4" if name == "C4" else "C5")
        fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
        rows = spec.m if name == "C4" else spec.m // 8
        return gen_fourier(fp, 0, 0, rows, device="cuda"), spec
    spec = config_spec(name)
    A = gen_config(name, 0)
    return torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), spec


def main():
    peak, _, _ = load_peaks()
    only = sys.argv[1:]
    cache = {}
    for case in CASES:
        name, fmt, k, eps = case[:4]
        formation = case[4] if len(case) > 4 else "auto"
        names = [a for a in only if a.startswith("C")]
        forms = [a for a in only if not a.startswith("C")]
        if (names and name not in names) or (forms and formation not in forms):
            continue
        if name not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[name] = device_matrix(name)
        At, spec = cache[name]
        n, m = At.shape
        scaling = spec.scaling.get(fmt, "pow2" if fmt == "fp16" else "none") if fmt != "fp64" else "none"
        host = not At.is_cuda
        h = mpid.MPID(At, k_max=k, m_global=m, fp64=fmt == "fp64", device="cuda", stream_host=host)
        reps = 5 if m * n < 1e9 else (1 if host else 3)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        times, st = [], None
        for it in range(reps + 1):
            torch.cuda.synchronize()
            ev[0].record()
            q = h.qrcp(fmt, scaling, k=k, eps=eps, formation=formation, allow_underflow=True)
            h.coeffs("lsq")
            e = h.error()
            ev[1].record()
            torch.cuda.synchronize()
            if it > 0:
                times.append(ev[0].elapsed_time(ev[1]))
                st = h.stats()
        t = statistics.median(times)
        fq, fc, fe = flops(m, n, q.k, "lsq")
        nb = st["nb"]
        sb = {"fp16": 2, "fp32": 4, "fp64": 8}[fmt]
        pb = alg_qrcp_bytes(m, n, q.k, sb)
        line = {"config": name, "m": m, "n": n, "fmt": fmt, "formation": formation, "formation_used": st["formation"],
                "k": q.k, "eps": eps, "nb": nb, "host_streamed": host,
                "ms_per_id": t, "tflops": (fq + fc + fe) / (t * 1e-3) / 1e12,
                "stages_ms": {"round": st["t_round_ms"], "qrcp": st["t_qrcp_ms"], "coef": st["t_coef_ms"],
                              "error": st["t_err_ms"]},
                "qrcp_alg_bytes_hbm_frac_of_measured": (pb / (st["t_qrcp_ms"] * 1e-3) / 1e9 / peak
                                                        if formation not in ("gram", "sketch") else None),
                "design_over_alg_bytes": (design_pass_bytes(m, n, q.k, nb, sb, st["formation"]) / pb
                                          if formation not in ("gram", "sketch") else None),
                "h2d_gbs_round": ((2 if fmt == "fp16" else 1) * m * n * 8 / (st["t_round_ms"] * 1e-3) / 1e9
                                  if host else None),
                "gram_tflops": (m * n * n) / (st["t_qrcp_ms"] * 1e-3) / 1e12 if formation == "gram" else None,
                "pivot_ms": st["t_qrcp_ms"],
                "rel_err_fro": e[1]}
        print(json.dumps(line), flush=True)
        h.close()


if __name__ == "__main__":
    main()
