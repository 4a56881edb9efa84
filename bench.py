#!/usr/bin/env python
"""Benchmark of the mixed-precision ID hot path (arXiv 2012.00706) on B200.

One "step" = one full rank-k ID of the workload through the C ABI:
  scale + round A_D -> A_L, low-precision pivoted Householder QR (k steps),
  fp64 coefficients P (LSQ refit), fp64 error ||A_D - A_D(:,I)P||_F.
Workload: BASELINE.json configs[3] ("C4", 128^3 x 1024,
64 Fourier modes, k = 100, fp16) — the largest config that fits one GPU
(configs[4] is 256 GiB).  With --gpus N (torchrun) every rank holds one C4-sized
row shard of an N x taller snapshot matrix (weak scaling; one NCCL allreduce per
QR step, the path's real exchange).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rank-k ID time & TFLOP/s (lowprec QRCP + fp64 coeffs) at 1/2/4/8 B200"


def flops(m, n, k, mode="lsq"):
    """Algorithmic flops: Householder QRCP, fp64 coefficients, error."""
    fq = sum(4.0 * (m - j) * (n - j - 1) + 3.0 * (m - j) for j in range(k)) + 2.0 * m * n
    fc = (4.0 * m * k * k + 2.0 * m * k * n + k * k * n) if mode == "lsq" else k * k * (n - k)
    fe = 2.0 * m * k * (n - k) + 3.0 * m * n
    return fq, fc, fe


def alg_qrcp_bytes(m, n, k, s):
    """SURVEY §8(d) B_QRCP, the algorithmic bytes of the low-precision QRCP: one read of the
    trailing matrix per step, s (m-j)(n-j), plus a write and a read of it at each panel end of
    the survey's blocked algorithm (panel width min(k, 128): panel ends at j = 128, 256, ...
    below k).  For C4 (k = 100) there is no panel end: 4.087e11 B."""
    nb_s = min(k, 128)
    tot = 0.0
    for j in range(k):
        e = (m - j) * (n - j) * s
        tot += e * (3.0 if (j > 0 and j % nb_s == 0) else 1.0)
    return tot


def design_pass_bytes(m, n, k, nb, s, formation):
    """Bytes the dominant kernel actually moves per ID with this design: every step reads the
    trailing matrix, store steps (every nb) also write it back, and the tcgen05 pass reads the
    panel's V operand (m rows x 16 pending per K chunk x 2 (hi, lo) x 2 B) once per step."""
    tot = 0.0
    for j in range(k):
        e = (m - j) * (n - j) * s
        tot += e * (2.0 if (j > 0 and j % nb == 0) else 1.0)
        if formation == 2:
            npend = j - (0 if j == 0 else nb * ((j - 1) // nb))
            tot += (m - j) * 64.0 * ((npend + 15) // 16)
    return tot


def load_fp64_peak():
    p = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
    d = json.load(open(p))
    return float(d["used_as_peak"]), "profiles/r02_fp64_peak.json (tools/dmma_probe.cu on a B200: DMMA register-resident; cuBLAS DGEMM 35.5)"


def full_id_roofline(m, n, k, s, hbm_gbs, f_coef, f_err, small_ms, t_total_ms, engine=1, i8_tops=None, engine_err=None):
    """SURVEY §8(d) full-ID floor: round (8 + 8 + s B per element: max|a| pass + rounding)
    and the ALGORITHMIC QRCP bytes (B_QRCP) at the measured HBM bandwidth, the fp64 work at
    its engine's peak, plus k times the measured per-step cost of the small kernels;
    fraction = floor / time.  fp64 engine 1 (DMMA): the coefficient and error flops at the
    measured DMMA peak (the error also bounded by one fp64 read of A_D(:, J)).  Engine 2 (int8
    tensor cores, Ozaki scheme, k_ozaki.cu): Q1 = A_I R11^-1 (2 m k^2) on DMMA; [G2 | W] and
    the error's A_I T cost 36 int8 multiply-adds per fp64 one (8 slices, the 36 pairs with
    p + q <= 7) at the int8 peak, each also bounded by one read of A_D(:, J)."""
    bw = hbm_gbs * 1e9
    p64, src = load_fp64_peak()
    t_round = (8.0 + 8.0 + s) * m * n / bw
    t_qrcp = alg_qrcp_bytes(m, n, k, s) / bw
    nj = n - k
    engine_err = engine if engine_err is None else engine_err
    if engine == 2 and i8_tops:
        t_coef = 2.0 * m * k * k / (p64 * 1e12) + max(36.0 * 2.0 * m * k * n / (i8_tops * 1e12),
                                                      8.0 * m * (n + k) / bw)
    else:
        t_coef = f_coef / (p64 * 1e12)
    if engine_err == 2 and i8_tops:
        t_err = max(36.0 * 2.0 * m * k * nj / (i8_tops * 1e12), 8.0 * m * nj / bw)
    else:
        t_err = max(f_err / (p64 * 1e12), 8.0 * m * nj / bw)
    t_roof = (t_round + t_qrcp + t_coef + t_err) * 1e3 + max(0.0, small_ms)
    return {"t_roof_ms": t_roof, "frac": t_roof / t_total_ms,
            "parts_ms": {"round": t_round * 1e3, "qrcp_pass": t_qrcp * 1e3, "coef": t_coef * 1e3,
                         "error": t_err * 1e3, "qrcp_small_kernels_measured": small_ms},
            "fp64_engine": {"coef": {1: "DMMA", 2: "int8 Ozaki"}.get(engine, str(engine)),
                            "error": {1: "DMMA", 2: "int8 Ozaki"}.get(engine_err, str(engine_err))},
            "peaks": {"hbm_gbs": hbm_gbs, "fp64_tflops": p64, "fp64_source": src,
                      "int8_tops": i8_tops,
                      "int8_source": "2 x MEASURED_PEAKS.json bf16_tflops (B200_PROFILING.md nominal int8 / bf16 = 4.5 / 2.25)"}}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_sample(rows, k, nb, fmt, seed=0, repeats=1):
    """The oracle, as it stands, on a bounded row sample of the workload: the first `rows`
    rows of C4, A_L by the oracle's rounding, the oracle's QRCP (oracle/cqrcp.c, the paper
    model, OpenMP over all host cores), its Householder LSQ coefficients and its error.
    Returns (seconds, flops, cores)."""
    import numpy as np
    from oracle.fast import qrcp_c
    from oracle.id import coeffs_lsq, id_error_blocked
    from oracle.qrcp import make_AL
    from synth import gen_config
    A = gen_config("C4", seed, row0=0, m_loc=rows)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    for _ in range(repeats):
        AL, s = make_AL(A, fmt, "pow2" if fmt == "fp16" else "none")
        r = qrcp_c(AL, k, fmt, nb=nb, model="paper", threads=cores)
        P = coeffs_lsq(A, r.I)
        id_error_blocked(A, r.I, P)
    dt = (time.perf_counter() - t0) / repeats
    fq, fc, fe = flops(rows, A.shape[1], k)
    return dt, fq + fc + fe, cores


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--fmt", default="fp16")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--nb", type=int, default=0, help="store interval; 0 = library default (tcgen05: 16, FFMA: 4)")
    ap.add_argument("--formation", default="auto", help="auto | tc | ffma")
    ap.add_argument("--mode", default="lsq")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--rows", type=int, default=0, help="override rows per GPU (debug)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the untimed variants / extra errors (ncu launch lists)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-rows", type=int, default=65536)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from synth import config_spec
    spec = config_spec(args.config)
    k = args.k or spec.ks[0]
    rows = args.rows or spec.m
    scaling = spec.scaling[args.fmt]

    nb_lib = args.nb or (16 if args.fmt == "fp16" and args.formation != "ffma" else 4)
    if args.impl == "reference":
        if rank != 0:
            return 0
        # the oracle, as it stands, on the host cores; each step one bounded sample
        wsteps = []
        for i in range(args.warmup + args.steps):
            dt, fl, cores = cpu_oracle_sample(args.cpu_rows, k, nb_lib, args.fmt, args.seed)
            if i >= args.warmup:
                wsteps.append(dt)
        T = sum(wsteps) / len(wsteps)
        val = fl / T / 1e12
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": T * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32+f64 (simulated fp16)" if args.fmt == "fp16" else "f32+f64",
                "data": "synthetic",
                "config": {"workload": f"{args.config} row sample", "rows": args.cpu_rows, "n": spec.n,
                           "k": k, "fmt": args.fmt, "nb": nb_lib, "coef": args.mode,
                           "oracle": "oracle/cqrcp.c paper model + numpy fp64 LSQ / error"},
                "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                                 "sample": f"first {args.cpu_rows} rows of {args.config} ({args.cpu_rows}x{spec.n}, k={k})"},
                "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2012_00706_b200 import mpid

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    mpid.lib()

    from paper_2012_00706_b200.dist import broadcast_bytes, max_over_ranks, shard_rows
    comm = None
    if world > 1:
        uid = broadcast_bytes(mpid.id_nccl_get_unique_id() if rank == 0 else None,
                              mpid.lib().id_nccl_unique_id_bytes(), device=dev)
        comm = mpid.id_nccl_comm_init(uid, world, rank)

    # ---- input: this rank's row shard, generated on device ------------------
    from synth import fourier_params, gen_fourier
    if args.config == "C5":          # strong: the 2^24-row matrix split over the ranks
        m_glob = spec.m
        row0, m_loc = shard_rows(m_glob, world, rank)
    else:                            # weak: every rank holds a config-sized shard
        m_loc = rows
        m_glob = rows * world
        row0 = rank * rows
    if args.config in ("C4", "C5"):
        fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, args.seed)
        A = gen_fourier(fp, args.seed, row0=row0, m_loc=m_loc, device=dev)
    else:
        from synth import gen_config
        A = torch.from_numpy(np.ascontiguousarray(gen_config(args.config, args.seed).T)).to(dev)
        m_loc = m_glob = A.shape[1]
    n = spec.n
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    h = mpid.MPID(A, k_max=k, m_global=m_glob, row_offset=row0, comm=comm, rank=rank, nranks=world,
                  stream=stream)
    s_bytes = 2 if args.fmt == "fp16" else 4

    def one_step(profile):
        q = h.qrcp(args.fmt, scaling, k=k, nb=args.nb, profile=profile, formation=args.formation)
        P = h.coeffs(args.mode)
        e = h.error()
        return q, P, e

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        q, P, e = one_step(True)
    st0 = h.stats()

    clocks = Clocks(local_rank)
    barrier()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    pass_ms, qr_ms, coef_ms, err_ms, round_ms = [], [], [], [], []
    ev0.record(stream)
    for _ in range(args.steps):
        q, P, e = one_step(True)
        st = h.stats()
        pass_ms.append(st["t_pass_ms"])
        qr_ms.append(st["t_qrcp_ms"])
        round_ms.append(st["t_round_ms"])
        coef_ms.append(st["t_coef_ms"])
        err_ms.append(st["t_err_ms"])
        st_last = st
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    t_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t_ms = max_over_ranks(t_ms, device=dev)
    ms_step = t_ms / args.steps
    fq, fc, fe = flops(m_glob, n, q.k, args.mode)
    value = (fq + fc + fe) / (ms_step * 1e-3) / 1e12

    # ---- the paper's other metrics, outside the timed region ----
    extra_err = {}
    try:
        if not args.no_extras:
            extra_err["rel_fro_low_skeleton"] = h.error_ex("AL", "fro")[1]
            extra_err["rel_2norm_mixed"] = h.error_ex("AD", 2, iters=40)[1]
            extra_err["rel_2norm_low_skeleton"] = h.error_ex("AL", 2, iters=40)[1]
    except Exception as ex:  # reported, never silently replaced
        extra_err["error"] = str(ex)

    # ---- NEXT-4 variants, timed separately (not the headline): Gram / sketched pivoting ----
    variants = {}
    if args.fmt == "fp16" and world == 1 and not args.no_extras:
        for name, form in (("gram_pivoting", "gram"), ("sketched_pivoting", "sketch")):
            try:
                ts = []
                for i in range(4):
                    torch.cuda.synchronize()
                    g0 = torch.cuda.Event(enable_timing=True)
                    g1 = torch.cuda.Event(enable_timing=True)
                    g0.record(stream)
                    qg = h.qrcp("fp16", scaling, k=k, formation=form, allow_underflow=True)
                    h.coeffs(args.mode)
                    eg = h.error()
                    g1.record(stream)
                    torch.cuda.synchronize()
                    if i > 0:
                        ts.append((g0.elapsed_time(g1), h.stats()["t_qrcp_ms"]))
                variants[name] = {
                    "ms_per_step": statistics.mean(t for t, _ in ts), "pivot_ms": statistics.mean(p for _, p in ts),
                    "k_out": qg.k, "rel_err_fro": eg[1],
                    "same_skeleton_as_householder": bool(sorted(qg.piv.tolist()) == sorted(q.piv.tolist())),
                    "note": f"formation {form} (DESIGN.md NEXT-4), 3 timed steps, CUDA events"}
            except Exception as ex:  # reported, never silently replaced
                variants[name] = {"error": str(ex)}
        # the paper's own Algorithm 2 coefficients (P_L = R11^-1 R12 from the low-precision R,
        # lines 5-6) instead of the LSQ refit: same QRCP, a k x n triangular solve
        try:
            ts = []
            for i in range(4):
                torch.cuda.synchronize()
                g0 = torch.cuda.Event(enable_timing=True)
                g1 = torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                qr = h.qrcp(args.fmt, scaling, k=k, nb=args.nb, formation=args.formation)
                h.coeffs("R")
                er = h.error()
                g1.record(stream)
                torch.cuda.synchronize()
                if i > 0:
                    ts.append((g0.elapsed_time(g1), h.stats()["t_coef_ms"]))
            variants["algorithm2_R_mode_coefficients"] = {
                "ms_per_step": statistics.mean(t for t, _ in ts), "coef_ms": statistics.mean(c for _, c in ts),
                "k_out": qr.k, "rel_err_fro": er[1],
                "note": "Householder QRCP as the headline, P = R11^-1 R12 (paper Algorithm 2) instead of LSQ"}
        except Exception as ex:  # reported, never silently replaced
            variants["algorithm2_R_mode_coefficients"] = {"error": str(ex)}
        # the headline handle state (last QRCP) is restored for the checks below
        q = h.qrcp(args.fmt, scaling, k=k, nb=args.nb, formation=args.formation)
        # the fp64 stage with each engine forced (same skeleton): DMMA and int8 (Ozaki scheme)
        for other in ("dmma", "int8"):
            vname = f"fp64_stage_all_{other}"
            try:
                cm, em = [], []
                h.set_fp64_engine(other)
                for i in range(3):
                    h.coeffs(args.mode)
                    ed = h.error()
                    sd = h.stats()
                    cm.append(sd["t_coef_ms"])
                    em.append(sd["t_err_ms"])
                h.set_fp64_engine("auto")
                variants[vname] = {
                    "coef_ms": statistics.mean(cm[1:]), "error_ms": statistics.mean(em[1:]), "rel_err_fro": ed[1],
                    "rel_err_fro_headline": e[1], "engines": [sd["fp64_engine"], sd["fp64_engine_err"]],
                    "note": f"same QRCP, coefficients + error with id_set_fp64_engine({other}); 2 timed calls"}
            except Exception as ex:  # reported, never silently replaced
                h.set_fp64_engine("auto")
                variants[vname] = {"error": str(ex)}
        h.coeffs(args.mode)
        h.error()

    # ---- roofline of the dominant kernel (the panel pass), per launch ----------
    # achieved = SURVEY §8(d)'s ALGORITHMIC bytes B_QRCP / the summed device time of the k
    # pass launches (CUDA events on the library's stream around each launch); the bytes the
    # design moves beyond B_QRCP (store-step write-backs every nb steps, the tcgen05 pass's V
    # operand) are reported separately, as is the ncu-measured DRAM traffic per launch.
    peak, peak_kind, peaks = load_peaks()
    form = int(st0["formation"])
    nb_used = int(st0["nb"])
    alg = alg_qrcp_bytes(m_loc, n, q.k, s_bytes)
    design = design_pass_bytes(m_loc, n, q.k, nb_used, s_bytes, form)
    pass_avg_ms = statistics.mean(pass_ms)
    achieved = alg / (pass_avg_ms * 1e-3) / 1e9          # GB/s of algorithmic bytes
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "pass_traffic.json")
    if os.path.exists(prof):
        try:
            pt = json.load(open(prof))
            ent = pt.get("kernels", {}).get("k_pass_tc" if form == 2 else "k_pass_ws")
            if ent and ent.get("nb") == nb_used and ent.get("workload") == args.config:
                traffic, traffic_src = ent["dram_bytes_per_launch"], ent["source"]
        except Exception:
            traffic = None

    # ---- e2e through the C ABI with host buffers ------------------------------
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty((n, m_loc), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A)
        del A
        h.close()
        torch.cuda.empty_cache()
        times = []
        for i in range(args.e2e_steps + 1):
            barrier()
            t0 = time.perf_counter()
            hh = mpid.MPID(Ah, k_max=k, m_global=m_glob, row_offset=row0, comm=comm, rank=rank,
                           nranks=world, stream=stream, device=dev)
            qq = hh.qrcp(args.fmt, scaling, k=k, nb=args.nb, formation=args.formation)
            PP = hh.coeffs(args.mode)
            P_host = PP.cpu()
            ee = hh.error()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            hh.close()
            del hh, PP
            if i > 0:
                times.append(dt)
        dt = statistics.mean(times)
        if world > 1:
            dt = max_over_ranks(dt, device=dev)
        e2e = {"value": (fq + fc + fe) / dt / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(m_loc * n * 8 * world),
               "d2h_bytes_per_step": int((k * n * 8 + k * 4 + 16) * world),
               "ms_per_step": dt * 1e3}

    cpu = None
    if rank == 0 and not args.no_cpu:
        dt_c, fl_c, cores = cpu_oracle_sample(args.cpu_rows, k, nb_used, args.fmt, args.seed)
        cpu = {"value": fl_c / dt_c / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
               "sample": f"first {args.cpu_rows} rows of {args.config} ({args.cpu_rows}x{n}, k={k}), one full ID",
               "seconds": dt_c}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if args.config == "C5" else "weak",
            "vs_baseline": None,
            "dtype": ("f16 storage / f32 arithmetic QRCP + f64 ID" if args.fmt == "fp16" else "f32 QRCP + f64 ID")
                     + (" (f64 error GEMM on the int8 tensor cores, Ozaki scheme)" if int(st_last.get("fp64_engine_err", 1)) == 2 else ""),
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {m_glob}x{n} fp64 Fourier snapshots, k={k}, "
                                   f"{args.fmt} QRCP ({'tcgen05' if form == 2 else 'FFMA'} pass, nb={nb_used}), "
                                   f"{args.mode.upper()} coefficients",
                       "rows_per_gpu": m_loc, "n": n, "k": k, "fmt": args.fmt, "nb": nb_used,
                       "coef": args.mode, "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU",
                       "fp64_engine": {"coef": {1: "dmma", 2: "int8-ozaki"}.get(int(st_last.get("fp64_engine", 1)), "?"),
                                       "error": {1: "dmma", 2: "int8-ozaki"}.get(int(st_last.get("fp64_engine_err", 1)), "?")},
                       "l2": "inputs larger than L2 (A_D 16 GiB, A_L 4 GiB per GPU); no flush"},
            "stages_ms": {"round": statistics.mean(round_ms), "qrcp": statistics.mean(qr_ms),
                          "coef": statistics.mean(coef_ms), "error": statistics.mean(err_ms),
                          "pass_total": pass_avg_ms},
            "tflops_parts": {"qrcp": fq / (statistics.mean(qr_ms) * 1e-3) / 1e12,
                             "fp64": (fc + fe) / ((statistics.mean(coef_ms) + statistics.mean(err_ms)) * 1e-3) / 1e12},
            "full_id_roofline": full_id_roofline(m_loc, n, q.k, s_bytes, peak, fc, fe,
                                                 statistics.mean(qr_ms) - pass_avg_ms, ms_step,
                                                 engine=int(st_last.get("fp64_engine", 1)),
                                                 i8_tops=2.0 * peaks["bf16_tflops"] if peaks.get("bf16_tflops") else None,
                                                 engine_err=int(st_last.get("fp64_engine_err", 1))),
            "k_out": q.k, "rel_err_fro": e[1], "errors_untimed": extra_err, "variants": variants,
            "roofline": {"kernel": ("k_pass_tc (tcgen05 panel pass)" if form == 2 else "k_pass_ws (FFMA panel pass)"),
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_kind": peak_kind, "launches_per_step": q.k,
                         "algorithmic_bytes_per_step": alg, "algorithmic_bytes_per_launch": alg / q.k,
                         "bytes_def": "SURVEY 8(d) B_QRCP: s * sum_j (m-j)(n-j) (+ 2 s (m-j)(n-j) per panel end of width min(k,128))",
                         "design_bytes_per_step": design, "design_extra_bytes": design - alg,
                         "design_over_algorithmic": design / alg,
                         "traffic_over_algorithmic": (traffic * q.k / alg) if traffic else None,
                         "formation": form, "nb": nb_used},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(st0["kernel_launches"]) * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line))
    if comm:
        mpid.id_nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
