"""Power / clock probe of the C4 QRCP (tcgen05 pass): runs the QRCP alone R times back to back
and, separately, with idle gaps, sampling nvidia-smi (SM clock, power, throttle reasons) every
50 ms.  Question it answers: is the pass's in-bench time (~88 ms per C4 ID) set by the SM clock
under sw_power_cap (the ncu launch list, serialised with gaps, sums to ~76 ms)?"""
import os
import statistics
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2012_00706_b200.mpid import MPID
from synth import config_spec, fourier_params, gen_fourier

Q = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap"


def sample(fn):
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=f, stderr=subprocess.DEVNULL)
    time.sleep(0.3)
    out = fn()
    p.terminate()
    p.wait(timeout=5)
    rows = [r.split(",") for r in open(f.name).read().strip().splitlines() if r.strip()]
    os.unlink(f.name)
    sm = [float(r[0]) for r in rows[6:]]
    pw = [float(r[1]) for r in rows[6:]]
    cap = sum(1 for r in rows[6:] if r[2].strip().lower() == "active")
    return out, {"sm_mhz_med": statistics.median(sm) if sm else None, "sm_mhz_min": min(sm) if sm else None,
                 "power_w_med": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None,
                 "power_cap_samples": cap, "samples": len(sm)}


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    spec = config_spec("C4")
    fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, 0)
    A = gen_fourier(fp, 0, row0=0, m_loc=spec.m, device="cuda")
    h = MPID(A, k_max=100)
    h.qrcp("fp16", "pow2", k=100, profile=True)          # warm-up (graphs, tensor maps)

    def loop(gap):
        t = []
        for _ in range(reps):
            h.qrcp("fp16", "pow2", k=100, profile=True)
            st = h.stats()
            t.append((st["t_qrcp_ms"], st["t_pass_ms"]))
            if gap:
                time.sleep(gap)
        return t

    for gap in (0.0, 0.5):
        t, clk = sample(lambda: loop(gap))
        print({"gap_s": gap, "t_qrcp_ms": [round(a, 2) for a, _ in t], "t_pass_ms": [round(b, 2) for _, b in t],
               "clocks": clk}, flush=True)


if __name__ == "__main__":
    main()
