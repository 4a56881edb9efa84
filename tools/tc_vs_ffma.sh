timeout 600 python -m pytest tests/test_gpu_smem.py -q -p no:cacheprovider -x > gpurun_out/smem_tests.log 2>&1; echo "rc $?" >> gpurun_out/smem_tests.log
python - <<'PY' > gpurun_out/tc_vs_ffma.log 2>&1
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2012_00706_b200.mpid import MPID
from synth import gen_config
from synth.generators import fourier_params, gen_fourier
def t(At, fmt, sc, k, form, nb=0, reps=3):
    h = MPID(At, k_max=k)
    ts = []
    for i in range(reps + 1):
        q = h.qrcp(fmt, sc, k=k, nb=nb, formation=form)
        st = h.stats()
        if i: ts.append(st["t_qrcp_ms"])
    h.close()
    return min(ts), st["formation"], st["nb"]
for name, k in (("C1", 32), ("C2", 128), ("C2", 64), ("C3", 256)):
    A = gen_config(name, 0)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    sc = "maxabs" if name == "C2" else "pow2"
    for form in (["smem", "ffma", "tc"] if name == "C1" else ["ffma", "tc"]):
        print(name, k, form, t(At, "fp16", sc, k, form), flush=True)
for N, n, L, k in ((64, 1024, 64, 100), (96, 1024, 64, 100), (128, 1024, 64, 100)):
    fp = fourier_params(N, L, n, 0)
    At = gen_fourier(fp, 0, device="cuda")
    for form in ("ffma", "tc"):
        print("fourier", N ** 3, k, form, t(At, "fp16", "pow2", k, form, reps=2), flush=True)
    del At; torch.cuda.empty_cache()
PY
