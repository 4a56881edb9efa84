"""Update profiles/pass_traffic.json's k_pass_tc entry from an ncu launch list that carries
gpu__time_duration.sum, dram__bytes_read.sum and dram__bytes_write.sum (tools/gpu_final3.sh:
bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras under ncu; the LAST k launches of
the kernel = the timed ID of C4).
usage: python tools/traffic_from_launches.py gpurun_out/launches_r02.csv profiles/<list>.txt [k=100]"""
import csv, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import alg_qrcp_bytes  # noqa: E402
from synth import config_spec  # noqa: E402

path, src = sys.argv[1], sys.argv[2]
k = int(sys.argv[3]) if len(sys.argv) > 3 else 100
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h, rows = rows[0], rows[1:]
iid, ik, im, iv, iu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0}
per = {}
for r in rows:
    if "k_pass_tc" not in r[ik]:
        continue
    per.setdefault(int(r[iid]), {})[r[im]] = float(r[iv].replace(",", "")) * mult.get(r[iu], 1)
ids = sorted(per)[-k:]
rd = sum(per[i]["dram__bytes_read.sum"] for i in ids) / len(ids)
wr = sum(per[i]["dram__bytes_write.sum"] for i in ids) / len(ids)
ms = sum(per[i]["gpu__time_duration.sum"] for i in ids)
spec = config_spec("C4")
alg = alg_qrcp_bytes(spec.m, spec.n, k, 2) / k
out = os.path.join(ROOT, "profiles", "pass_traffic.json")
pt = json.load(open(out))
pt.setdefault("kernels", {})["k_pass_tc"] = {
    "workload": "C4", "nb": 16, "source": f"{path} -> {src}",
    "dram_bytes_per_launch": rd + wr, "read_bytes_per_launch": rd, "write_bytes_per_launch": wr,
    "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
    "ncu_time_ms_per_id": ms, "launches": len(ids)}
json.dump(pt, open(out, "w"), indent=1)
print(json.dumps(pt["kernels"]["k_pass_tc"], indent=1))
