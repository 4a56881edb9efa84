"""Write profiles/pass_traffic.json from an ncu --set full capture of k_pass_ws launches.
usage: python tools/traffic_from_ncu.py gpurun_out/prof.ncu-rep <m> <n> <j of first launch> <fmt bytes>"""
import csv, io, json, subprocess, sys

path, m, n, j0, s = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = []
for i, r in enumerate(rows[2:]):
    d = dict(zip(h, r)); uu = dict(zip(h, u))
    if "k_pass" not in d.get("Kernel Name", ""):
        continue
    byt = sum(float(d[k]) * mult[uu[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    j = j0 + len(launches)
    alg = (m - j) * (n - j) * s
    launches.append({"kernel": d["Kernel Name"][:60], "step_j": j, "dram_bytes": byt,
                     "algorithmic_read_bytes": alg, "ratio": byt / alg})
res = {"source": path, "bytes_per_launch": launches[0]["dram_bytes"], "launches": launches,
       "note": "ncu --set full (cold cache, serialised) of non-store steps of the C4 workload; "
               "traffic / algorithmic read bytes ~ 1.0 means no re-reads"}
json.dump(res, open("profiles/pass_traffic.json", "w"), indent=1)
print(json.dumps(res, indent=1))
