"""One-off probe of the GPU box: host cores/RAM, fp64 GEMM rate, HBM copy, PCIe H2D."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["lscpu"] = subprocess.run(["bash", "-c", "lscpu | grep -E 'Model name|^CPU\\(s\\)|Thread|Socket|NUMA node\\(s\\)'"], capture_output=True, text=True).stdout
out["mem"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,clocks.max.sm,clocks.sm", "--format=csv"], capture_output=True, text=True).stdout
p = torch.cuda.get_device_properties(0)
out["sm"] = p.multi_processor_count; out["l2"] = p.L2_cache_size; out["totmem"] = p.total_memory
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(it):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for N in (4096, 8192):
    a = torch.randn(N, N, dtype=torch.float64, device="cuda"); b = torch.randn(N, N, dtype=torch.float64, device="cuda")
    ms = t(lambda: a @ b, 5)
    out[f"dgemm_{N}_tflops"] = 2 * N**3 / ms / 1e9
a = torch.empty(2**30, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
ms = t(lambda: b.copy_(a))
out["copy_GBs"] = 2 * 2**30 / ms / 1e6
h = torch.empty(2**30, dtype=torch.uint8, pin_memory=True)
ms = t(lambda: a.copy_(h, non_blocking=True), 5); out["h2d_GBs"] = 2**30 / ms / 1e6
ms = t(lambda: h.copy_(a, non_blocking=True), 5); out["d2h_GBs"] = 2**30 / ms / 1e6
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
