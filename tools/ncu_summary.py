"""Summarise an ncu report (run here, no GPU): key SOL / memory / issue metrics per launch.
usage: python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/x.txt"""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu summary of {path}")
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"\n## launch {d.get('ID')} {d.get('Kernel Name', '')[:100]}")
        for k in KEYS:
            if k in d and d[k] != "":
                print(f"  {k:75s} {d[k]} {u.get(k, '')}")
        try:
            t = float(d["gpu__time_duration.sum"])
            tu = u["gpu__time_duration.sum"]
            scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(tu, 1e-9)
            byt = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v = float(d[k]); uu = u[k]
                byt += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uu, 1)
            print(f"  => dram bytes {byt:.4g} B, {byt / (t * scale) / 1e9:.1f} GB/s over {t} {tu}")
        except Exception:
            pass


if __name__ == "__main__":
    main(sys.argv[1])
