"""Build libmpid.so in-tree for sm_100a with nvcc (no torch extension machinery).

    python -m paper_2012_00706_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["mpid_api.cu", "k_round.cu", "k_qrcp.cu", "k_pass.cu", "k_pass_tc.cu", "k_qrcp_smem.cu", "k_fp64.cu", "k_norm2.cu", "k_gram.cu", "k_ozaki.cu", "k_qrcp_coop.cu"]
LIB = os.path.join(HERE, "libmpid.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "mpid_internal.cuh"),
                   os.path.join(os.path.dirname(HERE), "include", "mpid.h")]
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(s):
        o = os.path.join(CSRC, os.path.basename(s).replace(".cu", ".o"))
        r = subprocess.run([NVCC, *FLAGS, "-c", s, "-o", o], capture_output=True, text=True)
        return s, o, r

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        for s, o, r in ex.map(compile_one, srcs):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {s}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(o)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
           "-ldl", "-lcudart", "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
