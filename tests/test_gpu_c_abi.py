"""The boundary is a plain C ABI: examples/id_c_example.c (no Python, no PyTorch) is
compiled with gcc against include/mpid.h and libmpid.so and runs one ID on the GPU
(an exact-rank-24 matrix, k = 24: the error must vanish)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_program_runs_an_id(tmp_path):
    exe = tmp_path / "id_c_example"
    cmd = ["gcc", "-O2", os.path.join(ROOT, "examples", "id_c_example.c"), "-I" + os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", "-L" + os.path.join(ROOT, "paper_2012_00706_b200"), "-lmpid",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + os.path.join(ROOT, "paper_2012_00706_b200"),
           "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "k_out = 24" in r.stdout
    rel = float(r.stdout.split("relative Frobenius error =")[1].split()[0])
    assert rel < 1e-6
