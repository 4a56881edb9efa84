"""The oracle's QRCP (O4a, right-looking form) compiled from plain C — oracle/cqrcp.c.

TEST INFRASTRUCTURE ONLY (see oracle/rounding.py header): only tests/,
__graft_entry__ (build + smoke) and bench.py's cpu_baseline / --impl reference legs
may import it.  It exists so the oracle reaches the full-size configurations (C3,
the C4 / C5 row analogues, full C4) in seconds to a minute on the GPU box's host
cores; it is the same algorithm as `oracle.qrcp.qrcp_householder(formation="fma")`
step for step and is pinned to it bit for bit (tests/test_oracle_c.py).  Threads
only split the set of columns, so results do not depend on the thread count.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .qrcp import QRCPResult
from .rounding import fmt_of, DOUBLE, HALF

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cqrcp.c")
LIB = os.path.join(HERE, "libcqrcp.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp -ffp-contract=off: no fused multiply-add, no reassociation."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = ["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           SRC, "-o", LIB, "-lm"]
    subprocess.run(cmd, check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        L.oracle_qrcp.restype = ctypes.c_int
        L.oracle_qrcp.argtypes = [P(ctypes.c_double), ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                  P(ctypes.c_int32), P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double),
                                  P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_double),
                                  P(ctypes.c_double)]
        _lib = L
    return _lib


def qrcp_c(A_L: np.ndarray, k_max: int, fmt: str = "fp16", nb: int = 1, eps: float = 0.0,
           model: str = "paper", threads: int = 0) -> QRCPResult:
    """qrcp_householder(A_L, k_max, fmt, nb, eps, model=...) (formation "fma", one shard)
    in C.  model "paper" = update rne + acc seq64; "kernel" = update fma + acc chain8.
    V and tau are not returned (empty arrays)."""
    upd, acc = {"paper": (1, 1), "kernel": (0, 0)}[model]
    f = fmt_of(fmt)
    code = 64 if f is DOUBLE else (16 if f is HALF else 32)
    A = np.asfortranarray(np.asarray(A_L, dtype=np.float64))
    m, n = A.shape
    if not (1 <= k_max <= min(m, n)):
        raise ValueError("k out of range (DimensionError)")
    perm = np.zeros(n, np.int32)
    R = np.zeros((k_max, n))
    top2 = np.zeros((k_max, 2))
    resid = np.zeros(k_max + 1)
    rl, ko, st = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    nal, mx0 = ctypes.c_double(), ctypes.c_double()
    P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))
    rc = lib().oracle_qrcp(P(A, ctypes.c_double), m, n, k_max, code, nb, float(eps), upd, acc, threads,
                           P(perm, ctypes.c_int32), P(R, ctypes.c_double), P(top2, ctypes.c_double),
                           P(resid, ctypes.c_double), ctypes.byref(rl), ctypes.byref(ko), ctypes.byref(st),
                           ctypes.byref(nal), ctypes.byref(mx0))
    if rc != 0:
        raise ValueError("oracle_qrcp: bad arguments or out of memory")
    k = ko.value
    return QRCPResult(perm.astype(np.int64), R[:k].copy(), k, "ok" if st.value == 0 else "underflow",
                      np.zeros((m, 0)), np.zeros(0), top2[:k].copy(), mx0.value, nal.value,
                      resid[: rl.value].tolist())
