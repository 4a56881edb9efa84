"""Thin Python binding of libmpid.so (include/mpid.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; PyTorch is used
for device memory (the workspace, A_D, outputs) and the CUDA stream.  There is
no CPU fallback: if libmpid.so is missing or cannot be loaded this module
raises at import of `lib()`.

The module-level functions carry the C names (id_create, id_qrcp_lowprec,
id_coeffs_fp64, id_error, ...); `MPID` is a convenience wrapper used by the
tests and bench.py.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MPID_LIB = another in-tree build of the library (A/B measurements of two builds)
LIB_PATH = os.path.join(HERE, os.environ.get("MPID_LIB", "libmpid.so"))

ID_FP16, ID_FP32, ID_FP64 = 1, 2, 3
ID_SCALE_NONE, ID_SCALE_MAXABS, ID_SCALE_POW2 = 0, 1, 2
ID_COEF_R, ID_COEF_LSQ = 0, 1
STATUS = {0: "OK", 1: "ARG", 2: "DIM", 3: "OVERFLOW", 4: "UNDERFLOW", 5: "DEGENERATE",
          6: "DOMAIN", 7: "CUDA", 8: "NCCL", 9: "OOM", 10: "STATE"}
FMT = {"fp16": ID_FP16, "fp32": ID_FP32, "fp64": ID_FP64}
SCALING = {"none": ID_SCALE_NONE, "maxabs": ID_SCALE_MAXABS, "pow2": ID_SCALE_POW2}
COEF = {"R": ID_COEF_R, "r": ID_COEF_R, "lsq": ID_COEF_LSQ, "LSQ": ID_COEF_LSQ}

# every function declared in include/mpid.h
EXPORTS = ["id_workspace_bytes", "id_create", "id_create_ex", "id_qrcp_lowprec", "id_coeffs_fp64", "id_error", "id_error_ex", "id_set_fp64_engine",
           "id_get_R", "id_get_R_fp64", "id_get_gram", "id_get_sketch", "id_get_perm", "id_get_AL", "id_round_only", "id_get_stats", "id_last_error", "id_destroy",
           "id_nccl_unique_id_bytes", "id_nccl_get_unique_id", "id_nccl_comm_init",
           "id_nccl_comm_destroy", "id_loopback_create", "id_loopback_calls", "id_loopback_destroy", "id_version"]


class IDError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"ID_ERR_{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class QRCPOpts(C.Structure):
    _fields_ = [("nb", C.c_int32), ("use_graph", C.c_int32), ("profile_pass", C.c_int32),
                ("formation", C.c_int32), ("sketch_oversample", C.c_int32), ("sketch_seed", C.c_int32),
                ("reserved", C.c_int32 * 2)]


class Stats(C.Structure):
    _fields_ = [("scale", C.c_double), ("normAL_fro", C.c_double), ("normAD_fro", C.c_double),
                ("resid_est", C.c_double), ("t_round_ms", C.c_double), ("t_qrcp_ms", C.c_double),
                ("t_coef_ms", C.c_double), ("t_err_ms", C.c_double), ("t_pass_ms", C.c_double),
                ("pass_launches", C.c_int64), ("kernel_launches", C.c_int64), ("k_out", C.c_int32),
                ("nb", C.c_int32), ("status_qrcp", C.c_int32), ("formation", C.c_int32),
                ("lsq_path", C.c_int32), ("fp64_engine", C.c_int32), ("fp64_engine_err", C.c_int32),
                ("reserved", C.c_int32 * 1), ("t_host_launch_ms", C.c_double),
                ("t_call_gpu_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


_LIB = None


def lib():
    """Load libmpid.so (raises OSError/RuntimeError when it is missing — no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2012_00706_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.id_workspace_bytes.restype = C.c_size_t
    L.id_workspace_bytes.argtypes = [i64, i64, i32, i32, C.c_int, i32]
    L.id_create.restype = C.c_int
    L.id_create.argtypes = [C.POINTER(vp), vp, i64, i64, i64, i64, i64, vp, C.c_size_t, vp, i32, i32, vp]
    L.id_create_ex.restype = C.c_int
    L.id_create_ex.argtypes = [C.POINTER(vp), vp, i64, i64, i64, i64, i64, vp, C.c_size_t, vp, i32, i32, vp, i32]
    L.id_qrcp_lowprec.restype = C.c_int
    L.id_qrcp_lowprec.argtypes = [vp, C.c_int, C.c_int, i32, dbl, C.POINTER(QRCPOpts),
                                  C.POINTER(i32), C.POINTER(i32)]
    L.id_coeffs_fp64.restype = C.c_int
    L.id_coeffs_fp64.argtypes = [vp, C.c_int, vp, i64]
    L.id_error.restype = C.c_int
    L.id_error.argtypes = [vp, C.POINTER(dbl), C.POINTER(dbl)]
    L.id_error_ex.restype = C.c_int
    L.id_set_fp64_engine.restype = C.c_int
    L.id_set_fp64_engine.argtypes = [vp, i32]
    L.id_error_ex.argtypes = [vp, i32, i32, i32, C.POINTER(dbl), C.POINTER(dbl)]
    L.id_get_R.restype = C.c_int
    L.id_get_R.argtypes = [vp, vp, i64]
    L.id_get_R_fp64.restype = C.c_int
    L.id_get_R_fp64.argtypes = [vp, vp, i64]
    L.id_get_gram.restype = C.c_int
    L.id_get_gram.argtypes = [vp, vp, i64]
    L.id_get_sketch.restype = C.c_int
    L.id_get_sketch.argtypes = [vp, vp, i64, C.POINTER(i32)]
    L.id_get_perm.restype = C.c_int
    L.id_get_perm.argtypes = [vp, C.POINTER(i32)]
    L.id_get_AL.restype = C.c_int
    L.id_get_AL.argtypes = [vp, vp, i64]
    L.id_round_only.restype = C.c_int
    L.id_round_only.argtypes = [vp, C.c_int, C.c_int]
    L.id_get_stats.restype = C.c_int
    L.id_get_stats.argtypes = [vp, C.POINTER(Stats)]
    L.id_last_error.restype = C.c_char_p
    L.id_last_error.argtypes = [vp]
    L.id_destroy.restype = None
    L.id_destroy.argtypes = [vp]
    L.id_nccl_unique_id_bytes.restype = i32
    L.id_nccl_unique_id_bytes.argtypes = []
    L.id_nccl_get_unique_id.restype = C.c_int
    L.id_nccl_get_unique_id.argtypes = [vp]
    L.id_nccl_comm_init.restype = C.c_int
    L.id_nccl_comm_init.argtypes = [C.POINTER(vp), vp, i32, i32]
    L.id_nccl_comm_destroy.restype = C.c_int
    L.id_nccl_comm_destroy.argtypes = [vp]
    L.id_loopback_create.restype = C.c_int
    L.id_loopback_create.argtypes = [C.POINTER(vp), i32]
    L.id_loopback_calls.restype = i64
    L.id_loopback_calls.argtypes = [vp]
    L.id_loopback_destroy.restype = None
    L.id_loopback_destroy.argtypes = [vp]
    L.id_version.restype = C.c_char_p
    L.id_version.argtypes = []
    _LIB = L
    return L


# ---------------------------------------------------------------------------
# C-named functions (marshalling only)
# ---------------------------------------------------------------------------
def id_workspace_bytes(m_local, n, k_max, nb=0, fmt=ID_FP16, host_AD=0) -> int:
    return int(lib().id_workspace_bytes(m_local, n, k_max, nb, fmt, host_AD))


def id_create(A_ptr, m_global, m_local, row_offset, n, ld, ws_ptr, ws_bytes, comm=None, rank=0,
              nranks=1, stream=None, flags=0):
    h = C.c_void_p()
    rc = lib().id_create_ex(C.byref(h), C.c_void_p(A_ptr), m_global, m_local, row_offset, n, ld,
                            C.c_void_p(ws_ptr), ws_bytes, C.c_void_p(comm) if comm else None, rank,
                            nranks, C.c_void_p(stream) if stream else None, flags)
    return rc, h


def id_qrcp_lowprec(h, fmt, scaling, k_max, eps=0.0, opts: QRCPOpts | None = None):
    k_out = C.c_int32(0)
    piv = (C.c_int32 * max(1, k_max))()
    rc = lib().id_qrcp_lowprec(h, fmt, scaling, k_max, eps, C.byref(opts) if opts else None,
                               C.byref(k_out), piv)
    return rc, k_out.value, np.frombuffer(piv, dtype=np.int32)[: k_out.value].copy()


def id_coeffs_fp64(h, mode, P_ptr, ldp):
    return lib().id_coeffs_fp64(h, mode, C.c_void_p(P_ptr), ldp)


def id_error(h):
    a, r = C.c_double(0), C.c_double(0)
    rc = lib().id_error(h, C.byref(a), C.byref(r))
    return rc, a.value, r.value


def id_last_error(h) -> str:
    s = lib().id_last_error(h)
    return s.decode() if s else ""


def id_destroy(h):
    lib().id_destroy(h)


def id_nccl_get_unique_id() -> bytes:
    buf = C.create_string_buffer(lib().id_nccl_unique_id_bytes())
    rc = lib().id_nccl_get_unique_id(buf)
    if rc:
        raise IDError(rc, "ncclGetUniqueId failed")
    return buf.raw


def id_nccl_comm_init(uid: bytes, nranks: int, rank: int) -> int:
    comm = C.c_void_p()
    buf = C.create_string_buffer(uid, len(uid))
    rc = lib().id_nccl_comm_init(C.byref(comm), buf, nranks, rank)
    if rc:
        raise IDError(rc, "ncclCommInitRank failed")
    return comm.value


def id_nccl_comm_destroy(comm: int):
    lib().id_nccl_comm_destroy(C.c_void_p(comm))


def id_loopback_create(nranks: int) -> int:
    comm = C.c_void_p()
    rc = lib().id_loopback_create(C.byref(comm), nranks)
    if rc:
        raise IDError(rc, "id_loopback_create failed")
    return comm.value


def id_loopback_calls(comm: int) -> int:
    return int(lib().id_loopback_calls(C.c_void_p(comm)))


def id_loopback_destroy(comm: int):
    lib().id_loopback_destroy(C.c_void_p(comm))


# ---------------------------------------------------------------------------
# convenience wrapper (torch for memory and stream)
# ---------------------------------------------------------------------------
@dataclass
class QRCPOut:
    k: int
    piv: np.ndarray
    status: int


class MPID:
    """One handle over a (shard of a) column-major fp64 matrix A_D.

    A_D: torch.float64 tensor of shape (n, m_local), contiguous — i.e. the
    column-major storage of the m_local x n shard — on the GPU, or a (pinned)
    CPU tensor for the host-buffer path (the library copies it in).
    """

    def __init__(self, A_D, k_max: int, m_global: int | None = None, row_offset: int = 0,
                 comm: int | None = None, rank: int = 0, nranks: int = 1, stream=None,
                 device=None, fp64: bool = False, stream_host: bool = False, stream_rows_log2: int = 0):
        """fp64=True sizes the workspace for the double ID too (fmt "fp64"); stream_host=True
        streams a host A_D in row blocks (id_create_ex ID_CREATE_STREAM_HOST) instead of
        copying it whole."""
        import torch
        assert A_D.dtype == torch.float64 and A_D.dim() == 2 and A_D.is_contiguous()
        n, m_local = A_D.shape
        self.n, self.m_local = int(n), int(m_local)
        self.m_global = int(m_global if m_global is not None else m_local)
        self.k_max = int(k_max)
        self.device = torch.device(device) if device is not None else (
            A_D.device if A_D.is_cuda else torch.device("cuda", torch.cuda.current_device()))
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        host = 0 if A_D.is_cuda else (2 if stream_host else 1)
        self.ws_bytes = id_workspace_bytes(self.m_local, self.n, self.k_max, 0, ID_FP64 if fp64 else ID_FP32,
                                           host)
        self.ws = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        self.ws_ptr = (base + 255) // 256 * 256
        self.A_D = A_D
        rc, h = id_create(A_D.data_ptr(), self.m_global, self.m_local, row_offset, self.n, self.m_local,
                          self.ws_ptr, self.ws_bytes, comm, rank, nranks, self.stream.cuda_stream,
                          flags=(1 | (stream_rows_log2 << 8)) if (host == 2) else 0)
        if rc:
            raise IDError(rc, "id_create failed")
        self.h = h
        self.k = 0

    def close(self):
        if getattr(self, "h", None):
            id_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, allow=()):
        if rc and rc not in allow:
            raise IDError(rc, id_last_error(self.h))
        return rc

    def qrcp(self, fmt="fp16", scaling="pow2", k=None, eps=0.0, nb=0, use_graph=True,
             profile=False, allow_underflow=False, formation=0, oversample=0, seed=0) -> QRCPOut:
        """formation: 0 auto, 1 / "ffma" CUDA-core FFMA, 2 / "tc" tcgen05, 3 / "gram" Gram pivoting (include/mpid.h)."""
        formation = {"auto": 0, "ffma": 1, "tc": 2, "gram": 3, "sketch": 4, "smem": 5, "coop": 6}.get(formation, formation)
        o = QRCPOpts(nb=nb, use_graph=1 if use_graph else -1, profile_pass=1 if profile else 0,
                     formation=formation, sketch_oversample=oversample, sketch_seed=seed)
        k = self.k_max if k is None else k
        rc, kout, piv = id_qrcp_lowprec(self.h, FMT[fmt] if isinstance(fmt, str) else fmt,
                                        SCALING[scaling] if isinstance(scaling, str) else scaling,
                                        k, eps, o)
        self._check(rc, allow=(4,) if allow_underflow else ())
        self.k = kout
        self.fmt = fmt
        return QRCPOut(kout, piv, rc)

    def round_only(self, fmt="fp16", scaling="pow2"):
        self._check(lib().id_round_only(self.h, FMT[fmt], SCALING[scaling]))
        self.fmt = fmt

    def coeffs(self, mode="lsq"):
        """P as a torch (k, n) fp64 view of column-major device storage."""
        import torch
        Pt = torch.empty((self.n, self.k), dtype=torch.float64, device=self.device)
        self._check(id_coeffs_fp64(self.h, COEF[mode], Pt.data_ptr(), self.k))
        return Pt.t()

    def set_fp64_engine(self, engine):
        """fp64 GEMM engine of coeffs / error (include/mpid.h id_set_fp64_engine): "auto",
        "dmma" or "int8" (the Ozaki scheme on the int8 tensor cores)."""
        e = {"auto": 0, "dmma": 1, "int8": 2, "ozaki": 2}[engine] if isinstance(engine, str) else int(engine)
        self._check(lib().id_set_fp64_engine(self.h, e))

    def error(self):
        rc, a, r = id_error(self.h)
        self._check(rc)
        return a, r

    def error_ex(self, skeleton="AD", norm="fro", iters=0):
        """Variant / metric of the paper (include/mpid.h id_error_ex): skeleton "AD" (mixed
        ID) or "AL" (low-precision skeleton); norm "fro" or 2 (power iteration)."""
        a, r = C.c_double(0), C.c_double(0)
        sk = {"AD": 0, "AL": 1}[skeleton] if isinstance(skeleton, str) else int(skeleton)
        nm = 0 if norm in ("fro", 0) else 2
        self._check(lib().id_error_ex(self.h, sk, nm, iters, C.byref(a), C.byref(r)))
        return a.value, r.value

    def get_R(self):
        import torch
        Rt = torch.empty((self.n, self.k), dtype=torch.float32, device=self.device)
        self._check(lib().id_get_R(self.h, C.c_void_p(Rt.data_ptr()), self.k))
        return Rt.t()

    def get_gram(self):
        import torch
        G = torch.empty((self.n, self.n), dtype=torch.float64, device=self.device)
        self._check(lib().id_get_gram(self.h, C.c_void_p(G.data_ptr()), self.n))
        return G.t()

    def get_sketch(self):
        """(Y, l): the sketch Omega A_L as an l x n fp64 torch view of column-major storage."""
        import torch
        ld = self.k_max + 4096
        Yt = torch.empty((self.n, ld), dtype=torch.float64, device=self.device)
        lo = C.c_int32(0)
        self._check(lib().id_get_sketch(self.h, C.c_void_p(Yt.data_ptr()), ld, C.byref(lo)))
        return Yt[:, :lo.value].t(), lo.value

    def get_R64(self):
        import torch
        Rt = torch.empty((self.n, self.k), dtype=torch.float64, device=self.device)
        self._check(lib().id_get_R_fp64(self.h, C.c_void_p(Rt.data_ptr()), self.k))
        return Rt.t()

    def get_perm(self) -> np.ndarray:
        buf = (C.c_int32 * self.n)()
        self._check(lib().id_get_perm(self.h, buf))
        return np.frombuffer(buf, dtype=np.int32).copy()

    def get_AL(self):
        import torch
        dt = {"fp16": torch.float16, "fp32": torch.float32, "fp64": torch.float64}[self.fmt]
        out = torch.empty((self.n, self.m_local), dtype=dt, device=self.device)
        self._check(lib().id_get_AL(self.h, C.c_void_p(out.data_ptr()), self.m_local))
        return out.t()

    def stats(self) -> dict:
        s = Stats()
        self._check(lib().id_get_stats(self.h, C.byref(s)))
        return s.as_dict()
