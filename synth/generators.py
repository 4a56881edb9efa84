"""Seeded generators for A_D (fp64, column-major) — no arithmetic of the method here.

Workloads:
  * decay  — the paper's Slow/Medium/Fast datasets: A = U diag(sigma) V^T with
             sigma_i = i^-p, p = 1, 2, 4 (Table 3), U, V Haar.
  * C1     — 256x128, sigma_j = 10^(-(j-1)/8)            (BASELINE.json configs[0])
  * C2     — 4096x1024, sigma_j = j^-2, + N(0, std 1e-8)  (configs[1]; reading R9: std)
  * C3     — 65536x2048, rank-300 factor sigma_j = exp(-j/30)
             + N(0, std 1e-6 ||A_clean||_F / sqrt(mn))   (configs[2])
  * C4/C5  — traveling Fourier-mode "turbulent snapshot" matrices (configs[3], [4]):
             rows = N^3 grid points, columns = time snapshots,
             A(x,t) = sum_l a_l cos(kappa_l . x - omega_l t + phi_l), a_l = sqrt(2 E_l),
             E_l = |kappa_l|^(-5/3), + 1e-4 relative Gaussian noise.  This stands in
             for the paper's particle-velocity data, which is not available.
  * planted — S = Q_k diag(rho^-(j-1)), A = [S, S C] + eta N, columns permuted
             (a spectral gap at k by construction; pivots known in closed form).
  * exact   — A = X Y^T, rank exactly k.

Haar factors use numpy's PCG64 `default_rng(seed)`; the additive noise uses a
counter-based generator keyed by (seed, stream, global row, global column) so
that any row shard of a matrix reproduces the same entries (reading
on sharding).  The same counter generator is implemented for numpy and torch.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# counter-based normal generator (SplitMix64 + Box-Muller)
# ----------------------------------------------------------------------------
_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def _s64(c: int) -> int:
    """Unsigned 64-bit constant as the equal-bits signed int64 (for torch)."""
    return c - (1 << 64) if c >= (1 << 63) else c


def _splitmix_np(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(_GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def _lsr_t(z, s: int):
    import torch  # noqa: F401
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix_t(z):
    z = z + _s64(_GOLDEN)
    z = (z ^ _lsr_t(z, 30)) * _s64(_M1)
    z = (z ^ _lsr_t(z, 27)) * _s64(_M2)
    return z ^ _lsr_t(z, 31)


def _stream_base(seed: int, stream: int) -> int:
    z = np.array([(seed * 1000003 + stream * 7919 + 12345) & _MASK64], dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(_splitmix_np(z)[0])


def counter_normal(seed: int, stream: int, rows, cols, device=None):
    """N(0,1) samples G[r, c] for global row indices `rows` and column indices `cols`.

    Returns an array of shape (len(cols), len(rows)) — i.e. column-major storage
    of the len(rows) x len(cols) block (each column contiguous).  With
    device=None a numpy array is returned, else a torch tensor on `device`.
    """
    base = _stream_base(seed, stream)
    if device is None:
        r = np.asarray(rows, dtype=np.uint64)[None, :]
        c = np.asarray(cols, dtype=np.uint64)[:, None]
        ctr = (r << np.uint64(13)) | c                      # cols < 8192, rows < 2^40
        with np.errstate(over="ignore"):
            z1 = _splitmix_np(np.uint64(base) + (ctr << np.uint64(1)))
            z2 = _splitmix_np(np.uint64(base) + (ctr << np.uint64(1)) + np.uint64(1))
        u1 = ((z1 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
        u2 = (z2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    import torch
    r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=device)[None, :]
    c = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=device)[:, None]
    ctr = (r << 13) | c
    b = _s64(base)
    z1 = _splitmix_t(b + (ctr << 1))
    z2 = _splitmix_t(b + (ctr << 1) + 1)
    u1 = (_lsr_t(z1, 11).to(torch.float64) + 1.0) * 2.0 ** -53
    u2 = _lsr_t(z2, 11).to(torch.float64) * 2.0 ** -53
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def counter_sign(seed: int, stream: int, rows, cols) -> np.ndarray:
    """Rademacher signs +-1 (int8) for global row indices `rows` and column indices
    `cols`: the top bit of SplitMix64(base + ((r << 13) | c)) selects -1.  Shape
    (len(cols), len(rows)).  The GPU's sketch kernel implements the same counter-based
    generator (random numbers the method draws are reproduced, not shared)."""
    base = _stream_base(seed, stream)
    r = np.asarray(rows, dtype=np.uint64)[None, :]
    c = np.asarray(cols, dtype=np.uint64)[:, None]
    ctr = (r << np.uint64(13)) | c
    with np.errstate(over="ignore"):
        z = _splitmix_np(np.uint64(base) + ctr)
    return np.where((z >> np.uint64(63)) != 0, -1, 1).astype(np.int8)


SKETCH_STREAM = 7


# ----------------------------------------------------------------------------
# Haar factors, decay matrices
# ----------------------------------------------------------------------------
def haar(rng: np.random.Generator, m: int, r: int) -> np.ndarray:
    """m x r with orthonormal columns: QR of an iid N(0,1) matrix, diag(R) > 0."""
    G = rng.standard_normal((m, r))
    Q, R = np.linalg.qr(G)
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return Q * d[None, :]


def _usv(rng, m, n, sigma):
    r = len(sigma)
    U = haar(rng, m, r)
    V = haar(rng, n, r)
    return np.asfortranarray((U * sigma[None, :]) @ V.T), U, V


def gen_decay(p: float, m: int = 1000, n: int = 1000, seed: int = 0):
    """The paper's Slow/Medium/Fast datasets, sigma_i = i^-p."""
    rng = np.random.default_rng([seed, 101])
    sigma = np.arange(1, min(m, n) + 1, dtype=np.float64) ** (-float(p))
    A, _, _ = _usv(rng, m, n, sigma)
    return A, sigma


def _noise(seed, stream, m, n, row0=0, device=None):
    return counter_normal(seed, stream, np.arange(row0, row0 + m), np.arange(n), device)


# ----------------------------------------------------------------------------
# Fourier-mode snapshot matrices (C4, C5)
# ----------------------------------------------------------------------------
@dataclass
class FourierParams:
    N: int
    L: int
    n: int
    kappa: np.ndarray      # (L, 3) int64
    amp: np.ndarray        # (L,)  a_l = sqrt(2 |kappa|^(-5/3))
    phi: np.ndarray        # (L,)
    omega: np.ndarray      # (L,)
    noise_rel: float = 1e-4

    @property
    def m(self) -> int:
        return self.N ** 3

    @property
    def clean_fro2(self) -> float:
        """||A_clean||_F^2 = (m/2) n sum a_l^2 (discrete orthogonality of distinct lattice modes)."""
        return 0.5 * self.m * self.n * float(np.sum(self.amp ** 2))

    @property
    def noise_std(self) -> float:
        return self.noise_rel * math.sqrt(self.clean_fro2 / (self.m * self.n))


def fourier_params(N: int, L: int, n: int, seed: int) -> FourierParams:
    rng = np.random.default_rng([seed, 404, N, L])
    ks, seen = [], set()
    while len(ks) < L:
        mag = math.exp(rng.uniform(0.0, math.log(N / 4)))
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        kv = tuple(int(x) for x in np.rint(mag * d))
        if kv == (0, 0, 0) or any(abs(x) >= N // 2 for x in kv):
            continue
        neg = tuple(-x for x in kv)
        if kv in seen or neg in seen:
            continue
        seen.add(kv)
        ks.append(kv)
    kappa = np.array(ks, dtype=np.int64)
    kn = np.linalg.norm(kappa.astype(np.float64), axis=1)
    amp = np.sqrt(2.0 * kn ** (-5.0 / 3.0))
    phi = rng.uniform(0.0, 2 * math.pi, L)
    omega = rng.uniform(0.0, math.pi, L)
    return FourierParams(N, L, n, kappa, amp, phi, omega)


def gen_fourier(fp: FourierParams, seed: int, row0: int = 0, m_loc: int | None = None,
                device=None, noise: bool = True, col_chunk: int = 128):
    """Rows [row0, row0+m_loc) of the Fourier snapshot matrix, column-major.

    numpy (device=None): returns an (m_loc, n) Fortran-ordered float64 array.
    torch (device given): returns a contiguous (n, m_loc) float64 tensor, i.e.
    the column-major storage of the m_loc x n shard.
    """
    N = fp.N
    m_loc = fp.m - row0 if m_loc is None else m_loc
    rows = np.arange(row0, row0 + m_loc, dtype=np.int64)
    i1, i2, i3 = rows % N, (rows // N) % N, rows // (N * N)
    t = np.arange(fp.n, dtype=np.float64)
    if device is None:
        ph = (np.outer(i1, fp.kappa[:, 0]) + np.outer(i2, fp.kappa[:, 1])
              + np.outer(i3, fp.kappa[:, 2])) % N                       # exact integers
        theta = 2 * math.pi * ph.astype(np.float64) / N + fp.phi[None, :]
        X = np.concatenate([np.cos(theta) * fp.amp, np.sin(theta) * fp.amp], axis=1)
        T = np.concatenate([np.cos(np.outer(fp.omega, t)), np.sin(np.outer(fp.omega, t))], axis=0)
        A = np.asfortranarray(X @ T)
        if noise:
            for c0 in range(0, fp.n, col_chunk):
                c1 = min(fp.n, c0 + col_chunk)
                A[:, c0:c1] += fp.noise_std * counter_normal(seed, 5, rows, np.arange(c0, c1)).T
        return A
    import torch
    dev = torch.device(device)
    i1t, i2t, i3t = (torch.as_tensor(v, device=dev) for v in (i1, i2, i3))
    kap = torch.as_tensor(fp.kappa, device=dev)
    ph = (i1t[:, None] * kap[None, :, 0] + i2t[:, None] * kap[None, :, 1]
          + i3t[:, None] * kap[None, :, 2]) % N
    theta = 2 * math.pi * ph.to(torch.float64) / N + torch.as_tensor(fp.phi, device=dev)[None, :]
    amp = torch.as_tensor(fp.amp, device=dev)
    X = torch.cat([torch.cos(theta) * amp, torch.sin(theta) * amp], dim=1)      # m_loc x 2L
    del theta, ph
    wt = torch.outer(torch.as_tensor(fp.omega, device=dev), torch.as_tensor(t, device=dev))
    T = torch.cat([torch.cos(wt), torch.sin(wt)], dim=0)                      # 2L x n
    At = torch.empty((fp.n, m_loc), dtype=torch.float64, device=dev)          # col-major storage
    for c0 in range(0, fp.n, col_chunk):
        c1 = min(fp.n, c0 + col_chunk)
        blk = (X @ T[:, c0:c1]).T                                              # (c1-c0) x m_loc
        if noise:
            blk = blk + fp.noise_std * counter_normal(seed, 5, rows, np.arange(c0, c1), dev)
        At[c0:c1] = blk
    return At


# ----------------------------------------------------------------------------
# planted skeleton and exact rank
# ----------------------------------------------------------------------------
def gen_planted(m: int, n: int, k: int, rho: float, eta: float, seed: int, c_max=None):
    """A = [S, S C] Pi + eta N with S = Q_k diag(rho^-(j-1)).

    Returns (A, skel, C): skel[j] = position of the j-th planted column after the
    column permutation (the expected pivot order), C the k x (n-k) coefficients.
    """
    rng = np.random.default_rng([seed, 606, m, n, k])
    Q = haar(rng, m, k)
    s = rho ** (-np.arange(k, dtype=np.float64))
    S = Q * s[None, :]
    c = 0.5 * math.sqrt(1.0 - rho ** -2) if c_max is None else c_max
    C = rng.uniform(-c, c, size=(k, n - k))
    B = np.concatenate([S, S @ C], axis=1)
    pi = rng.permutation(n)                # column pi[i] of A is column i of B
    A = np.empty_like(B)
    A[:, pi] = B
    if eta > 0:
        A += eta * counter_normal(seed, 6, np.arange(m), np.arange(n)).T
    return np.asfortranarray(A), pi[:k].copy(), C


def gen_exact_rank(m: int, n: int, k: int, seed: int):
    rng = np.random.default_rng([seed, 707, m, n, k])
    X = rng.standard_normal((m, k))
    Y = rng.standard_normal((n, k))
    return np.asfortranarray(X @ Y.T)


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------
@dataclass
class ConfigSpec:
    name: str
    m: int
    n: int
    ks: tuple
    fmts: tuple
    scaling: dict          # fmt -> "none" | "maxabs" | "pow2"
    nb: int = 0            # 0 = library default
    eps: float = 0.0
    desc: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "C1": ConfigSpec("C1", 256, 128, (32,), ("fp16", "fp32"), {"fp16": "pow2", "fp32": "none"},
                     desc="256x128 Haar U,V, sigma_j = 10^-(j-1)/8, k=32 (configs[0])"),
    "C2": ConfigSpec("C2", 4096, 1024, (16, 64, 128), ("fp32", "fp16"), {"fp16": "maxabs", "fp32": "none"},
                     desc="4096x1024 Haar U,V, sigma_j = j^-2 + N(0,1e-8) (configs[1])"),
    "C3": ConfigSpec("C3", 65536, 2048, (256,), ("fp16",), {"fp16": "pow2"}, eps=1e-3,
                     desc="65536x2048 rank-300 exp(-j/30) + 1e-6 rel noise; k=256 or eps=1e-3 (configs[2])"),
    "C4": ConfigSpec("C4", 128 ** 3, 1024, (100,), ("fp16", "fp32"), {"fp16": "pow2", "fp32": "none"},
                     desc="128^3 x 1024 Fourier snapshots, 64 modes, k=100 (configs[3])",
                     extra={"N": 128, "L": 64}),
    "C5": ConfigSpec("C5", 256 ** 3, 2048, (512,), ("fp16",), {"fp16": "pow2"},
                     desc="256^3 x 2048 Fourier snapshots, 256 modes, k=512, row-sharded (configs[4])",
                     extra={"N": 256, "L": 256}),
}


def config_spec(name: str) -> ConfigSpec:
    return CONFIGS[name]


def gen_config(name: str, seed: int = 0, row0: int = 0, m_loc: int | None = None, device=None):
    """A_D for config `name` (rows [row0, row0+m_loc) for the sharded C4/C5)."""
    if name == "C1":
        rng = np.random.default_rng([seed, 1])
        sigma = 10.0 ** (-np.arange(128, dtype=np.float64) / 8.0)
        A, _, _ = _usv(rng, 256, 128, sigma)
        return A
    if name == "C2":
        rng = np.random.default_rng([seed, 2])
        sigma = np.arange(1, 1025, dtype=np.float64) ** -2.0
        A, _, _ = _usv(rng, 4096, 1024, sigma)
        A += 1e-8 * _noise(seed, 2, 4096, 1024).T
        return A
    if name == "C3":
        rng = np.random.default_rng([seed, 3])
        m, n = 65536, 2048
        sigma = np.exp(-np.arange(1, 301, dtype=np.float64) / 30.0)
        A, _, _ = _usv(rng, m, n, sigma)
        std = 1e-6 * math.sqrt(float(np.sum(sigma ** 2))) / math.sqrt(m * n)
        for c0 in range(0, n, 256):
            A[:, c0:c0 + 256] += std * counter_normal(seed, 3, np.arange(m), np.arange(c0, c0 + 256)).T
        return A
    if name in ("C4", "C5"):
        spec = CONFIGS[name]
        fp = fourier_params(spec.extra["N"], spec.extra["L"], spec.n, seed)
        return gen_fourier(fp, seed, row0, m_loc, device)
    raise KeyError(name)
