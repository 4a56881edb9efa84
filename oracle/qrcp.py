"""O4 — rank-k column-pivoted QR in the paper's low precision, written plainly.

TEST INFRASTRUCTURE ONLY (see oracle/rounding.py header).  Never imported by
the product path; imports nothing from it.

What is computed:
  * Algorithm 2 line 2: A_L = fl(A) — done by the caller with
    `rounding.round_to`, optionally after range scaling (`scale_matrix`).
  * Algorithm 2 line 4 and Eq. (6)-(7): A Z = Q R, rank k,
    column pivoting on the largest remaining column norm.  The paper's QR is
    modified Gram-Schmidt; BASELINE.json's north_star asks for Householder.
    `qrcp_householder` is the Householder form (reading R3) and
    `qrcp_mgs` is the paper-literal MGS form of SPEC S:189-197, kept as an
    independent cross-check (same pivots and |R| in exact arithmetic).
  * Simulated low precision: values are "cast to half or single" but
    "accumulate error exclusively in single precision".  Precision model used by
    both this oracle and the CUDA path (readings R4-R6):
      - element arithmetic (the reflector update W <- W - v f^T) in fp32;
      - the working matrix is re-stored (rounded) to the low format every `nb`
        steps, after that step's pivot is chosen and before its reflector is
        formed — nb = 1 is SPEC's store-after-every-update, nb > 1 the blocked
        implementation the paper names as future work;
      - reductions over rows (column norms, W^T u): either ("chain8") fp32
        fused multiply-add chains over 8-row groups ("accumulate in single",
        P:209), the group partials added in fp64 (reading R5: sequential fp32
        sums stagnate at m = 2^24 rows), or ("seq64") the exact fp32 x fp32
        products added in fp64 in increasing row order — the plain definition
        of the sum, independent of any kernel's order;
      - the update W <- W - v f^T: "fma" one rounding per entry, or "rne" the
        paper's per-operation rounding (north_star "correct RNE after
        every op"): fl(W - fl(v f));
      - model="paper" = update "rne" + acc "seq64": the oracle the CUDA path is
        compared with by tolerance (DESIGN.md §2 R4b/R5, §Oracle); the "fma" +
        "chain8" model is kept as the round-1 regression model of the FFMA pass;
      - pivot norms: the exact norms of the trailing matrix formed at step j-1,
        downdated by one step (reading R6); the recompute-every-step form of
        SPEC S:215 is kept as a cross-check (norms="recompute");
      - ties broken toward the lowest original column index;
      - R rows normalised so that R_jj >= 0.
    fmt = "fp64" runs the same algorithm entirely in fp64 (Algorithm 1).
  * Tolerance-driven rank (reading R8; "||A - BC|| << eps"): stop before
    step j when sqrt(sum_{i>=j} ||W(j:m, i)||^2) <= eps * ||A_L||_F.
  * Underflow: status "underflow" when the selected pivot norm
    squared underflows the fp32 normal range or the pivot column is zero.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rounding import fmt_of, round_to, DOUBLE, SINGLE


@dataclass
class QRCPResult:
    perm: np.ndarray            # (n,) 0-based original column index at each position
    R: np.ndarray               # (k_out, n) float64 holding working-precision values, pivoted order
    k_out: int
    status: str                 # "ok" | "underflow"
    V: np.ndarray               # (m, k_out) Householder vectors (v_j = 1, zeros above)
    tau: np.ndarray             # (k_out,)
    top2: np.ndarray            # (k_out, 2) the two largest candidate norms at each step
    maxnorm0: float             # max_i ||A_L(:, i)|| (scale for tie certification)
    normAL: float               # ||A_L||_F
    resid: list = field(default_factory=list)   # exact sqrt(sum of remaining norms^2) before each step (+ after the last)

    @property
    def I(self) -> np.ndarray:
        return self.perm[: self.k_out].copy()


def scale_factor(A_D: np.ndarray, scaling: str) -> float:
    """Range scaling s applied before rounding (BASELINE.json configs[1]; reading R7).

    "none": s = 1; "maxabs": s = 1/max|a_ij| (literal C2 text); "pow2":
    s = 2^-ceil(log2 max|a_ij|), an exact power of two.
    """
    if scaling == "none":
        return 1.0
    mx = float(np.max(np.abs(A_D)))
    if mx == 0.0:
        return 1.0
    if scaling == "maxabs":
        return 1.0 / mx
    if scaling == "pow2":
        return math.ldexp(1.0, -math.ceil(math.log2(mx)))
    raise ValueError(scaling)


def make_AL(A_D: np.ndarray, fmt: str, scaling: str = "none"):
    """A_L = fl_L(s * A_D) with a single RNE rounding from fp64 (reading R7)."""
    s = scale_factor(A_D, scaling)
    A_D = np.asarray(A_D, dtype=np.float64)
    if A_D.size <= (1 << 24):
        AL = round_to(A_D * s, fmt).reshape(A_D.shape)
        return np.asfortranarray(AL), s
    # large inputs: the same elementwise rounding, 16 columns at a time (bounded temporaries)
    AL = np.empty(A_D.shape, dtype=np.float64, order="F")
    for c0 in range(0, A_D.shape[1], 16):
        blk = A_D[:, c0:c0 + 16] * s
        AL[:, c0:c0 + 16] = round_to(blk, fmt).reshape(blk.shape)
    return AL, s


def _work_dtype(fmt):
    return np.float64 if fmt_of(fmt) is DOUBLE else np.float32


def _fma(a, b, c, wdt):
    """fl(a*b + c) with one rounding to the working precision (emulated: the
    product of two fp32 values is exact in fp64; reading R4b)."""
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(wdt)


def chain8(X: np.ndarray, Y: np.ndarray, wdt) -> np.ndarray:
    """Column sums of X*Y in the blocked order of reading R5: within each group of
    8 consecutive rows a working-precision FMA chain (p = x0*y0; p = fma(xi, yi, p)),
    then the group partials added in fp64.  X: (8G, c); Y: (8G, c) or (8G, 1)."""
    G = X.shape[0] // 8
    Xg = X.reshape(G, 8, -1)
    Yg = Y.reshape(G, 8, -1)
    acc = (Xg[:, 0].astype(np.float64) * Yg[:, 0].astype(np.float64)).astype(wdt)
    for i in range(1, 8):
        acc = _fma(Xg[:, i], Yg[:, i], acc, wdt)
    if G == 0:
        return np.zeros(X.shape[1])
    return np.add.accumulate(acc.astype(np.float64), axis=0)[-1].copy()


def seq64(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Column sums of X*Y: each product formed in fp64 (exact for fp32 / fp16 inputs) and
    the products added in fp64 in increasing row order (np.add.accumulate is a
    sequential running sum).  X: (r, c); Y: (r, c) or (r, 1)."""
    P = X.astype(np.float64) * Y.astype(np.float64)
    if P.shape[0] == 0:
        return np.zeros(P.shape[1])
    return np.add.accumulate(P, axis=0)[-1].copy()


def _sum1(x) -> float:
    """Sequential fp64 sum of a vector (first term first)."""
    x = np.asarray(x, dtype=np.float64)
    return float(np.add.accumulate(x)[-1]) if x.size else 0.0


class _Local:
    """Single-process 'communicator': the sum over ranks of one rank is itself."""
    rank, size = 0, 1

    @staticmethod
    def sum(x):
        return np.asarray(x, dtype=np.float64)


def qrcp_householder(A_L: np.ndarray, k_max: int, fmt: str = "fp16", nb: int = 1,
                     eps: float = 0.0, norms: str = "downdate", acc: str = "auto",
                     row_offset: int = 0, comm=None, formation: str = "fma",
                     update: str = "fma", model: str | None = None) -> QRCPResult:
    """Householder QRCP of the already-rounded A_L, in the precision model above.

    Step j (0-based), following Eq. (6)-(7):
      1. p = argmax vn_i over i >= j (ties: lowest original index); swap j <-> p   [pivot, Z]
         vn: initial exact column norms^2 of A_L; then (norms="downdate", reading
         R6 / SURVEY A2) the one-step downdate vn_i = s_i - R(j-1, i)^2 of the
         exact norms s of the previous step's trailing matrix; (norms="recompute")
         the exact norms of the current trailing matrix (cross-check).
      2. every nb steps (j > 0, j % nb == 0): W(j:, j:) <- fl_L(W(j:, j:))      [store point, R4]
      3. s_i = ||W(j:m, i)||^2, w = W(j:m, j:)^T u with u = W(j:m, j), summed in
         the order `acc` ("chain8": 8-row fp32 FMA chains + fp64, R5; "seq64":
         exact products summed in fp64 in row order; "fp64": exact products,
         numpy's fp64 sum; "auto": seq64 for formation="tc", else chain8)
      4. beta = -sign(u_0) sqrt(s_j); c = 1/(u_0 - beta); v = fl(u c), v_0 = 1;
         tau = (beta - u_0)/beta; R(j, i) = w_i / beta (row sign-normalised so
         R_jj = |beta|); f = fl(x - w/beta) with x = W(j, j:) (= tau W^T v)
      5. W(j:m, j:) <- fl(W - v f^T): update="fma" one rounding per entry, "rne"
         fl(W - fl(v f)) (the product rounded, then the difference)            [update, R4b]
    The tolerance stop (reading R8) is tested before step j >= 1 on the exact
    norms of step 3: sqrt(sum_{i >= j} s_i) <= eps ||A_L||_F -> k = j.

    Row sharding: A_L may be this rank's rows [row_offset,
    row_offset + m_loc) of the global matrix (row_offset % 8 == 0, so 8-row groups
    align).  Every column reduction (initial norms, s, w = W^T u) and the pivot
    row x = W(j, j:) (owner rank only, zeros elsewhere) is then summed over ranks
    with comm.sum (fp64) — the one exchange per step — and every decision (pivot,
    beta, R, f, norms) is taken identically on all ranks from the summed values.
    With comm=None the matrix is the whole A_L.

    formation="tc" (reading R14; SURVEY's D-OTF form of the
    tensor-core pass): W is the stored matrix S, updated only at store points,
    and each step forms the trailing block as X = fl32(S - V_p F_p^T), the exact
    trailing block rounded ONCE to fp32 (V_p F_p^T of the pending fp32 v / f
    vectors evaluated in fp64: each product is exact and the <= 32-term sum is
    within 2^-48 relative).  The pivot column u = X(:, 0), X(j, :) is the pivot
    row, and at a store point fl_L(X) becomes the new S.

    model="paper" selects update="rne", acc="seq64" (the default oracle the
    CUDA path is compared with by tolerance); model="kernel" selects the
    round-1 FFMA-pass model update="fma", acc="chain8".
    """
    if model == "paper":
        update, acc = "rne", "seq64"
    elif model == "kernel":
        update, acc = "fma", "chain8"
    elif model is not None:
        raise ValueError(model)
    if update not in ("fma", "rne"):
        raise ValueError(update)
    fmtL = fmt_of(fmt)
    wdt = _work_dtype(fmt)
    comm = _Local if comm is None else comm
    A_L = np.asarray(A_L, dtype=np.float64)
    m, n = A_L.shape                                        # m = rows of this shard
    if row_offset % 8:
        raise ValueError("row_offset must be a multiple of 8")
    m_glob = int(comm.sum(np.array([float(m)]))[0])
    if not (1 <= k_max <= min(m_glob, n)):
        raise ValueError("k out of range (DimensionError)")
    m8 = (m + 7) // 8 * 8
    W = np.zeros((m8, n), dtype=wdt, order="F")
    W[:m] = A_L
    perm = np.arange(n)
    R = np.zeros((k_max, n), dtype=np.float64)
    V = np.zeros((m, k_max), dtype=np.float64)
    tau = np.zeros(k_max)
    top2 = np.zeros((k_max, 2))
    if acc == "auto":
        acc = "seq64" if formation == "tc" else "chain8"
    col2 = comm.sum(seq64(A_L, A_L))                        # fp16 squares add exactly in fp64
    normAL = math.sqrt(_sum1(col2))
    maxnorm0 = math.sqrt(float(np.max(col2))) if n else 0.0
    vn = col2.copy()                                        # exact initial norms^2
    tiny = DOUBLE.min_normal if fmtL is DOUBLE else SINGLE.min_normal

    def reduce(X, Y):
        if acc == "chain8":
            return comm.sum(chain8(X, Y, wdt))
        if acc == "seq64":
            return comm.sum(seq64(X, Y))
        if acc == "fp64":
            return comm.sum(np.sum(X.astype(np.float64) * Y.astype(np.float64), axis=0))
        raise ValueError(acc)

    def local(jg):
        """first local row whose global index is >= jg, and the first row of its 8-row group"""
        jl = min(max(jg - row_offset, 0), m8)
        return jl, (jl // 8) * 8

    tc = formation == "tc"
    if tc and fmtL is DOUBLE:
        raise ValueError("formation='tc' models the low-precision tensor-core pass")
    Vp = np.zeros((m8, 0))                                  # tc: pending v (full length) and f rows
    Fp = np.zeros((0, n))

    def form_tc(j):
        """(X, u): the formed trailing block W(:, j:) and the pivot column u = X(:, 0)
        (formation='tc')."""
        D = (Vp @ Fp[:, j:]) if Fp.shape[0] else np.zeros((m8, n - j))
        X = (W[:, j:].astype(np.float64) - D).astype(wdt)
        return X, X[:, 0].copy()

    resid = []
    status, k_out = "ok", k_max
    for j in range(k_max):
        jl, g0 = local(j)                                   # local row of j / of its 8-row group
        if tc and norms == "recompute":
            raise ValueError("formation='tc' uses the downdated exact norms")
        if norms == "recompute":
            Wj = W[g0:, j:].copy()
            Wj[: jl - g0] = 0
            vn[j:] = reduce(Wj, Wj)
        cand = vn[j:]
        c_ = np.flatnonzero(cand == cand.max())             # step 1, tie -> lowest original index
        best = int(c_[np.argmin(perm[j + c_])])
        srt = np.sort(cand)[::-1]
        top2[j] = [math.sqrt(max(srt[0], 0.0)), math.sqrt(max(srt[1], 0.0)) if len(srt) > 1 else 0.0]
        p = j + best
        if p != j:
            W[:, [j, p]] = W[:, [p, j]]
            R[:j, [j, p]] = R[:j, [p, j]]
            perm[[j, p]] = perm[[p, j]]
            vn[[j, p]] = vn[[p, j]]
            Fp[:, [j, p]] = Fp[:, [p, j]]
        if tc:
            X, ucol = form_tc(j)
            if j > 0 and j % nb == 0:                       # store point: S <- fl_L(X)
                X = round_to(X.astype(np.float64), fmtL).reshape(m8, n - j).astype(wdt)
                ucol = X[:, 0].copy()
                W[:, j:] = X
                Vp, Fp = np.zeros((m8, 0)), np.zeros((0, n))
            Wj = X[g0:].copy()
            Wj[: jl - g0] = 0
            u = ucol[g0:].copy().reshape(-1, 1)
            u[: jl - g0] = 0
        else:
            if j > 0 and j % nb == 0 and fmtL is not DOUBLE:    # step 2, store point
                W[jl:, j:] = round_to(W[jl:, j:].astype(np.float64), fmtL).reshape(m8 - jl, n - j)
            Wj = W[g0:, j:].copy()                              # step 3 (rows < j masked to 0)
            Wj[: jl - g0] = 0
            u = Wj[:, :1]
        s = reduce(Wj, Wj)
        resid.append(math.sqrt(_sum1(s)))                  # exact remaining mass before step j
        if eps > 0.0 and j > 0 and resid[-1] <= eps * normAL:
            k_out = j                                       # tolerance stop (reading R8)
            break
        w = reduce(Wj, u)
        owner = row_offset <= j < row_offset + m
        xsrc = X[j - row_offset] if tc and owner else (W[j - row_offset, j:] if owner else None)
        x = comm.sum(xsrc.astype(np.float64) if owner else np.zeros(n - j))
        sj = float(s[0])
        if not (sj >= tiny):
            status, k_out = "underflow", j
            break
        u0 = float(x[0])                                    # step 4 (= W(j, j))
        beta = -math.copysign(math.sqrt(sj), u0)
        c = 1.0 / (u0 - beta)
        uu = (ucol[jl:] if tc else W[jl:, j]).astype(np.float64)
        v = (uu * c).astype(wdt)
        if owner:
            v[0] = 1.0
        tau[j] = (beta - u0) / beta
        Rraw = w / beta
        f = (x - Rraw).astype(wdt)
        R[j, j:] = (Rraw * math.copysign(1.0, beta)).astype(wdt)
        vn[j + 1:] = s[1:] - Rraw[1:] ** 2                  # one-step downdate (R6)
        if tc:                                              # step 5 deferred: pending (v, f)
            vfull = np.zeros(m8)
            vfull[jl:] = v
            frow = np.zeros(n)
            frow[j:] = f
            Vp = np.concatenate([Vp, vfull[:, None]], axis=1)
            Fp = np.concatenate([Fp, frow[None, :]], axis=0)
        else:
            if update == "fma":
                W[jl:, j:] = _fma(-v[:, None], f[None, :], W[jl:, j:], wdt)   # step 5
            else:                                           # fl(W - fl(v f)), per-op RNE
                W[jl:, j:] = W[jl:, j:] - (v.astype(wdt)[:, None] * f.astype(wdt)[None, :])
        V[jl:, j] = v[: max(m - jl, 0)]
    if status == "ok" and k_out == k_max and k_max < min(m_glob, n):
        jl, g0 = local(k_max)
        Wj = (form_tc(k_max)[0][g0:] if tc else W[g0:, k_max:]).copy()
        Wj[: jl - g0] = 0
        resid.append(math.sqrt(_sum1(reduce(Wj, Wj))))     # exact mass after k steps
    R = R[:k_out]
    return QRCPResult(perm, R, k_out, status, V[:, :k_out], tau[:k_out], top2[:k_out],
                      maxnorm0, normAL, resid)


def qrcp_mgs(A_L: np.ndarray, k: int, fmt: str = "fp64"):
    """Paper-literal pivoted MGS, the O4b cross-check.

    For j = 1..k: (a) recompute the norms of the trailing columns; (b) swap the
    max-norm column (ties: lowest index) into position j; (c) r_jj = norm;
    (d) q_j = w_j / r_jj stored to the low format; (e) for i > j:
    r_ji = fl_L(q_j . w_i), w_i = fl_L(w_i - r_ji q_j).  Arithmetic in the
    accumulation format (fp32 for fp16/fp32, fp64 for fp64).
    Returns (perm, R (k x n), Q (m x k)).
    """
    fmtL = fmt_of(fmt)
    wdt = _work_dtype(fmt)
    st = (lambda a: a.astype(wdt)) if fmtL is DOUBLE else (
        lambda a: round_to(np.asarray(a, dtype=np.float64), fmtL).astype(wdt))
    A = np.array(A_L, dtype=wdt, order="F")
    m, n = A.shape
    perm = np.arange(n)
    R = np.zeros((k, n))
    Q = np.zeros((m, k))
    for j in range(k):
        nrm = np.sqrt(np.sum(A[:, j:].astype(np.float64) ** 2, axis=0))
        p = j + int(np.argmax(nrm))          # argmax returns the first (lowest index) maximum
        if p != j:
            A[:, [j, p]] = A[:, [p, j]]
            R[:j, [j, p]] = R[:j, [p, j]]
            perm[[j, p]] = perm[[p, j]]
        rjj = float(st(np.array([math.sqrt(float(np.sum(A[:, j].astype(np.float64) ** 2)))]))[0])
        q = st(A[:, j].astype(np.float64) / rjj)
        R[j, j] = rjj
        qd = q.astype(np.float64)
        rj = st(qd @ A[:, j + 1:].astype(np.float64)).astype(np.float64)   # r_ji = fl_L(q_j . w_i)
        R[j, j + 1:] = rj
        A[:, j + 1:] = st(A[:, j + 1:].astype(np.float64) - np.outer(qd, rj)).reshape(m, n - j - 1)
        Q[:, j] = q
    return perm, R, Q


def form_Q(V: np.ndarray, tau: np.ndarray) -> np.ndarray:
    """Q(:, 0:k) = H_0 H_1 ... H_{k-1} I(:, 0:k) in fp64, H_j = I - tau_j v_j v_j^T."""
    m, k = V.shape
    Q = np.eye(m, k)
    for j in reversed(range(k)):
        v = V[:, j]
        Q -= tau[j] * np.outer(v, v @ Q)
    return Q


def certified_steps(res: QRCPResult, c_tie: float = 64.0, u_acc: float = SINGLE.u) -> np.ndarray:
    """Boolean per step: top-2 margin > c_tie * u_acc * max_i ||a_i|| (reading R10)."""
    thr = c_tie * u_acc * res.maxnorm0
    return (res.top2[:, 0] - res.top2[:, 1]) > thr
