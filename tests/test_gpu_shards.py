"""The library's row-sharded path (north_star "A is row-sharded ... NCCL
allreduce combines the per-shard column norms, the Householder inner products v^T A")
executed on ONE GPU: P handles over contiguous row shards of the same matrix share a
loopback group (include/mpid.h id_loopback_create) in place of an NCCL communicator,
each driven by its own host thread and CUDA stream.  Every allreduce site of the library
runs: the scale max, the initial norms, the per-step payload [W^T u, s, pivot row], the
LSQ Grams and W, the error scalar, the power iteration's vectors, the Gram matrix and
the sketch.

Checked against the same library at P = 1 and against the oracle:
  * results are bitwise identical on every shard (every decision is taken from
    allreduced data);
  * pivots equal the P = 1 pivots (ordered, up to the oracle's first uncertified step),
    R within a few fp32 units, P within 1e-10, errors within 1e-9;
  * shard boundaries that are not multiples of the pass tile (256 rows), and shards
    smaller than k, so the owner of the pivot row j moves between ranks.
Also: an nranks = 1 NCCL communicator captured inside the QRCP's CUDA graph.
"""
import threading

import numpy as np
import pytest

from oracle.fast import qrcp_c
from oracle.qrcp import make_AL
from synth import gen_config, gen_planted
from synth.generators import fourier_params, gen_fourier
from tests.gpu_helpers import C_TIE, prefix_match, run_gpu

pytestmark = pytest.mark.gpu


def run_sharded(A, fmt, scaling, k, bounds, nb=0, formation="auto", mode="lsq", extras=True):
    import torch
    from paper_2012_00706_b200 import mpid
    m, n = A.shape
    P = len(bounds) - 1
    comm = mpid.id_loopback_create(P)
    outs = [None] * P
    errs = [None] * P

    def work(r):
        try:
            r0, r1 = bounds[r], bounds[r + 1]
            At = torch.from_numpy(np.ascontiguousarray(A[r0:r1].T)).cuda()
            st = torch.cuda.Stream()
            h = mpid.MPID(At, k_max=k, m_global=m, row_offset=r0, comm=comm, rank=r, nranks=P, stream=st)
            q = h.qrcp(fmt, scaling, k=k, nb=nb, formation=formation, allow_underflow=True)
            o = {"k": q.k, "piv": q.piv, "R": h.get_R().cpu().numpy().astype(np.float64), "perm": h.get_perm()}
            o["P"] = h.coeffs(mode).cpu().numpy()
            o["err"] = h.error()
            if extras:
                o["err_AL"] = h.error_ex("AL", "fro")
                o["err_2"] = h.error_ex("AD", 2, iters=30)
            o["stats"] = h.stats()
            h.close()
            outs[r] = o
        except Exception as ex:                      # surfaced by the main thread
            errs[r] = ex

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    calls = mpid.id_loopback_calls(comm)
    mpid.id_loopback_destroy(comm)
    for e in errs:
        if e is not None:
            raise e
    return outs, calls


def single(A, fmt, scaling, k, nb=0, formation="auto", mode="lsq", extras=True):
    import torch
    from paper_2012_00706_b200 import mpid
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    h = mpid.MPID(At, k_max=k)
    q = h.qrcp(fmt, scaling, k=k, nb=nb, formation=formation, allow_underflow=True)
    o = {"k": q.k, "piv": q.piv, "R": h.get_R().cpu().numpy().astype(np.float64), "P": h.coeffs(mode).cpu().numpy(),
         "err": h.error()}
    if extras:
        o["err_AL"] = h.error_ex("AL", "fro")
        o["err_2"] = h.error_ex("AD", 2, iters=30)
    h.close()
    return o


def check(A, fmt, scaling, k, bounds, nb=0, formation="auto", oracle_model="paper", oracle_nb=None):
    outs, calls = run_sharded(A, fmt, scaling, k, bounds, nb=nb, formation=formation)
    assert calls >= k                                    # >= one collective per QR step
    o0 = outs[0]
    for o in outs[1:]:                                   # identical on every shard
        assert o["k"] == o0["k"] and np.array_equal(o["piv"], o0["piv"])
        assert np.array_equal(o["R"], o0["R"]) and np.array_equal(o["P"], o0["P"])
        assert o["err"] == o0["err"] and o["err_AL"] == o0["err_AL"] and o["err_2"] == o0["err_2"]
    s = single(A, fmt, scaling, k, nb=nb, formation=formation)
    assert s["k"] == o0["k"]
    AL, _ = make_AL(A, fmt, scaling)
    r = qrcp_c(AL, k, fmt, nb=oracle_nb or o0["stats"]["nb"], model=oracle_model)
    agree, fu = prefix_match(s["piv"], r, c_tie=C_TIE)
    same = 0
    while same < k and o0["piv"][same] == s["piv"][same]:
        same += 1
    assert same >= min(fu, agree), (same, fu, agree)
    if same == k:
        # R: the shards group rows differently into the pass's fp32 partial sums, so R rows
        # differ at u32 level, and at the store steps a few fp16 roundings flip (u16 each)
        mx = np.max(np.abs(s["R"]))
        assert np.max(np.abs(o0["R"] - s["R"])) <= 1e-4 * mx
        assert np.linalg.norm(o0["P"] - s["P"]) <= 1e-10 * np.linalg.norm(s["P"])
        assert abs(o0["err"][1] - s["err"][1]) <= 1e-9 * s["err"][1]
        assert abs(o0["err_AL"][1] - s["err_AL"][1]) <= 1e-9 * s["err_AL"][1]
        # the 2-norm is not stationary in P (unlike the LSQ Frobenius residual): a 1e-10
        # relative change of P moves it by ~1e-10 of ||A||_2, i.e. absolute in these units
        assert abs(o0["err_2"][1] - s["err_2"][1]) <= 1e-6 * s["err_2"][1] + 1e-8
    return outs, s


@pytest.mark.parametrize("fmt,sc", [("fp16", "pow2"), ("fp32", "none")])
def test_C1_two_and_four_shards_owner_moves(fmt, sc):
    A = gen_config("C1", 0)
    check(A, fmt, sc, 32, [0, 128, 256])
    check(A, fmt, sc, 32, [0, 24, 72, 160, 256])          # shards < k: row j's owner moves


def test_C2_shards_not_tile_aligned():
    A = gen_config("C2", 1)
    check(A, "fp16", "maxabs", 64, [0, 1000, 2600, 4096])
    check(A, "fp32", "none", 64, [0, 8, 2048, 4096])


def test_planted_four_shards_set_and_order():
    A, skel, C = gen_planted(4096, 512, 64, rho=1.05, eta=1e-9, seed=2)
    outs, s = check(A, "fp16", "pow2", 64, [0, 40, 1032, 3000, 4096])
    assert np.array_equal(outs[0]["piv"], skel)


def test_C4_analogue_two_and_four_shards():
    fp = fourier_params(32, 64, 1024, 0)
    A = gen_fourier(fp, 0)
    check(A, "fp16", "pow2", 100, [0, 16384, 32768])
    check(A, "fp16", "pow2", 100, [0, 8000, 16000, 24008, 32768])


@pytest.mark.parametrize("formation", ["gram", "sketch"])
def test_next4_pivoting_sharded(formation):
    A = gen_config("C2", 0)
    outs, calls = run_sharded(A, "fp16", "maxabs", 64, [0, 1024, 2048, 4096], formation=formation, extras=False)
    s = single(A, "fp16", "maxabs", 64, formation=formation, extras=False)
    for o in outs[1:]:
        assert np.array_equal(o["piv"], outs[0]["piv"]) and np.array_equal(o["P"], outs[0]["P"])
    # the Gram (and the sketch) are sums over the shards' rows in another order; Gram pivoting
    # squares the conditioning (reading R17), so the sequences may part early — the error
    # (the quantity the pivots serve) must agree
    assert abs(outs[0]["err"][1] - s["err"][1]) <= 0.05 * s["err"][1]


def test_nccl_single_rank_communicator_inside_cuda_graph():
    """nranks = 1 with a real NCCL communicator: the library still calls ncclAllReduce for
    every reduction, and the QRCP's k-step loop (with its NCCL calls) is captured in a
    CUDA graph; the sums over one rank leave the results bitwise unchanged."""
    import torch
    from paper_2012_00706_b200 import mpid
    A = gen_config("C1", 1)
    base = single(A, "fp16", "pow2", 32, formation="ffma", extras=False)
    uid = mpid.id_nccl_get_unique_id()
    comm = mpid.id_nccl_comm_init(uid, 1, 0)
    try:
        At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
        h = mpid.MPID(At, k_max=32, comm=comm, rank=0, nranks=1)
        for _ in range(2):                               # capture, then replay the graph
            q = h.qrcp("fp16", "pow2", k=32, use_graph=True, formation="ffma")
            P = h.coeffs("lsq").cpu().numpy()
            e = h.error()
        h.close()
    finally:
        mpid.id_nccl_comm_destroy(comm)
    assert np.array_equal(q.piv, base["piv"]) and np.array_equal(P, base["P"]) and e == base["err"]
