"""The row-sharded (N > 1) path on CPU: world-size-2 `gloo` process groups.

What is covered:
  * shard geometry (paper_2012_00706_b200.dist.shard_rows) tiles the rows with
    8-aligned offsets;
  * the NCCL-unique-id broadcast and the max-over-ranks timing reduction that
    bench.py uses, over a real 2-process group;
  * the data-parallel decomposition the kernels implement: each rank reduces its
    own rows (8-row fp32 chains, fp64 partials), ONE fp64 allreduce per step
    combines [W^T u, s, pivot row], and every decision is taken from the summed
    values — run with the oracle on 2 gloo ranks, it gives the same pivots as the
    unsharded oracle and bitwise-identical results on both ranks.
"""
import os
import socket

import numpy as np
import pytest

from paper_2012_00706_b200.dist import shard_rows


@pytest.mark.parametrize("m,world", [(256, 2), (1000, 2), (4099, 4), (16, 8), (8, 2), (2 ** 21, 8)])
def test_shard_rows_tile_exactly(m, world):
    covered = 0
    for r in range(world):
        row0, m_loc = shard_rows(m, world, r)
        assert row0 == covered and row0 % 8 == 0 and m_loc >= 0
        covered += m_loc
    assert covered == m


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2012_00706_b200.dist import broadcast_bytes, max_over_ranks, sum_over_ranks
        from oracle.qrcp import make_AL, qrcp_householder
        from synth import gen_config
        out = {}
        uid = bytes(range(128)) if rank == 0 else None
        out["uid"] = broadcast_bytes(uid, 128)
        out["max"] = max_over_ranks(10.0 + rank)

        class Comm:
            @staticmethod
            def sum(x):
                return sum_over_ranks(x)

        A = gen_config("C1", 0)
        AL, _ = make_AL(A, "fp16", "pow2")
        row0, m_loc = shard_rows(A.shape[0], world, rank)
        r = qrcp_householder(AL[row0:row0 + m_loc], 32, "fp16", nb=4, row_offset=row0, comm=Comm)
        out["perm"] = r.perm.copy()
        out["R"] = r.R.copy()
        out["top2"] = r.top2.copy()
        out["resid"] = list(r.resid)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_sharded_qrcp_matches_unsharded():
    import torch.multiprocessing as mp
    from oracle.qrcp import certified_steps, make_AL, qrcp_householder
    from synth import gen_config
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res[0], res[1]
    assert a["uid"] == b["uid"] == bytes(range(128))
    assert a["max"] == b["max"] == 11.0
    # identical on all ranks (replicated decisions from allreduced data)
    assert np.array_equal(a["perm"], b["perm"]) and np.array_equal(a["R"], b["R"])
    # same as the unsharded oracle on every certified step
    A = gen_config("C1", 0)
    AL, _ = make_AL(A, "fp16", "pow2")
    ref = qrcp_householder(AL, 32, "fp16", nb=4)
    cert = certified_steps(ref)
    fu = int(np.argmin(cert)) if not cert.all() else 32
    assert np.array_equal(a["perm"][:fu], ref.perm[:fu])
    # the only difference is the fp64 order of the cross-rank partial sums
    assert np.allclose(a["R"][:fu], ref.R[:fu], rtol=0, atol=1e-5 * ref.maxnorm0)


def _gram_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2012_00706_b200.dist import sum_over_ranks
        from oracle.gram import gram, pivoted_cholesky
        from oracle.qrcp import make_AL
        from synth import gen_config
        A = gen_config("C2", 0)[:, :200]
        AL, _ = make_AL(A, "fp16", "pow2")
        row0, m_loc = shard_rows(A.shape[0], world, rank)
        # Gram pivoting at N > 1: each rank's G_r = A_r^T A_r, ONE allreduce
        # of the n x n Gram, then the pivoted Cholesky replicated on every rank
        G = sum_over_ranks(gram(AL[row0:row0 + m_loc]))
        r = pivoted_cholesky(np.asarray(G), 40)
        q.put((rank, {"perm": r.perm.copy(), "R": r.R.copy()}))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gram_pivoting_matches_unsharded():
    import torch.multiprocessing as mp
    from oracle.gram import certified_gram_steps, gram, pivoted_cholesky
    from oracle.qrcp import make_AL
    from synth import gen_config
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gram_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res[0], res[1]
    assert np.array_equal(a["perm"], b["perm"]) and np.array_equal(a["R"], b["R"])
    A = gen_config("C2", 0)[:, :200]
    AL, _ = make_AL(A, "fp16", "pow2")
    ref = pivoted_cholesky(gram(AL), 40)
    cert = certified_gram_steps(ref, gamma=1e-13)
    fu = int(np.argmin(cert)) if not cert.all() else 40
    assert fu > 10
    assert np.array_equal(a["perm"][:fu], ref.perm[:fu])
    assert np.allclose(a["R"][:fu, :fu], ref.R[:fu, :fu], rtol=0, atol=1e-10 * np.sqrt(ref.d0max))
