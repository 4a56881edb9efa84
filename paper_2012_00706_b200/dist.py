"""Host-side plumbing of the row-sharded (N > 1) path — no arithmetic of the method.

DESIGN.md §7: rank r owns the contiguous rows [row0, row0 + m_loc) of A_D; the
library's per-step exchange is an NCCL allreduce on the library's own
communicator, whose 128-byte unique id is broadcast from rank 0 with
torch.distributed (any backend: gloo on CPU in the tests, nccl on the GPU box).
Timing is the maximum over ranks (bench.py).
"""
from __future__ import annotations


def shard_rows(m_global: int, world: int, rank: int, align: int = 8):
    """(row0, m_loc) of `rank`: contiguous blocks, every row0 a multiple of `align`
    (the library's 8-row groups must not straddle shards), sizes as equal as the
    alignment allows; the blocks tile [0, m_global) exactly."""
    if world < 1 or not (0 <= rank < world) or m_global < 0:
        raise ValueError("bad shard geometry")
    groups = (m_global + align - 1) // align
    per, extra = divmod(groups, world)
    g0 = rank * per + min(rank, extra)
    g1 = g0 + per + (1 if rank < extra else 0)
    row0 = min(g0 * align, m_global)
    row1 = min(g1 * align, m_global)
    return row0, row1 - row0


def broadcast_bytes(payload: bytes | None, nbytes: int, group=None, device=None) -> bytes:
    """Broadcast `nbytes` bytes from rank 0 (e.g. the NCCL unique id) over the
    torch.distributed default group.  Rank 0 passes the payload, others None."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        if payload is None or len(payload) != nbytes:
            raise ValueError("rank 0 must provide exactly nbytes")
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, 0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def max_over_ranks(x: float, group=None, device=None) -> float:
    """max of a host scalar over all ranks (multi-GPU times are the slowest rank's)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x, group=None, device=None):
    """fp64 elementwise sum of a numpy vector over all ranks (the gloo stand-in for
    the library's NCCL allreduce in the CPU tests)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device) if device else \
        torch.from_numpy(np.array(x, dtype=np.float64, copy=True))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()
