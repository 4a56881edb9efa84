"""A host-resident A_D streamed in row blocks (SURVEY §8(b) ownership clause; include/mpid.h
id_create_ex ID_CREATE_STREAM_HOST): the rounding, the LSQ product W = Q1^T A_D(:, J) and the
error read A_D block by block through two staging buffers.

Checked against the same library with A_D in device memory: A_L bit for bit, pivots / R /
the tolerance rank identical (the QRCP sees the same A_L), P within 1e-12 and the error
within 1e-12 (the W and error sums are reassociated over blocks), with several blocks and a
ragged last block; also row-sharded over a loopback group (the streamed round's max and
norm reductions across ranks), and against the oracle (P from the GPU's I)."""
import threading

import numpy as np
import pytest

from oracle.id import coeffs_lsq, id_error
from synth import gen_config

pytestmark = pytest.mark.gpu


def _run(A, fmt, sc, k, stream, eps=0.0, log2=10, comm=None, rank=0, nranks=1, rows=None):
    import torch
    from paper_2012_00706_b200.mpid import MPID
    m, n = A.shape
    r0, r1 = rows if rows else (0, m)
    blk = np.ascontiguousarray(A[r0:r1].T)
    At = torch.from_numpy(blk).pin_memory() if stream else torch.from_numpy(blk).cuda()
    st = torch.cuda.Stream() if comm else None
    h = MPID(At, k_max=k, m_global=m, row_offset=r0, comm=comm, rank=rank, nranks=nranks, stream=st,
             device="cuda", stream_host=stream, stream_rows_log2=log2 if stream else 0)
    h.round_only(fmt, sc)
    AL = h.get_AL().cpu().numpy()
    q = h.qrcp(fmt, sc, k=k, eps=eps)
    out = {"AL": AL, "k": q.k, "piv": q.piv, "R": h.get_R().cpu().numpy(), "P": h.coeffs("lsq").cpu().numpy(),
           "err": h.error(), "stats": h.stats()}
    h.close()
    return out


@pytest.mark.parametrize("fmt,sc,k,eps", [("fp16", "pow2", 64, 0.0), ("fp32", "none", 64, 0.0),
                                          ("fp16", "maxabs", 200, 1e-2)])
def test_streamed_equals_device(fmt, sc, k, eps):
    A = np.asfortranarray(gen_config("C2", 1)[:4099, :700])       # 5 blocks of 1024 rows, ragged
    d = _run(A, fmt, sc, k, False, eps=eps)
    h = _run(A, fmt, sc, k, True, eps=eps)
    assert h["AL"].tobytes() == d["AL"].tobytes()
    assert h["k"] == d["k"] and np.array_equal(h["piv"], d["piv"]) and np.array_equal(h["R"], d["R"])
    assert np.linalg.norm(h["P"] - d["P"]) <= 1e-12 * np.linalg.norm(d["P"])
    assert abs(h["err"][1] - d["err"][1]) <= 1e-12 * d["err"][1]
    P_ref = coeffs_lsq(A, h["piv"])
    assert np.linalg.norm(h["P"] - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    assert abs(id_error(A, h["piv"], h["P"])[1] - h["err"][1]) <= 1e-9 * h["err"][1]


def test_streamed_rejects_device_only_variants():
    import torch
    from paper_2012_00706_b200.mpid import MPID, IDError
    A = np.asfortranarray(gen_config("C1", 0))
    h = MPID(torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory(), k_max=8, device="cuda", stream_host=True,
             stream_rows_log2=8)
    h.qrcp("fp16", "pow2", k=8)
    h.coeffs("lsq")
    h.error()
    with pytest.raises(IDError):
        h.error_ex("AD", 2)
    h.close()


def test_streamed_row_shards_loopback():
    from paper_2012_00706_b200 import mpid
    A = np.asfortranarray(gen_config("C2", 0)[:, :512])
    d = _run(A, "fp16", "maxabs", 48, False)
    bounds = [0, 1304, 4096]
    comm = mpid.id_loopback_create(2)
    outs, errs = [None, None], [None, None]

    def work(r):
        try:
            outs[r] = _run(A, "fp16", "maxabs", 48, True, log2=9, comm=comm, rank=r, nranks=2,
                           rows=(bounds[r], bounds[r + 1]))
        except Exception as ex:
            errs[r] = ex

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    mpid.id_loopback_destroy(comm)
    for e in errs:
        if e is not None:
            raise e
    o0, o1 = outs
    assert np.array_equal(o0["piv"], o1["piv"]) and np.array_equal(o0["P"], o1["P"]) and o0["err"] == o1["err"]
    assert np.vstack([o0["AL"], o1["AL"]]).tobytes() == d["AL"].tobytes()
    same = 0
    while same < 48 and o0["piv"][same] == d["piv"][same]:
        same += 1
    assert same >= 40
    if same == 48:
        assert np.linalg.norm(o0["P"] - d["P"]) <= 1e-10 * np.linalg.norm(d["P"])
        assert abs(o0["err"][1] - d["err"][1]) <= 1e-9 * d["err"][1]
