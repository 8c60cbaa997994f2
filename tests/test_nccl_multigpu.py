"""NCCL mode of the C library (one process per GPU, boundary states over NCCL send/recv).

Needs >= 2 GPUs (skipped otherwise; the single-GPU boxes of this run exercise the same per-rank
code through logical ranks in test_gpu_parity.py and the schedule over gloo in
test_multirank_cpu.py).  Checks that world = 2 over NCCL is bitwise identical to world = 1 (P9).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, q):
    import torch.distributed as dist
    import paper_1505_07959_b200 as mf
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    obj = [bytes(torch.cuda.nccl.unique_id()) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, 8, 1, 8, world=world, rank=rank, device=rank, nccl_uid=obj[0])
    info = s.solve(8, 1e-12, mf.STOP_DELTA)
    X = s.result()
    im = s.solve(8, 1e-9, mf.STOP_MAX_SLICE)          # SPEC stop: ncclAllReduce(max) of the slice metrics
    Xm = s.result()
    if rank == 0:
        q.put((info["k_done"], X, im["k_done"], Xm, info["ms_comm"]))
    s.close()
    dist.destroy_process_group()


def test_nccl_two_ranks_bitwise():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    import paper_1505_07959_b200 as mf
    import workloads
    w = workloads.random_spd(96, 5)
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, 8, 1, 8)
    i1 = s.solve(8, 1e-12, mf.STOP_DELTA)
    X1 = s.result()
    im1 = s.solve(8, 1e-9, mf.STOP_MAX_SLICE)
    Xm1 = s.result()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, w.A, q)) for r in range(2)]
    for p in ps:
        p.start()
    k, X, km, Xm, ms_comm = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert k == i1["k_done"]
    assert np.array_equal(X, X1)
    assert km == im1["k_done"] and np.array_equal(Xm, Xm1)
    assert ms_comm > 0.0


def test_nccl_one_rank_communicator_bitwise():
    """NCCL mode with a one-rank communicator (runs on a single GPU): the NCCL code path (metric
    broadcasts, stop-flag copies, result broadcast) gives bitwise the result of the default mode,
    including speculative overlap with a tolerance stop and the sqrt flow's residual stop."""
    import paper_1505_07959_b200 as mf
    import workloads
    w = workloads.random_spd(96, 5)
    for flow, T, N, mG, mF, K, tol, stop in ((mf.FLOW_INVERSE, 1.0, 8, 1, 8, 8, 1e-12, mf.STOP_DELTA),
                                             (mf.FLOW_INVERSE, 1.0, 6, 1, 4, 3, 0.0, mf.STOP_FIXED_K),
                                             (mf.FLOW_INVERSE, 1.0, 8, 1, 8, 8, 1e-9, mf.STOP_MAX_SLICE)):
        s = mf.Solver(w.A, flow, T, N, mG, mF)
        i1 = s.solve(K, tol, stop)
        X1 = s.result()
        s.close()
        uid = bytes(torch.cuda.nccl.unique_id())   # one unique id per communicator (one-shot bootstrap)
        s = mf.Solver(w.A, flow, T, N, mG, mF, world=1, rank=0, device=0, nccl_uid=uid)
        i2 = s.solve(K, tol, stop)
        X2 = s.result()
        s.close()
        assert i1["k_done"] == i2["k_done"]
        assert np.array_equal(X1, X2)
    m = 8
    import numpy as _np
    A = workloads.laplacian_2d(m) + _np.eye(m * m)
    s = mf.Solver(A, mf.FLOW_SQRT, 20.0, 64, 2, 16)
    i1 = s.solve(4, 1e-10, mf.STOP_RESIDUAL)
    X1 = s.result()
    s.close()
    s = mf.Solver(A, mf.FLOW_SQRT, 20.0, 64, 2, 16, world=1, rank=0, device=0,
                  nccl_uid=bytes(torch.cuda.nccl.unique_id()))
    i2 = s.solve(4, 1e-10, mf.STOP_RESIDUAL)
    X2 = s.result()
    s.close()
    assert i1["k_done"] == i2["k_done"]
    assert np.array_equal(X1, X2)
