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
    if rank == 0:
        q.put((info["k_done"], X))
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
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, w.A, q)) for r in range(2)]
    for p in ps:
        p.start()
    k, X = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert k == i1["k_done"]
    assert np.array_equal(X, X1)
