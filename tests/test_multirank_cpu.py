"""World-size-2 (and 3) CPU tests of the multi-rank schedule over torch.distributed 'gloo'.

The CUDA driver (paper_1505_07959_b200/csrc/driver.cu) partitions the N time slices into
contiguous blocks (mfode_partition, the library's host-only function used here too), keeps U
ping-pong buffered by sweep parity, skips slices n < k in sweep k, and moves the boundary state
rank g -> g+1 after Step 0 and after each correction sweep, and broadcasts the stop metric from
the last rank.  This test runs exactly that schedule with the CPU oracle's propagators in one
process per rank, exchanging boundary states with gloo send/recv, and checks the result is
bitwise identical to the single-process oracle (P9: results do not depend on the rank count).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1505_07959_b200 as mf
import workloads
from oracle import dense


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, A, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T, N, mG, mF, K_max, tol, stop = cfg
    n = A.shape[0]
    s0, nloc = mf.partition(N, world, rank)
    s1 = s0 + nloc
    rhs = dense.make_rhs(A, dense.FLOW_INVERSE)
    hG, hF = T / (N * mG), T / (N * mF)
    G = lambda x: dense.euler(rhs, x, hG, mG)
    F = lambda x: dense.rk4(rhs, x, hF, mF)
    I = np.eye(n)
    U = [[None] * (nloc + 1), [None] * (nloc + 1)]
    Fk = [None] * nloc
    Gold = [None] * nloc

    def send(x):
        if rank < world - 1:
            dist.send(torch.from_numpy(np.ascontiguousarray(x)), dst=rank + 1)

    def recv():
        t = torch.empty((n, n), dtype=torch.float64)
        dist.recv(t, src=rank - 1)
        return t.numpy()

    # Step 0
    U[0][0] = I if rank == 0 else recv()
    if rank == 0:
        U[1][0] = I
    for j in range(nloc):
        g = G(U[0][j])
        U[0][j + 1] = g
        Gold[j] = g
    send(U[0][nloc])
    k_done = 0
    K_eff = min(K_max, N)
    for k in range(K_eff):
        cur, nxt = k % 2, (k + 1) % 2
        # fine (active slices n >= k)
        if k < s1:
            for j in range(max(0, k - s0), nloc):
                Fk[j] = F(U[cur][j])
        # correction
        if k < s1:
            j0 = max(0, k - s0)
            if k < s0:
                U[nxt][0] = recv()
            for j in range(j0, nloc):
                v = U[cur][j0] if (j == j0 and k >= s0) else U[nxt][j]
                g = G(v)
                U[nxt][j + 1] = Fk[j] + (g - Gold[j])
                Gold[j] = g
            send(U[nxt][nloc])
        # stop metric from the last rank
        m = torch.zeros(1, dtype=torch.float64)
        if rank == world - 1:
            m[0] = dense.frob(U[nxt][nloc] - U[cur][nloc]) / dense.frob(U[nxt][nloc])
        dist.broadcast(m, src=world - 1)
        k_done = k + 1
        if stop == dense.STOP_DELTA and m.item() <= tol:
            break
    if rank == world - 1:
        q.put((k_done, U[k_done % 2][nloc]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_schedule_bitwise(world):
    w = workloads.random_spd(12, 7)
    cfg = (1.0, 7, 1, 5, 7, 1e-12, dense.STOP_DELTA)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, w.A, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    k_done, X = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = dense.solve(w.A, dense.FLOW_INVERSE, *cfg[:5], tol=cfg[5], stop=cfg[6])
    assert k_done == ref["k_done"]
    assert np.array_equal(X, ref["X"])


def test_bench_multi_gpu_request_fails_loudly_without_gpus():
    """bench.py --gpus 2 outside torchrun re-launches itself as 2 ranks only when 2 GPUs are visible;
    on a box with fewer it exits non-zero with a message instead of timing one rank."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "0",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 3
    assert "--gpus 2" in r.stderr and "CUDA device" in r.stderr
    # under torchrun the world size must match --gpus
    env.update(WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "0",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 3 and "WORLD_SIZE=3" in r.stderr


def test_bench_spawn_path_with_gloo():
    """bench.py --gpus 2 re-launches itself as two ranks through torch.distributed.run; the plumbing
    test mode runs that path on CPU with gloo: barrier, max over ranks, rank 0 prints one line with
    n_gpus = 2 and the contiguous slice blocks (the spawn path is checked with gloo)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plumbing-test"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["rank_slice_blocks"] == [[0, 32], [32, 32]]
    assert d["max_rank_ms"] >= 19.0      # rank 1 sleeps 20 ms: the max over ranks, not rank 0's time
