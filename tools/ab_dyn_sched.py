"""A/B of the DMMA GEMM tile schedule (option "dyn_sched"): the bench workload (cfg[4]) solve time and
a batched n = 4096 GEMM, ticketed vs round-robin, same process.  python tools/ab_dyn_sched.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 4096
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    outs = {}
    for mode in (1, 0, 1, 0):
        s = mf.Solver(np.eye(8), mf.FLOW_INVERSE, 1.0, 2, 1, 1)
        s.set_option("dyn_sched", mode)
        D = mf.dgemm(A, B)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            mf.dgemm(A, B, out=D)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        outs.setdefault(mode, D.clone())
        assert torch.equal(outs[mode], D)
        print(json.dumps({"dyn_sched": mode, "gemm_n": n, "ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}), flush=True)
        s.close()
    assert torch.equal(outs[0], outs[1])
    w = workloads.config(4, with_eig=False)
    s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
    X = {}
    for mode in (1, 0, 1):
        s.set_option("dyn_sched", mode)
        i = s.solve(w.K_max, w.tol, w.stop)
        X.setdefault(mode, s.result())
        assert np.array_equal(X[mode], s.result())
        print(json.dumps({"dyn_sched": mode, "workload": w.name, "ms": i["ms_total"], "k_done": i["k_done"],
                          "fine_kernel_tflops": i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12}),
              flush=True)
    assert np.array_equal(X[0], X[1])


if __name__ == "__main__":
    main()
