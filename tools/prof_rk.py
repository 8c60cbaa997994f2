"""Profiling target: one cfg[4] solve (the bench headline: n = 4096 sqrt flow, 64 slices), for the ncu
launch list and the --set full capture of one fused RK-stage GEMM launch (profiles/ncu_*_r02*.md).
    python tools/prof_rk.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    w = workloads.config(4, with_eig=False)
    s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
    info = s.solve(w.K_max, w.tol, w.stop)
    print("k_done", info["k_done"], "ms", info["ms_total"], flush=True)
    s.close()
