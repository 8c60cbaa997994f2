"""Profiling target: one cfg[0] solve (K6 shared-memory kernels) and one cfg[1] solve (K10 fused fine
kernel), for ncu captures (profiles/ncu_*_r02.md).  python tools/prof_small.py [0|1|both]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    torch.cuda.set_device(0)
    for c in ((0, 1) if which == "both" else (int(which),)):
        w = workloads.config(c, with_eig=False)
        s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
        s.solve(w.K_max, w.tol, w.stop)
        s.close()
