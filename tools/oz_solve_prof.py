"""Short emulated cfg[4]-shaped solve (n = 4096, N = 64, m_F = 1) for ncu launch lists.
python tools/oz_solve_prof.py [sym] [nmod] [m_F]"""
import sys

sys.path.insert(0, ".")
import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

sym = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nmod = int(sys.argv[2]) if len(sys.argv) > 2 else 16
mF = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = workloads.config(4, with_eig=False)
s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, mF)
s.set_option("emulation", nmod)
if sym:
    s.set_option("symmetric", 1)
info = s.solve(1, w.tol, w.stop)
print(info["k_done"], info["fine_kernel_ms"], info["fine_kernel_launches"])
