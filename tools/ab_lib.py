"""Same-box A/B of two builds of the library (e.g. _base/ = an earlier commit vs the working tree):
each measurement runs in a fresh process that imports the chosen package copy.
    python tools/ab_lib.py <root_a> <root_b> [reps] [solve 0|1]"""
import os
import subprocess
import sys

CHILD = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1505_07959_b200 as mf
import workloads
torch.cuda.set_device(0)
if len(sys.argv) > 3 and sys.argv[3] != "-":   # process-wide option key=value, when the build knows it
    _s = mf.Solver(np.eye(8), mf.FLOW_INVERSE, 1.0, 2, 1, 1)
    _k, _v = sys.argv[3].split("=")
    try:
        _s.set_option(_k, int(_v))
    except Exception:
        pass
    _s.close()
n = 4096
g = torch.Generator(device="cuda").manual_seed(1)
Y = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
X = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
S = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
Yn = torch.empty_like(Y)
A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
for _ in range(3):
    mf.rk_stage(Y, Y, X, S, Yn, 2, 1e-3, C=A, alpha=-1.0, beta=1.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mf.rk_stage(Y, Y, X, S, Yn, 2, 1e-3, C=A, alpha=-1.0, beta=1.0)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 20
out = {"lib": sys.argv[1], "opt": sys.argv[3] if len(sys.argv) > 3 else None, "rk_stage_ms": ms,
       "rk_stage_tflops": 2 * n ** 3 / ms / 1e9}
if sys.argv[2] == "1":
    w = workloads.config(4, with_eig=False)
    s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
    i = s.solve(w.K_max, w.tol, w.stop)
    out.update(cfg4_ms=i["ms_total"],
               cfg4_fine_kernel_tflops=i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12)
print(json.dumps(out), flush=True)
"""

if __name__ == "__main__":
    a, b = sys.argv[1], sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    solve = sys.argv[4] if len(sys.argv) > 4 else "1"
    opts = sys.argv[5].split(",") if len(sys.argv) > 5 else ["-"]
    for r in range(reps):
        for root in (a, b):
            for o in (opts if root == b else ["-"]):
                subprocess.run([sys.executable, "-c", CHILD, os.path.abspath(root), solve, o], check=False)
