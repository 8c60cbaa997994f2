"""K10 fine-phase TF/s of a fixed-K=1 sweep (n = 256, 16 slices, m_F = 32), for same-box A/B of package
copies:  python tools/fused_ab.py <root> [<root> ...]"""
import json
import subprocess
import sys

CHILD = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1505_07959_b200 as mf
import workloads
torch.cuda.set_device(0)
out = {"lib": sys.argv[1]}
for n, N, mF in ((256, 16, 32), (256, 32, 32), (512, 16, 16)):
    A = np.eye(n) + 0.25 * workloads.laplacian_1d(n)
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, N, 1, mF)
    def solve1():
        try:
            return s.solve(1)
        except mf.MfodeError as e:   # diagnostic builds may produce garbage; the timing is still valid
            return e.info
    solve1()
    best = 0.0
    for _ in range(3):
        i = solve1()
        best = max(best, i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12)
    out[f"n{n}_N{N}"] = round(best, 3)
    s.close()
print(json.dumps(out), flush=True)
"""

if __name__ == "__main__":
    for r in range(2):
        for root in sys.argv[1:]:
            subprocess.run([sys.executable, "-c", CHILD, root], check=False)
