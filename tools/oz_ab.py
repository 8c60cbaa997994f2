"""Same-box A/B of package copies on the f3(ii) emulated path: a short cfg[4]-shaped solve (n = 4096,
N = 64, m_F = 4) with emulation = 16, plain and symmetric, fine-phase ms and the result's bits.
    python tools/oz_ab.py <root> [<root> ...]"""
import subprocess
import sys

CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1505_07959_b200 as mf
import workloads
torch.cuda.set_device(0)
w = workloads.config(4, with_eig=False)
out = {"lib": sys.argv[1]}
for sym in (0, 1):
    s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, 4)
    s.set_option("emulation", 16)
    if sym:
        s.set_option("symmetric", 1)
    s.solve(1)
    best = None
    for _ in range(2):
        i = s.solve(1)
        best = i["fine_kernel_ms"] if best is None else min(best, i["fine_kernel_ms"])
    out[f"sym{sym}_fine_ms"] = round(best, 2)
    out[f"sym{sym}_md5"] = hashlib.md5(s.result().tobytes()).hexdigest()[:12]
    s.close()
print(json.dumps(out), flush=True)
"""

if __name__ == "__main__":
    for r in range(2):
        for root in sys.argv[1:]:
            subprocess.run([sys.executable, "-c", CHILD, root], check=False)
