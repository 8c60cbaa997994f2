"""Same-box A/B of K10 builds (package copies under given roots): fine-kernel TFLOP/s of one fixed-K=1
sweep (inverse flow) at several n / N, and the cfg[1] time-to-tol, each root in a fresh process,
roots interleaved over `rounds`.
    python tools/ab_k10.py <root> [<root> ...] [--rounds R]"""
import subprocess
import sys

CHILD = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1505_07959_b200 as mf
import workloads
torch.cuda.set_device(0)
out = {"root": sys.argv[1]}
for n, N, mF in ((256, 16, 32), (256, 32, 32), (512, 16, 16), (384, 16, 16), (128, 64, 32)):
    A = np.eye(n) + 0.25 * workloads.laplacian_1d(n)
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, N, 1, mF)
    s.set_option("fused", 1)
    s.solve(1)
    best = 0.0
    for _ in range(3):
        i = s.solve(1)
        best = max(best, i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12)
    s.close()
    out[f"n{n}_N{N}"] = round(best, 3)
w = workloads.config(1, with_eig=False)
s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
s.solve(w.K_max, w.tol, w.stop)
ms = min(s.solve(w.K_max, w.tol, w.stop)["ms_total"] for _ in range(3))
out["cfg1_ms"] = round(ms, 3)
print(json.dumps(out), flush=True)
"""

if __name__ == "__main__":
    args = sys.argv[1:]
    rounds = 2
    if "--rounds" in args:
        k = args.index("--rounds")
        rounds = int(args[k + 1])
        del args[k:k + 2]
    for _ in range(rounds):
        for root in args:
            r = subprocess.run([sys.executable, "-c", CHILD, root], capture_output=True, text=True)
            print(r.stdout.strip() if r.returncode == 0 else f'{{"root": "{root}", "error": {r.returncode}}}',
                  flush=True)
            occ = sorted(set(l for l in r.stderr.splitlines() if l.startswith("K10 cfg")))
            if occ:
                print("  # " + "; ".join(occ), flush=True)
            if r.returncode != 0:
                print(r.stderr[-2000:], file=sys.stderr)
