"""Compare the solve result of two package copies bitwise (debug helper):
    python tools/ab_compare.py <root_a> <root_b> n flow N mF [K]"""
import os
import subprocess
import sys

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1505_07959_b200 as mf
import workloads
n, flow, N, mF, K = map(int, sys.argv[2:7])
w = workloads.random_spd(n, 7)
A = w.A if flow == 0 else w.A + np.eye(n)
s = mf.Solver(A, flow, 1.0, N, 1, mF)
import os
for kv in filter(None, os.environ.get("AB_OPTS", "").split(",")):
    k, v = kv.split("=")
    s.set_option(k, int(v))
info = s.solve(K, 0.0, 0)
np.save(sys.argv[7], s.result())
print(sys.argv[1], info["k_done"], info["deltas"], flush=True)
"""

if __name__ == "__main__":
    import numpy as np
    a, b = sys.argv[1], sys.argv[2]
    args = sys.argv[3:8] if len(sys.argv) > 7 else sys.argv[3:7] + ["1"]
    outs = []
    for i, root in enumerate((a, b)):
        f = f"/tmp/abc_{i}.npy"
        subprocess.run([sys.executable, "-c", CHILD, os.path.abspath(root), *args, f], check=True)
        outs.append(np.load(f))
    d = np.abs(outs[0] - outs[1])
    print("args", args, "bitwise equal", bool(np.array_equal(outs[0], outs[1])), "max diff", float(d.max()),
          "rows with diffs", int((d.max(axis=1) > 0).sum()), "cols", int((d.max(axis=0) > 0).sum()), flush=True)
