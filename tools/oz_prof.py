"""One emulated GEMM at n (default 4096) for ncu captures.  python tools/oz_prof.py [n] [nmod] [pair]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_07959_b200 as mf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nmod = int(sys.argv[2]) if len(sys.argv) > 2 else 16
pair = int(sys.argv[3]) if len(sys.argv) > 3 else 1
s = mf.Solver(np.eye(2), mf.FLOW_INVERSE, 1.0, 1, 1, 1)
s.set_option("oz_pair", pair)
s.close()
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
B = torch.randn(n, n, dtype=torch.float64, device="cuda")
out = torch.empty_like(A)
for _ in range(2):
    mf.dgemm_emulated(A, B, out=out, n_moduli=nmod)
torch.cuda.synchronize()
