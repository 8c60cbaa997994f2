"""Achieved HBM bandwidth of the element-wise kernels that are not fused into a GEMM epilogue
(SURVEY §8(d) M4): the deterministic Frobenius-norm reduction K5 (mfode_frobenius: reads X and Y)
at n = 16384 (2 GiB per matrix, far beyond L2).  CUDA events around repeated calls; the call
synchronises and copies 16 bytes to the host, included in the time.
    python tools/hbm_kernels.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_07959_b200 as mf  # noqa: E402

n = 16384
X = torch.randn(n, n, dtype=torch.float64, device="cuda")
Y = torch.randn(n, n, dtype=torch.float64, device="cuda")
mf.frobenius(X, Y)
torch.cuda.synchronize()
reps = 10
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    mf.frobenius(X, Y)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(json.dumps({"kernel": "k_frob_partial + k_reduce_final (||X - Y||_F, ||X||_F)", "n": n,
                  "bytes": 2 * 8 * n * n, "ms": ms, "GB_per_s": 2 * 8 * n * n / (ms * 1e-3) / 1e9}))
