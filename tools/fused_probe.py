"""K10 probe: fine-phase TFLOP/s of one fixed-K=1 sweep for n / N / fused on-off (CUDA-event timed by
the library around each fine chunk).  python tools/fused_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402


def run(n, N, mF, fused, flow=mf.FLOW_INVERSE, reps=3):
    A = np.eye(n) + 0.25 * workloads.laplacian_1d(n)
    s = mf.Solver(A, flow, 1.0, N, 1, mF)
    s.set_option("fused", fused)
    s.solve(1)
    best = None
    for _ in range(reps):
        i = s.solve(1)
        tf = i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12
        best = tf if best is None else max(best, tf)
    s.close()
    return {"n": n, "N": N, "mF": mF, "fused": fused, "flow": flow, "fine_tflops": best,
            "ms_fine": i["fine_kernel_ms"], "launches": i["gpu_launches"]}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    cases = [(256, 16, 32), (256, 32, 32), (256, 64, 32), (128, 64, 32), (512, 16, 16), (384, 16, 16)]
    for n, N, mF in cases:
        for fused in (1, 0):
            print(json.dumps(run(n, N, mF, fused)), flush=True)
