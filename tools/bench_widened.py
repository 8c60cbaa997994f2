"""Measurement of the widened rows on one B200: exp and trig flows (f1), Algorithm 5
cos(A) (f1), modified parareal Algorithms 3 and 4 (f2), accelerated inverse Algorithm 8 (f4).  Each line:
time, algorithmic FP64 TFLOP/s of its GEMM work, and the fraction of the measured DMMA peak.
    python tools/bench_widened.py > profiles/widened_rows_r02.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

PEAK = 37.055


def line(**kw):
    if "tflops" in kw and kw["tflops"] is not None:
        kw["frac_of_dmma_peak"] = kw["tflops"] / PEAK
    print(json.dumps(kw), flush=True)


def fine_rate(i):
    return i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12 if i["fine_kernel_ms"] > 0 else None


def main():
    torch.cuda.set_device(0)
    n = 2048
    w = workloads.random_spd(n, 70, lo=0.5, hi=1.5)
    A = w.A / 1.5
    # f1: exp flow dQ/dt = A Q (Example 2) and the trig block flow (Example 3), classical parareal, fixed K
    for flow, name in ((mf.FLOW_EXP, "exp_flow"), (mf.FLOW_TRIG, "trig_flow")):
        s = mf.Solver(A, flow, 1.0, 32, 2, 32)
        s.solve(2)
        i = s.solve(4)
        line(row="f1", what=name, n=n, N=32, m_G=2, m_F=32, K=4, ms=i["ms_total"],
             tflops_whole=i["fine_flops"] / (i["ms_total"] * 1e-3) / 1e12, tflops=fine_rate(i),
             gpu_launches=i["gpu_launches"])
        s.close()
    # f1: Algorithm 5, cos(A) = parareal on the trig flow for 2^-m A, then m double-angle GEMMs
    B = 3.0 * A
    mf.cosine(B, 32, 2, 32, 4)
    t0 = time.perf_counter()
    C, m, info = mf.cosine(B, 32, 2, 32, 4)
    wall = time.perf_counter() - t0
    line(row="f1", what="cosine_algorithm5", n=n, m=m, wall_ms_incl_create_and_copies=wall * 1e3,
         solve_ms=info["ms_total"], tflops=fine_rate(info))
    # f2: modified parareal, Algorithm 3 (exp flow) and Algorithm 4 (affine flow, Example 5's I - A X)
    n2 = 1024
    w2 = workloads.random_spd(n2, 71, lo=0.5, hi=2.0)
    s = mf.Solver(w2.A, mf.FLOW_EXP, 1.0, 16, 1, 32)
    s.solve_modified(2)
    i = s.solve_modified(4)
    line(row="f2", what="modified_parareal_alg3_exp", n=n2, N=16, m_F=32, K=4, ms=i["ms_total"],
         basis=i["basis_size"], tflops_fine=fine_rate(i), ms_correct=i["ms_correct"],
         fine_flops=i["fine_flops"], tflops=i["fine_flops"] / (i["ms_total"] * 1e-3) / 1e12)
    s.close()
    s = mf.Solver(-w2.A, mf.FLOW_AFFINE, 8.0, 16, 2, 32)
    s.set_affine(np.eye(n2), np.zeros((n2, n2)))
    s.solve_modified(2)
    i = s.solve_modified(4)
    line(row="f2", what="modified_parareal_alg4_affine", n=n2, N=16, m_F=32, K=4, ms=i["ms_total"],
         basis=i["basis_size"], ms_correct=i["ms_correct"], fine_flops=i["fine_flops"],
         tflops=i["fine_flops"] / (i["ms_total"] * 1e-3) / 1e12)
    s.close()
    # f4: Algorithm 8, accelerated steady-state inverse (one batched GEMM of (X, u) per step)
    n4 = 4096
    w4 = workloads.config(3, with_eig=False)
    A4 = w4.A / np.linalg.norm(w4.A, 2) if False else w4.A / 3.0
    steps = 100
    mf.accel_inverse(A4, None, 0.5, 5)
    t0 = time.perf_counter()
    X, k, res, st = mf.accel_inverse(A4, None, 0.5, steps)
    wall = time.perf_counter() - t0
    flops = steps * 2 * 2.0 * n4 ** 3
    line(row="f4", what="accel_inverse_alg8", n=n4, steps=k, wall_ms_incl_create_and_copies=wall * 1e3,
         tflops=flops / wall / 1e12, residual=res, note="wall clock incl. create (H2D) and D2H of X")


if __name__ == "__main__":
    main()
