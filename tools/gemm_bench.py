"""K1 in isolation: the library's FP64 DMMA GEMM (mfode_dgemm, and the fused RK-stage epilogue via
mfode_rk_stage) vs cuBLAS DGEMM (torch.matmul float64) at the BASELINE sizes, CUDA-event timed on
the launching stream (warm-up, best and mean of `reps`).  Prints one JSON object per line.

    python tools/gemm_bench.py [--sizes 256 1024 4096] [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402

PEAK = 37.055


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sum(ts) / len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[256, 1024, 2048, 4096, 8192])
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    for n in args.sizes:
        A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
        C = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
        D = torch.empty_like(A)
        X, S, Y = C.clone(), C.clone(), torch.empty_like(A)
        flop = 2.0 * n ** 3
        rows = {}
        best, mean = timeit(lambda: torch.matmul(A, B, out=D), args.reps)
        rows["cublas_dgemm"] = (best, mean)
        for tile in (0, 1, 2):
            best, mean = timeit(lambda: mf.dgemm(A, B, out=D, tile=tile), args.reps)
            rows[f"mfode_dgemm_tile{tile}"] = (best, mean)
        best, mean = timeit(lambda: mf.rk_stage(A, B, X, S, Y, 2, 1e-3, C=C, alpha=-1.0, beta=1.0), args.reps)
        rows["mfode_rk_stage2_sqrt_epilogue"] = (best, mean)
        for k, (b, m) in rows.items():
            print(json.dumps({"n": n, "kernel": k, "best_ms": b, "mean_ms": m, "tflops_best": flop / b / 1e9,
                              "tflops_mean": flop / m / 1e9, "frac_of_dmma_peak": flop / b / 1e9 / PEAK}),
                  flush=True)
        del A, B, C, D, X, S, Y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
