"""Per-config measurement: wall time, k_done, fine TFLOP/s and the dominant
kernel's TFLOP/s for BASELINE configs on one B200, plus the sequential-fine time (P/K context).

    python tools/bench_configs.py --configs 0 1 2 [--seq] > gpurun_out/configs.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--seq", action="store_true")
    ap.add_argument("--opt", nargs="*", default=[])
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for c in args.configs:
        w = workloads.config(c, with_eig=False)
        s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
        for o in args.opt:
            k, v = o.split("=")
            s.set_option(k, int(v))
        s.solve(w.K_max, w.tol, w.stop)   # warm-up
        infos = []
        t0 = time.perf_counter()
        for _ in range(args.reps):
            infos.append(s.solve(w.K_max, w.tol, w.stop))
        wall = (time.perf_counter() - t0) / args.reps
        i = infos[-1]
        ms = float(np.mean([x["ms_total"] for x in infos]))
        rec = {"config": w.name, "n": w.n, "N": w.N, "m_G": w.m_G, "m_F": w.m_F, "k_done": i["k_done"],
               "status": i["status"], "ms_solve_device": ms, "ms_solve_wall": wall * 1e3,
               "fine_tflops_whole_solve": i["fine_flops"] / (ms * 1e-3) / 1e12,
               "fine_kernel_tflops": (i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12
                                      if i["fine_kernel_ms"] > 0 else None),
               "launches_per_solve": i["gpu_launches"], "deltas": i["deltas"], "residual": s.residual(),
               "phases_ms": {k: i[k] for k in ("ms_coarse", "ms_correct", "ms_comm", "ms_metric", "ms_fine",
                                                "fine_kernel_ms")},
               "opts": args.opt}
        if args.seq:
            q = s.sequential_fine()
            rec["ms_sequential_fine"] = q["ms_total"]
            rec["parareal_speedup_vs_seq_1gpu"] = q["ms_total"] / ms
        print(json.dumps(rec), flush=True)
        s.close()


if __name__ == "__main__":
    main()
