"""BASELINE cfg[3] end to end on one B200 (M2: parareal time-to-tol at n = 4096, inverse flow):
A = I + G^T G / (2n), N = 64, m_G = 1, m_F = 128, delta <= 1e-10, K_max = 12.  Full-output parity
against the spectral oracle (eigh of A on the host, then the scalar parareal per eigenvalue), then
the same solve in the f3 symmetric mode.  Prints JSON lines.  ~20 + ~11 GPU-minutes.

    python tools/run_cfg3.py [--skip-full] [--skip-sym]
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
from oracle import spectral  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--skip-sym", action="store_true")
    ap.add_argument("--modes", nargs="*", default=None,
                    help="subset of: full symmetric emulated emulated_symmetric seqfine (default: full symmetric)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    t0 = time.time()
    w = workloads.config(3, with_eig=True)
    print(json.dumps({"stage": "inputs", "seconds": time.time() - t0}), flush=True)
    t0 = time.time()
    sp = spectral.solve(w.eigvals, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    ref = spectral.reconstruct(w.eigvecs, sp["X"])
    print(json.dumps({"stage": "spectral_oracle", "seconds": time.time() - t0, "k_done": sp["k_done"],
                      "deltas": sp["deltas"]}), flush=True)
    s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
    table = {"full": (0, 0), "symmetric": (1, 0), "emulated": (0, 16), "emulated_symmetric": (1, 16)}
    names = args.modes
    if names is None:
        names = [m for m, skip in (("full", args.skip_full), ("symmetric", args.skip_sym)) if not skip]
    if "seqfine" in names:   # the K = N reference: 64 slices x 128 RK4 steps, sequential
        names = [m for m in names if m != "seqfine"]
        q = s.sequential_fine()
        X = s.result()
        rel = float(np.linalg.norm(X - ref) / np.linalg.norm(ref))
        print(json.dumps({"stage": "sequential_fine", "ms": q["ms_total"],
                          "fine_tflops": q["fine_flops"] / (q["ms_total"] * 1e-3) / 1e12,
                          "rel_frob_vs_spectral_parareal": rel, "launches": q["gpu_launches"]}), flush=True)
    modes = [(m, *table[m]) for m in names]
    for name, sym, emu in modes:
        s.set_option("symmetric", sym)
        s.set_option("emulation", emu)
        info = s.solve(w.K_max, w.tol, w.stop)
        X = s.result()
        rel = float(np.linalg.norm(X - ref) / np.linalg.norm(ref))
        print(json.dumps({"stage": name, "time_to_tol_ms": info["ms_total"], "k_done": info["k_done"],
                          "status": info["status"], "deltas": info["deltas"], "rel_frob_vs_spectral": rel,
                          "fine_algorithmic_tflops": info["fine_flops"] / (info["ms_total"] * 1e-3) / 1e12,
                          "fine_kernel_tflops": (info["fine_kernel_flops"] / (info["fine_kernel_ms"] * 1e-3) / 1e12
                                                 if info["fine_kernel_ms"] > 0 else None),
                          "residual": s.residual(), "launches": info["gpu_launches"]}), flush=True)


if __name__ == "__main__":
    main()
