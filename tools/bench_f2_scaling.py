"""How the modified parareal (Algorithm 3) scales with the slice count N on
one B200: the device-side Gram-Schmidt (CGS2, R23) and the sequential update grow with the basis size
nb <= (N + 1)(K + 1), the fine images with nb.  Each line: N, basis size, solve time, fine-kernel time,
the sequential update (projections + coarse G), the rest (Gram-Schmidt, host syncs), and the fine
work's TFLOP/s over the whole solve.
    python tools/bench_f2_scaling.py [package_root] > profiles/f2_scaling_r02.jsonl
"""
import json
import os
import sys

ROOT = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import hashlib  # noqa: E402

import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    n, K, mF = 1024, 4, 32
    w = workloads.random_spd(n, 71, lo=0.5, hi=2.0)
    for N in (16, 32, 64):
        s = mf.Solver(w.A, mf.FLOW_EXP, 1.0, N, 1, mF)
        s.solve_modified(1)   # warm-up (allocates the basis storage)
        i = s.solve_modified(K)
        d = {k: v for k, v in i.items() if not isinstance(v, (list, tuple))}
        fine_ms = d.get("ms_fine") or 0.0
        print(json.dumps({
            "row": "f2", "what": "modified_parareal_alg3_exp", "n": n, "N": N, "m_F": mF, "K": K,
            "basis": d["basis_size"], "ms_total": d["ms_total"], "ms_fine_span": fine_ms,
            "ms_update": d["ms_correct"], "ms_rest": d["ms_total"] - fine_ms - d["ms_correct"],
            "fine_flops": d["fine_flops"], "tflops_whole": d["fine_flops"] / (d["ms_total"] * 1e-3) / 1e12,
            "gpu_launches": d["gpu_launches"], "result_md5": hashlib.md5(s.result().tobytes()).hexdigest()[:12],
            "lib": ROOT}), flush=True)
        s.close()
