"""Fine-phase TF/s of one K = 1 sweep by DMMA tile configuration (option tile: 1 = 128 x 128, one CTA per
SM; 2 = 64 x 64, two CTAs per SM, one CTA's epilogue overlapping the other's main loop).
    python tools/tile_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    for n, N, mF in ((1024, 64, 8), (2048, 32, 4), (4096, 16, 2)):
        A = np.eye(n) + 0.25 * workloads.laplacian_1d(n)
        for flow in (mf.FLOW_INVERSE, mf.FLOW_SQRT):
            for tile in (1, 2):
                s = mf.Solver(A, flow, 1.0, N, 1, mF)
                s.set_option("tile", tile)
                s.solve(1)
                best = 0.0
                for _ in range(2):
                    i = s.solve(1)
                    best = max(best, i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12)
                print(json.dumps({"n": n, "N": N, "mF": mF, "flow": flow, "tile": tile, "fine_tflops": best}),
                      flush=True)
                s.close()
