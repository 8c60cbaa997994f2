"""Bounded persistence vs SMs held by other kernels (NCCL kernels parked on SMs add a tail to
every persistent fine launch).  cfg[4] solve time with cta_share_us 2000 / 500, with and without 8 SMs
occupied by a spinning kernel on another stream.  python tools/ab_sm_hog.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    hog = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsmhog.so"))
    hog.hog_launch.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
    w = workloads.config(4, with_eig=False)
    s = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F)
    side = torch.cuda.Stream()
    s.solve(w.K_max, w.tol, w.stop)
    for share in (2000, 500):
        s.set_option("cta_share_us", share)
        for nsm in (0, 8):
            if nsm:
                hog.hog_launch(nsm, 60.0, ctypes.c_void_p(side.cuda_stream))
            i = s.solve(w.K_max, w.tol, w.stop)
            print(json.dumps({"cta_share_us": share, "hogged_sms": nsm, "ms": i["ms_total"],
                              "fine_kernel_tflops": i["fine_kernel_flops"] / (i["fine_kernel_ms"] * 1e-3) / 1e12}),
                  flush=True)
            torch.cuda.synchronize()
