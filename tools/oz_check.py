"""Quick GPU check of the emulated FP64 GEMM (mfode_dgemm_emulated): error vs the a-priori bound and
timing against the DMMA GEMM.  python tools/oz_check.py [n ...]"""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_07959_b200 as mf  # noqa: E402

U = 2.0 ** -53


def abits(nmod, n):
    mods = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193][:nmod]
    l2 = sum(math.log2(m) for m in mods)
    kb = max(0, math.ceil(math.log2(n))) if n > 1 else 0
    return math.floor((l2 - 2 - kb) / 2 - 1e-9)


def bound(A, B, a):
    ea = np.ceil(np.log2(np.maximum(np.abs(A).max(1), 1e-300)) + 1e-15)
    eb = np.ceil(np.log2(np.maximum(np.abs(B).max(0), 1e-300)) + 1e-15)
    sa = 2.0 ** ea
    sb = 2.0 ** eb
    q = 2.0 ** -(a + 1)
    return (q * (sa[:, None] * np.abs(B).sum(0)[None, :] + sb[None, :] * np.abs(A).sum(1)[:, None])
            + 2 * A.shape[0] * U * (np.abs(A) @ np.abs(B)) + q * q * A.shape[0] * sa[:, None] * sb[None, :])


def check(n, nmod=16, ld=None):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (1, n)))
    ld = ld or ((n + 15) // 16 * 16)
    dA = torch.zeros((n, ld), dtype=torch.float64, device="cuda")[:, :n]
    dB = torch.zeros((n, ld), dtype=torch.float64, device="cuda")[:, :n]
    dA.copy_(torch.from_numpy(A))
    dB.copy_(torch.from_numpy(B))
    D = mf.dgemm_emulated(dA, dB, n_moduli=nmod)
    torch.cuda.synchronize()
    D = D.cpu().numpy()
    ref = A @ B
    err = np.abs(D - ref)
    b = bound(A, B, abits(nmod, n))
    print(f"n={n} nmod={nmod} a={abits(nmod, n)} max|err|={err.max():.3e} max(err/bound)={(err / b).max():.3f} "
          f"relF={np.linalg.norm(D - ref) / np.linalg.norm(ref):.3e}", flush=True)
    return float((err / b).max())


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def set_pair(v):
    s = mf.Solver(np.eye(2), mf.FLOW_INVERSE, 1.0, 1, 1, 1)
    s.set_option("oz_pair", v)
    s.close()


if __name__ == "__main__":
    ns = [int(x) for x in sys.argv[1:]] or [1, 8, 30, 100, 128, 129, 256, 300, 1000]
    for pair in (1, 0):
        set_pair(pair)
        print("oz_pair", pair)
        for n in ns:
            check(n)
        for nmod in (8, 12, 14, 16):
            check(512, nmod)
    n = 4096
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    B = torch.randn(n, n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(A)
    t = timeit(lambda: mf.dgemm(A, B, out=out))
    print(f"dmma n={n}: {t:.3f} ms {2 * n ** 3 / t / 1e9:.1f} TF/s", flush=True)
    for pair in (0, 1):
        set_pair(pair)
        for nmod in (12, 14, 16):
            t = timeit(lambda: mf.dgemm_emulated(A, B, out=out, n_moduli=nmod))
            print(f"pair={pair} emulated nmod={nmod} n={n}: {t:.3f} ms {2 * n ** 3 / t / 1e9:.1f} TF/s "
                  f"(FP64-equivalent)", flush=True)
    ref = torch.matmul(A, B)
    D = mf.dgemm_emulated(A, B, n_moduli=16)
    print("relF vs cuBLAS", float(torch.linalg.norm(D - ref) / torch.linalg.norm(ref)))
