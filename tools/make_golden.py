"""Writes tests/golden/scalar_parareal_mp50.txt: 50-digit values of the scalar parareal iterate
u^K_N(lam) (inverse flow T=1, sqrt flow T=4), computed by oracle.spectral.mp_parareal_scalar only.
Key: flow:lam:N:m_G:m_F:K."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mpmath as mp  # noqa: E402

from oracle import spectral  # noqa: E402

CASES = [
    (0, 0.5, 8, 1, 64, 4), (0, 1.5, 8, 1, 64, 4), (0, 1.25, 16, 1, 128, 6), (0, 0.1, 8, 2, 32, 3),
    (0, 10.0, 8, 2, 32, 3), (1, 2.0, 8, 2, 16, 2), (1, 9.0, 8, 2, 16, 2),
]

out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "scalar_parareal_mp50.txt")
with open(out, "w") as f:
    f.write("# u^K_N(lam) of scalar classical parareal, 50 digits (oracle.spectral.mp_parareal_scalar).\n")
    f.write("# Written by tools/make_golden.py; key = flow:lam:N:m_G:m_F:K (flow 0 T=1, flow 1 T=4).\n")
    for flow, lam, N, mG, mF, K in CASES:
        T = 1 if flow == 0 else 4
        x, _ = spectral.mp_parareal_scalar(lam, flow, T, N, mG, mF, K)
        f.write(f"{flow}:{lam}:{N}:{mG}:{mF}:{K} = {mp.nstr(x, 30)}\n")
print("wrote", out)
