"""Spectral oracle: the parareal iteration run per eigenvalue (SURVEY.md §8(c) pin P1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

With X0 = I every quantity of the algorithm (Euler/RK4 stages, corrections) is a polynomial in A
with scalar coefficients, so for A = V diag(lam) V^T every iterate is U^k_n = V diag(u^k_n(lam)) V^T
where u^k_n is the SAME algorithm applied to the scalar ODE
    inverse: q' = q ((1 - lam) q)        (the eigen-image of X (I - A) X)
    sqrt:    x' = lam - x^2              (the eigen-image of A - X^2)
    exp:     x' = lam x                  (the eigen-image of A X, Example 2 P:193-201)
    affine:  x' = lam x + gamma          (the eigen-image of A U + G when G = V diag(gamma) V^T
                                          commutes with A, eq. (eq1))
with x0 = 1 (the affine flow takes any x0 = eigen-coefficients of a U0 that commutes with A).  This is the paper's own diagonalisation argument.  Frobenius norms of
V diag(u) V^T are 2-norms of u (V orthogonal), so the delta/residual stop tests carry over.
The state of the generic dense.parareal is then a length-n vector of scalars (elementwise ops).

mp_parareal_scalar runs the same recursion in mpmath with `dps` digits: a high-precision twin
used to pin the FP64 paths (P2).
"""
from __future__ import annotations

import math

import numpy as np

from . import dense


def scalar_rhs(lam, flow: int, gamma=None):
    if flow == dense.FLOW_INVERSE:
        b = 1.0 - lam
        return lambda q: q * (b * q)
    if flow == dense.FLOW_SQRT:
        return lambda x: lam - x * x
    if flow == dense.FLOW_EXP:
        return lambda x: lam * x
    if flow == dense.FLOW_TRIG:       # state (s, c): s' = lam c, c' = -lam s  (eq. eqB per eigenvalue)
        return lambda u: np.stack([lam * u[1], -(lam * u[0])])
    if flow == dense.FLOW_AFFINE:
        return lambda x: lam * x + gamma
    raise ValueError(flow)


def solve(eigvals: np.ndarray, flow: int, T: float, N: int, m_G: int, m_F: int, K_max: int,
          tol: float = 0.0, stop: int = dense.STOP_FIXED_K, keep_history: bool = False,
          gamma=None, x0=None) -> dict:
    """Scalar parareal for every eigenvalue at once (vectorised over lam). Returns the dense
    dict shape with X/U entries as eigen-coefficient vectors u (reconstruct with `reconstruct`).
    Affine flow: gamma = eigen-coefficients of the source, x0 = those of U0 (default 1)."""
    lam = np.asarray(eigvals, dtype=np.float64)
    if flow == dense.FLOW_AFFINE:
        gamma = np.broadcast_to(np.asarray(0.0 if gamma is None else gamma, dtype=np.float64), lam.shape).copy()
    rhs = scalar_rhs(lam, flow, gamma)
    if x0 is not None:
        x0 = np.broadcast_to(np.asarray(x0, dtype=np.float64), lam.shape).copy()
    elif flow == dense.FLOW_TRIG:
        x0 = np.stack([np.zeros_like(lam), np.ones_like(lam)])
    else:
        x0 = np.ones_like(lam)
    norm = lambda u: float(np.sqrt(np.sum(u * u)))
    if flow == dense.FLOW_INVERSE:
        # ||A X - I||_F / sqrt(n) = ||lam u - 1||_2 / sqrt(n)
        residual = lambda u: norm(lam * u - 1.0) / math.sqrt(lam.size)
    elif flow in (dense.FLOW_EXP, dense.FLOW_TRIG, dense.FLOW_AFFINE):
        residual = None
    else:
        # ||A - X^2||_F / ||A||_F = ||lam - u^2||_2 / ||lam||_2
        residual = lambda u: norm(lam - u * u) / norm(lam)
    return dense.parareal(rhs, x0, T, N, m_G, m_F, K_max, tol, stop, norm, residual,
                          skip_prefix=True, keep_history=keep_history)


def reconstruct(V: np.ndarray, u: np.ndarray) -> np.ndarray:
    """V diag(u) V^T (for a trig state (2, n): the stack [V diag(s) V^T; V diag(c) V^T])."""
    if u.ndim == 2:
        return np.vstack([(V * u[0]) @ V.T, (V * u[1]) @ V.T])
    return (V * u) @ V.T


def mp_parareal_scalar(lam, flow: int, T, N: int, m_G: int, m_F: int, K_max: int, dps: int = 50):
    """The scalar recursion in mpmath at `dps` digits; returns (u_N as mpf, deltas)."""
    import mpmath as mp
    with mp.workdps(dps):
        lam_ = mp.mpf(lam)
        rhs = scalar_rhs(lam_, flow)
        out = dense.parareal(rhs, mp.mpf(1), mp.mpf(T), N, m_G, m_F, K_max, 0.0,
                             dense.STOP_FIXED_K, norm=lambda x: abs(x), skip_prefix=False)
        return out["X"], out["U"]
