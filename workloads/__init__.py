"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no flow, propagator or parareal step): it only
builds the input matrix A of each BASELINE.json config plus, where known, its eigen-decomposition
(which the spectral oracle needs).  Both sides read the same bytes of A.

Configs (BASELINE.json "configs", 0-based; recipes SURVEY.md §8(d)):
  0  inverse, n=32,   A = Q diag(lam) Q^T, Q from QR of default_rng(0) N(0,1), lam ~ U[0.5,1.5)
  1  inverse, n=256,  A = I + 0.25 tridiag(-1,2,-1)                (shifted 1D Laplacian)
  2  inverse, n=1024, A = Q diag(lam) Q^T, default_rng(2), lam = 10^U[-1,1)
  3  inverse, n=4096, A = I + G^T G / (2n), G ~ default_rng(3) N(0,1)
  4  sqrt,    n=4096, A = 2D 5-point Laplacian on a 64x64 grid (Dirichlet) + I   (P:702 analogue)
The paper's workloads are synthetic Laplacians; no dataset is involved.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

FLOW_INVERSE = 0   # F(X) = X (I - A) X, X0 = I, T = 1   => X(1) = A^{-1}    (eq. eqQ)
FLOW_SQRT = 1      # F(X) = A - X^2,     X0 = I, T large => X* = A^{1/2}   (north star)
FLOW_EXP = 2       # F(X) = A X,         X0 = I, T = 1   => X(1) = exp(A)   (Example 2)

STOP_FIXED_K = 0   # run exactly K_max correction sweeps
STOP_DELTA = 1     # ||U_N^{k+1} - U_N^k||_F / ||U_N^{k+1}||_F <= tol   (BJ cfg[1]; reading R6)
STOP_RESIDUAL = 2  # ||A - U_N^2||_F / ||A||_F <= tol, checked for k >= 1  (BJ cfg[4]; reading R10)


@dataclasses.dataclass
class Workload:
    name: str
    A: np.ndarray                 # (n, n) float64, C-contiguous, row-major
    flow: int
    T: float
    N: int                        # time slices
    m_G: int                      # coarse Euler steps per slice
    m_F: int                      # fine RK4 steps per slice
    K_max: int
    tol: float
    stop: int
    eigvecs: Optional[np.ndarray] = None   # V with A = V diag(eigvals) V^T (None if unknown)
    eigvals: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return self.A.shape[0]


def _symmetrise(A: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(0.5 * (A + A.T))


def spd_from_spectrum(n: int, rng: np.random.Generator, lam: np.ndarray):
    """A = Q diag(lam) Q^T with Q from the QR of a seeded N(0,1) matrix (draw order: Z first)."""
    Z = rng.standard_normal((n, n))
    Q, _ = np.linalg.qr(Z)
    A = _symmetrise((Q * lam) @ Q.T)
    return A, Q


def laplacian_1d(n: int) -> np.ndarray:
    """tridiag(-1, 2, -1), unscaled (reading R11)."""
    L = 2.0 * np.eye(n)
    i = np.arange(n - 1)
    L[i, i + 1] = -1.0
    L[i + 1, i] = -1.0
    return L


def laplacian_1d_eig(n: int):
    """Closed-form eigenpairs of tridiag(-1,2,-1): v_j(i) = sqrt(2/(n+1)) sin(i j pi/(n+1)),
    mu_j = 4 sin^2(j pi / (2(n+1))), i, j = 1..n."""
    j = np.arange(1, n + 1)
    V = np.sqrt(2.0 / (n + 1)) * np.sin(np.outer(j, j) * np.pi / (n + 1))
    mu = 4.0 * np.sin(j * np.pi / (2.0 * (n + 1))) ** 2
    return V, mu


def laplacian_2d(m: int) -> np.ndarray:
    """5-point Dirichlet Laplacian on an m x m grid (diag 4, -1 neighbours), n = m^2, dense."""
    L1 = laplacian_1d(m)
    I = np.eye(m)
    return np.kron(L1, I) + np.kron(I, L1)


def config(i: int, *, with_eig: bool = True) -> Workload:
    """The i-th BASELINE.json config (0-based)."""
    if i == 0:
        rng = np.random.default_rng(0)
        n = 32
        Z = rng.standard_normal((n, n))
        Q, _ = np.linalg.qr(Z)
        lam = rng.uniform(0.5, 1.5, n)
        A = _symmetrise((Q * lam) @ Q.T)
        return Workload("cfg0_inverse_n32", A, FLOW_INVERSE, 1.0, 8, 1, 64, 4, 0.0, STOP_FIXED_K, Q, lam)
    if i == 1:
        n = 256
        A = np.eye(n) + 0.25 * laplacian_1d(n)
        V, mu = laplacian_1d_eig(n)
        return Workload("cfg1_inverse_n256", A, FLOW_INVERSE, 1.0, 16, 1, 128, 16, 1e-10, STOP_DELTA,
                        V, 1.0 + 0.25 * mu)
    if i == 2:
        rng = np.random.default_rng(2)
        n = 1024
        Z = rng.standard_normal((n, n))
        Q, _ = np.linalg.qr(Z)
        lam = 10.0 ** rng.uniform(-1.0, 1.0, n)
        A = _symmetrise((Q * lam) @ Q.T)
        return Workload("cfg2_inverse_n1024", A, FLOW_INVERSE, 1.0, 64, 2, 256, 16, 1e-10, STOP_DELTA, Q, lam)
    if i == 3:
        rng = np.random.default_rng(3)
        n = 4096
        G = rng.standard_normal((n, n))
        A = _symmetrise(np.eye(n) + (G.T @ G) / (2.0 * n))
        V = lam = None
        if with_eig:
            lam, V = np.linalg.eigh(A)
        return Workload("cfg3_inverse_n4096", A, FLOW_INVERSE, 1.0, 64, 1, 128, 12, 1e-10, STOP_DELTA, V, lam)
    if i == 4:
        m = 64
        A = np.ascontiguousarray(laplacian_2d(m) + np.eye(m * m))
        V1, mu1 = laplacian_1d_eig(m)
        V = np.kron(V1, V1) if with_eig else None
        lam = 1.0 + (mu1[:, None] + mu1[None, :]).reshape(-1)
        # T = 20, N = 64, fine h = 5/512 (reading R8: dt=0.01 -> m_F = 32), m_G = 2 (reading R9)
        return Workload("cfg4_sqrt_n4096", A, FLOW_SQRT, 20.0, 64, 2, 32, 8, 1e-10, STOP_RESIDUAL, V, lam)
    raise ValueError(f"no config {i}")


def random_spd(n: int, seed: int, lo: float = 0.5, hi: float = 1.5) -> Workload:
    """Small seeded SPD case with a known spectrum (ragged sizes for parity tests)."""
    rng = np.random.default_rng(1000 + seed)
    Z = rng.standard_normal((n, n))
    Q, _ = np.linalg.qr(Z)
    lam = rng.uniform(lo, hi, n)
    A = _symmetrise((Q * lam) @ Q.T)
    return Workload(f"spd_n{n}_s{seed}", A, FLOW_INVERSE, 1.0, 4, 1, 8, 4, 0.0, STOP_FIXED_K, Q, lam)


def random_nonsymmetric(n: int, seed: int, scale: float = 0.3) -> np.ndarray:
    """I + scale * N(0,1)/sqrt(n): well conditioned, NOT symmetric (catches transposed operands)."""
    rng = np.random.default_rng(2000 + seed)
    return np.ascontiguousarray(np.eye(n) + scale * rng.standard_normal((n, n)) / np.sqrt(n))


def random_state(n: int, seed: int) -> np.ndarray:
    """A seeded dense state matrix (for kernel-level GEMM / elementwise parity)."""
    rng = np.random.default_rng(3000 + seed)
    return rng.standard_normal((n, n))
