"""Dense FP64 oracle: classical parareal (Algorithm 1) for a matrix ODE dX/dt = F(X).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain, slow, obviously correct: every step
below is written in the order and notation of the paper; the only library primitive is the
matrix product (numpy ``@``).  No blocking, fusion or reordering.

Citations (P:n = PAPER.md line n):
  * inverse flow F(X) = X (I - A) X, X(0) = I, X(1) = A^{-1}             P:44 (§1); eq. (eqQ)
  * steady-state flow dX/dt = F(X), F(X*) = 0 <=> X* = f(A)              P:46-51 eq. (stat)
    (instance F(X) = A - X^2, X* = A^{1/2}: BASELINE.json north star)
  * exponential flow dQ/dt = A Q, Q(0) = I, Q(1) = exp(A)                 Example 2
  * affine (linear inhomogeneous) flow dU/dt = A U + G, U(0) = U0          eq. (eq1) P:72-76 with a
    matrix state; Example 5's dX/dt = I - A X is the instance (A, G) -> (-A, I)
  * modified parareal: Algorithm 3 (homogeneous), Algorithm 4 (inhomogeneous,
    Step -1 and eq. (update2))
  * coarse propagator G = forward Euler                                   P:129, P:182 ("Euler explicit")
  * fine propagator F = Runge-Kutta ("Runge Kutta method can be applied") P:44; classical RK4 (R1)
  * Algorithm 1, Step 0 U^0_{n+1} = G(U^0_n), U^0_0 = u0                 P:136-139 eq. (eqStep0)
  * Step k+1: F(U^k_n) in parallel; U^{k+1}_{n+1} = G(U^{k+1}_n) + F(U^k_n) - G(U^k_n)
                                                                          P:143-147 eq. (eqStepk+1)
Readings:
  R1 classical RK4, S = ((k1 + 2 k2) + 2 k3) + k4, X <- X + (h/6) S
  R2 F(X) = X (B X) with B = I - A formed once
  R3 correction evaluated as F(U^k_n) + (G(U^{k+1}_n) - G(U^k_n))
  R4 U^{k+1}_0 = X0
  R5 K = number of correction sweeps after Step 0 (K = 0: coarse only)
  R6 stop on delta_{k+1} = ||U^{k+1}_N - U^k_N||_F / ||U^{k+1}_N||_F <= tol (or fixed K); the SPEC
     rule max_n ||U^{k+1}_n - U^k_n||_F / max(1, ||U_0||_F) <= tol is STOP_MAX_SLICE
  R10 residual stop ||A - U_N^2||_F / ||A||_F <= tol evaluated only for k >= 1
"""
from __future__ import annotations

import math
from typing import Callable, Optional

import numpy as np

FLOW_INVERSE = 0
FLOW_SQRT = 1
FLOW_EXP = 2
FLOW_TRIG = 3
FLOW_AFFINE = 4
STOP_FIXED_K = 0
STOP_DELTA = 1
STOP_RESIDUAL = 2
STOP_MAX_SLICE = 3   # SPEC classical_parareal: max_n ||U^{k+1}_n - U^k_n|| <= tol max(1, ||U_0||)


# ----------------------------------------------------------------------------------------------
# Right-hand sides F(X)
# ----------------------------------------------------------------------------------------------
def rhs_inverse(B: np.ndarray) -> Callable:
    """F(X) = X (I - A) X with B = I - A (R2: X @ (B @ X))."""
    return lambda X: X @ (B @ X)


def rhs_sqrt(A: np.ndarray) -> Callable:
    """F(X) = A - X^2 (steady state X* = A^{1/2}; P:46-51 with the north-star instance)."""
    return lambda X: A - X @ X


def rhs_exp(A: np.ndarray) -> Callable:
    """F(X) = A X, X(0) = I  =>  X(1) = exp(A) (Example 2, eq. eqQ)."""
    return lambda X: A @ X


def rhs_trig(A: np.ndarray) -> Callable:
    """Example 3, eq. (eqB) with X0 = 0: U = (X; Y) stacked 2n x n,
    dX/dt = A Y, dY/dt = -A X, U(0) = (0; I)  =>  U(1) = (sin A; cos A)."""
    n = A.shape[0]
    return lambda U: np.vstack([A @ U[n:], -(A @ U[:n])])


def rhs_affine(A: np.ndarray, Gsrc: np.ndarray) -> Callable:
    """F(U) = A U + G: the linear inhomogeneous problem du/dt = A u + g of eq. (eq1) with
    a matrix state (the "linear inhomogeneous case" of §3)."""
    return lambda U: A @ U + Gsrc


def initial_state(n: int, flow: int) -> np.ndarray:
    """X0 = I; the trig block flow starts at (sin 0; cos 0) = (0; I).
    The affine flow's default U0 is I as well (any U0 may be passed to the drivers)."""
    if flow == FLOW_TRIG:
        return np.vstack([np.zeros((n, n)), np.eye(n)])
    return np.eye(n)


def make_rhs(A: np.ndarray, flow: int, source: Optional[np.ndarray] = None) -> Callable:
    if flow == FLOW_INVERSE:
        B = np.eye(A.shape[0]) - A          # formed once (R2)
        return rhs_inverse(B)
    if flow == FLOW_SQRT:
        return rhs_sqrt(A)
    if flow == FLOW_EXP:
        return rhs_exp(A)
    if flow == FLOW_TRIG:
        return rhs_trig(A)
    if flow == FLOW_AFFINE:
        n = A.shape[0]
        return rhs_affine(A, np.zeros((n, n)) if source is None else np.asarray(source, dtype=np.float64))
    raise ValueError(f"unknown flow {flow}")


# ----------------------------------------------------------------------------------------------
# Propagators
# ----------------------------------------------------------------------------------------------
def euler(rhs: Callable, X, h: float, m: int):
    """Coarse propagator G: m forward-Euler steps X <- X + h F(X)."""
    for _ in range(m):
        X = X + h * rhs(X)
    return X


def rk4(rhs: Callable, X, h: float, m: int):
    """Fine propagator F: m classical RK4 steps (P:44 'Runge Kutta'; reading R1)."""
    for _ in range(m):
        k1 = rhs(X)
        k2 = rhs(X + (h / 2) * k1)
        k3 = rhs(X + (h / 2) * k2)
        k4 = rhs(X + h * k3)
        S = ((k1 + 2 * k2) + 2 * k3) + k4
        X = X + (h / 6) * S
    return X


def frob(X) -> float:
    return float(np.sqrt(np.sum(np.asarray(X, dtype=np.float64) ** 2)))


# ----------------------------------------------------------------------------------------------
# Algorithm 1 (classical parareal), generic over the state type
# ----------------------------------------------------------------------------------------------
def parareal(rhs: Callable, X0, T: float, N: int, m_G: int, m_F: int, K_max: int,
             tol: float = 0.0, stop: int = STOP_FIXED_K, norm: Callable = frob,
             residual: Optional[Callable] = None, skip_prefix: bool = False,
             keep_history: bool = False) -> dict:
    """Classical parareal on [0, T] with N uniform slices.

    G(x) = euler(rhs, x, T/(N m_G), m_G); F(x) = rk4(rhs, x, T/(N m_F), m_F).
    Returns dict(X=U_N, U=[U_0..U_N], k_done, deltas, residuals, converged[, history]).

    skip_prefix: at sweep k (0-based), F(U^k_n) for n < k equals the previous sweep's value
    bitwise and the correction leaves U_{n+1} unchanged (R3/R14), so both are skipped.  The
    literal algorithm (skip_prefix=False) is the default; tests check the two agree bitwise.
    """
    if K_max < 0 or N < 1 or m_G < 1 or m_F < 1:
        raise ValueError("invalid parareal parameters")
    hG = T / (N * m_G)
    hF = T / (N * m_F)
    G = lambda x: euler(rhs, x, hG, m_G)
    F = lambda x: rk4(rhs, x, hF, m_F)

    # Step 0 (eq. eqStep0): U^0_{n+1} = G(U^0_n), U^0_0 = u0
    U = [X0]
    Gold = []
    for n in range(N):
        g = G(U[n])
        Gold.append(g)
        U.append(g)
    deltas, residuals = [], []
    history = [list(U)] if keep_history else None
    res0 = residual(U[N]) if residual is not None else None
    k_done = 0
    converged = stop == STOP_FIXED_K
    Fk = [None] * N
    for k in range(K_max):
        # Step k+1, part 1: F(U^k_n) for all n ("compute in parallel")
        first = k if skip_prefix else 0
        for n in range(first, N):
            Fk[n] = F(U[n])
        # Step k+1, part 2: sequential correction (eq. eqStepk+1), evaluated as F + (Gnew - Gold)
        V = list(U)
        V[0] = X0                                             # R4
        for n in range(first, N):
            g = G(V[n])
            V[n + 1] = Fk[n] + (g - Gold[n])                  # R3
            Gold[n] = g
        if stop == STOP_MAX_SLICE:
            delta = max(norm(V[n] - U[n]) for n in range(N + 1)) / max(1.0, norm(X0))
        else:
            delta = norm(V[N] - U[N]) / norm(V[N])
        U = V
        k_done = k + 1
        deltas.append(delta)
        if residual is not None:
            residuals.append(residual(U[N]))
        if keep_history:
            history.append(list(U))
        if stop in (STOP_DELTA, STOP_MAX_SLICE) and delta <= tol:
            converged = True
            break
        if stop == STOP_RESIDUAL and residuals[-1] <= tol:      # k >= 1 by construction (R10)
            converged = True
            break
        if k_done == N:
            # After N sweeps U^N_n is the sequential fine solution (Remark P:155-157); further
            # sweeps are identities, so the iteration stops here converged (reading R15).
            converged = True
            break
    out = dict(X=U[N], U=U, k_done=k_done, deltas=deltas, residuals=residuals,
               residual0=res0, converged=converged)
    if keep_history:
        out["history"] = history
    return out


def frob_inner(A, B) -> float:
    """<A, B>_F = tr(B^T A)."""
    return float(np.sum(np.asarray(A) * np.asarray(B)))


def global_qr(Z: list, Q: list, rank_tol: float = 1e-12, passes: int = 2):
    """Algorithm 2 (globalQR), extending an existing F-orthonormal family Q (the Remark
    of Algorithm 3: the basis of S^k completes that of S^{k-1}).  For each block Z_i in order:
    Q = Z_i; for j: r_ji = <Q, Q_j>_F, Q = Q - r_ji Q_j; r_ii = ||Q||_F; keep Q / r_ii unless
    r_ii is zero -- read as r_ii <= rank_tol * max(1, ||Z_i||_F) (reading R16).
    Floating-point reading R17: the j-loop runs `passes` = 2 times ("twice is enough"
    reorthogonalisation).  In exact arithmetic the second pass subtracts exact zeros, so it is
    Algorithm 2; in FP64 a single pass loses orthogonality once the iterates become nearly
    dependent (they converge), and the modified parareal then diverges (tests pin both).
    Returns the list of indices (into Z) of the kept blocks; Q is extended in place."""
    kept = []
    for i, Zi in enumerate(Z):
        q = Zi
        for _ in range(passes):
            for Qj in Q:
                r = frob_inner(q, Qj)
                q = q - r * Qj
        rii = frob(q)
        if rii > rank_tol * max(1.0, frob(Zi)):
            Q.append(q / rii)
            kept.append(i)
    return kept


def modified_parareal(rhs: Callable, X0, T: float, N: int, m_G: int, m_F: int, K_max: int,
                      tol: float = 0.0, stop: int = STOP_FIXED_K, rank_tol: float = 1e-12,
                      keep_history: bool = False) -> dict:
    """Algorithm 3: modified parareal for a linear homogeneous flow.
      Step 0: U^0_{n+1} = G(U^0_n), U^0_0 = U_0; S^{-1} = {}.
      Step k+1: S^k = span(S^{k-1} u {U^k_n, n = 0..N}) by globalQR (basis Q, completed);
                F(Q_new) "in parallel" for the new blocks only (autonomous flow on a uniform grid:
                one image per block serves every n);
                U^{k+1}_{n+1} = F(P^k U^{k+1}_n) + G((I - P^k) U^{k+1}_n)          eq. (eq_update)
                with P^k U = sum_i alpha_i Q_i, alpha = Q^T <> U, F(P U) = sum_i alpha_i F(Q_i).
    """
    hG = T / (N * m_G)
    hF = T / (N * m_F)
    G = lambda x: euler(rhs, x, hG, m_G)
    F = lambda x: rk4(rhs, x, hF, m_F)
    U = [X0]
    for n in range(N):
        U.append(G(U[n]))
    Q, FQ = [], []
    deltas = []
    history = [list(U)] if keep_history else None
    k_done = 0
    converged = stop == STOP_FIXED_K
    for k in range(min(K_max, N)):
        nb_old = len(Q)
        global_qr(U, Q, rank_tol)
        for Qi in Q[nb_old:]:
            FQ.append(F(Qi))
        V = [X0]
        for n in range(N):
            alpha = [frob_inner(Qi, V[n]) for Qi in Q]
            PV = sum(a * Qi for a, Qi in zip(alpha, Q))
            FPV = sum(a * Fi for a, Fi in zip(alpha, FQ))
            V.append(FPV + G(V[n] - PV))
        delta = frob(V[N] - U[N]) / frob(V[N])
        U = V
        k_done = k + 1
        deltas.append(delta)
        if keep_history:
            history.append(list(U))
        if stop == STOP_DELTA and delta <= tol:
            converged = True
            break
        if k_done == N:
            converged = True
            break
    out = dict(X=U[N], U=U, k_done=k_done, deltas=deltas, converged=converged, basis=len(Q))
    if keep_history:
        out["history"] = history
    return out


def modified_parareal_inhom(rhs: Callable, X0, T: float, N: int, m_G: int, m_F: int, K_max: int,
                            tol: float = 0.0, stop: int = STOP_FIXED_K, rank_tol: float = 1e-12,
                            keep_history: bool = False) -> dict:
    """Algorithm 4: modified parareal for a linear INhomogeneous (affine) flow.
      Step -1: F(T_{n+1}, T_n, 0) and G(T_{n+1}, T_n, 0) -- the flow is autonomous and the grid
               uniform, so one F(0) and one G(0) serve every n (the same reading R18 as the fine
               images of Algorithm 3).
      Step 0:  identical to the homogeneous case, U^0_{n+1} = G(U^0_n), U^0_0 = U_0.
      Step k+1: enhance S^k with U^k_0..U^k_N by globalQR (basis completed), F(Q_new) in parallel,
               then eq. (update2):
                 U^{k+1}_{n+1} = F(P_k U^{k+1}_n) + G((I - P_k) U^{k+1}_n) - G(0)
               with the affine computation of the Remark:
                 F(P_k U) = sum_i alpha_i {F(Q_i) - F(0)} + F(0),   P_k U = sum_i alpha_i Q_i.
    With a zero source F(0) = G(0) = 0 exactly and this is Algorithm 3 bitwise (pinned)."""
    hG = T / (N * m_G)
    hF = T / (N * m_F)
    G = lambda x: euler(rhs, x, hG, m_G)
    F = lambda x: rk4(rhs, x, hF, m_F)
    Z0 = np.zeros_like(X0)
    F0 = F(Z0)                                               # Step -1
    G0 = G(Z0)
    U = [X0]                                                 # Step 0
    for n in range(N):
        U.append(G(U[n]))
    Q, FQ = [], []
    deltas = []
    history = [list(U)] if keep_history else None
    k_done = 0
    converged = stop == STOP_FIXED_K
    for k in range(min(K_max, N)):
        nb_old = len(Q)
        global_qr(U, Q, rank_tol)
        for Qi in Q[nb_old:]:
            FQ.append(F(Qi))
        V = [X0]
        for n in range(N):
            alpha = [frob_inner(Qi, V[n]) for Qi in Q]
            PV = sum(a * Qi for a, Qi in zip(alpha, Q))
            FPV = sum(a * (Fi - F0) for a, Fi in zip(alpha, FQ)) + F0     # Remark
            V.append(FPV + G(V[n] - PV) - G0)                              # eq. (update2)
        delta = frob(V[N] - U[N]) / frob(V[N])
        U = V
        k_done = k + 1
        deltas.append(delta)
        if keep_history:
            history.append(list(U))
        if stop == STOP_DELTA and delta <= tol:
            converged = True
            break
        if k_done == N:
            converged = True
            break
    out = dict(X=U[N], U=U, k_done=k_done, deltas=deltas, converged=converged, basis=len(Q), F0=F0, G0=G0)
    if keep_history:
        out["history"] = history
    return out


def solve_modified(A: np.ndarray, flow: int, T: float, N: int, m_G: int, m_F: int, K_max: int,
                   tol: float = 0.0, stop: int = STOP_FIXED_K, keep_history: bool = False,
                   source: Optional[np.ndarray] = None, X0: Optional[np.ndarray] = None) -> dict:
    """Algorithm 3 for the homogeneous flows (exp, trig); Algorithm 4 for the affine flow."""
    A = np.asarray(A, dtype=np.float64)
    x0 = initial_state(A.shape[0], flow) if X0 is None else np.asarray(X0, dtype=np.float64)
    if flow == FLOW_AFFINE:
        return modified_parareal_inhom(make_rhs(A, flow, source), x0, T, N, m_G, m_F, K_max, tol, stop,
                                       keep_history=keep_history)
    if flow not in (FLOW_EXP, FLOW_TRIG):
        raise ValueError("Algorithm 3 is for linear homogeneous flows (exp, trig); Algorithm 4 for affine")
    return modified_parareal(make_rhs(A, flow), x0, T, N, m_G, m_F, K_max, tol,
                             stop, keep_history=keep_history)


def sequential_fine(rhs: Callable, X0, T: float, N: int, m_F: int) -> list:
    """The reference the paper compares against: S_0 = X0, S_{n+1} = F(S_n)."""
    hF = T / (N * m_F)
    S = [X0]
    for n in range(N):
        S.append(rk4(rhs, S[n], hF, m_F))
    return S


# ----------------------------------------------------------------------------------------------
# Flow-level drivers and residuals (the matrix-function view, Example 1 P:167-176)
# ----------------------------------------------------------------------------------------------
def residual_inverse(A: np.ndarray, X: np.ndarray) -> float:
    """||A X - I||_F / sqrt(n): X(1) = A^{-1}."""
    n = A.shape[0]
    return frob(A @ X - np.eye(n)) / math.sqrt(n)


def residual_sqrt(A: np.ndarray, X: np.ndarray) -> float:
    """||A - X^2||_F / ||A||_F: F(X*) = 0 at the steady state."""
    return frob(A - X @ X) / frob(A)


def flow_residual(A: np.ndarray, flow: int) -> Optional[Callable]:
    if flow == FLOW_INVERSE:
        return lambda X: residual_inverse(A, X)
    if flow == FLOW_SQRT:
        return lambda X: residual_sqrt(A, X)
    return None     # the exp and trig flows have no residual of this kind


def solve(A: np.ndarray, flow: int, T: float, N: int, m_G: int, m_F: int, K_max: int,
          tol: float = 0.0, stop: int = STOP_FIXED_K, skip_prefix: bool = True,
          keep_history: bool = False, source: Optional[np.ndarray] = None,
          X0: Optional[np.ndarray] = None) -> dict:
    """f(A) by parareal on the flow's ODE with X0 = I; the affine flow takes a source G
    and an optional U0."""
    A = np.asarray(A, dtype=np.float64)
    rhs = make_rhs(A, flow, source)
    X0 = initial_state(A.shape[0], flow) if X0 is None else np.asarray(X0, dtype=np.float64)
    # the residual is recorded for every flow; it drives the stop only for STOP_RESIDUAL
    return parareal(rhs, X0, T, N, m_G, m_F, K_max, tol, stop, frob, flow_residual(A, flow),
                    skip_prefix, keep_history)


def solve_sequential_fine(A: np.ndarray, flow: int, T: float, N: int, m_F: int,
                          source: Optional[np.ndarray] = None, X0: Optional[np.ndarray] = None) -> np.ndarray:
    A = np.asarray(A, dtype=np.float64)
    x0 = initial_state(A.shape[0], flow) if X0 is None else np.asarray(X0, dtype=np.float64)
    return sequential_fine(make_rhs(A, flow, source), x0, T, N, m_F)[N]


def accel_inverse(A: np.ndarray, E0, dt: float, steps: int, X0=None):
    """Algorithm 8 (Example 5), literally:
      X^(0) = X0; u^(0) = e (given, e ~ A^{-1} - X0);
      for k: X^(k+1) = X^(k) + dt (I - A X^(k) + u^(k));  u^(k+1) = (I - dt A) u^(k).
    Returns the list of iterates X^(0..steps)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    I = np.eye(n)
    X = np.zeros((n, n)) if X0 is None else np.asarray(X0, dtype=np.float64)
    u = np.zeros((n, n)) if E0 is None else np.asarray(E0, dtype=np.float64)
    out = [X]
    for _ in range(steps):
        X, u = X + dt * ((I - A @ X) + u), u - dt * (A @ u)
        out.append(X)
    return out


def cosine_algorithm5(A: np.ndarray, N: int, m_G: int, m_F: int, K_max: int, tol: float = 0.0,
                      stop: int = STOP_FIXED_K):
    """Algorithm 5, steps in the paper's order:
      1. the smallest non-negative integer m with 2^{-m} ||A||_inf <= 1;
      2. A0 = 2^{-m} A;
      3. C0 = cos(A0) by parareal on the trig block flow (eq. eqB, T = 1; classical parareal here);
      4. C_{i+1} = 2 C_i^2 - I for i = 0..m-1;  X = C_m.
    Returns (C_m, m, parareal output)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    norm_inf = np.abs(A).sum(axis=1).max()
    m = 0
    while 2.0 ** (-m) * norm_inf > 1.0:
        m += 1
    A0 = A * 2.0 ** (-m)
    out = solve(A0, FLOW_TRIG, 1.0, N, m_G, m_F, K_max, tol, stop)
    C = out["X"][n:]
    for _ in range(m):
        C = 2.0 * (C @ C) - np.eye(n)
    return C, m, out
