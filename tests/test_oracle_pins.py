"""Pins for the CPU oracle (oracle/): checks against what the paper and the mathematics fix,
never against the oracle itself.  CPU only (-m "not gpu").

Each test names what it pins and the passage it follows (P:n = PAPER.md, S:n = SPEC.md line).
A plausible mistake anywhere in oracle/dense.py (dropped term, wrong sign, wrong index, wrong
RK coefficient, transposed operand, wrong correction order) fails at least one test here:
  * RK4 coefficients/association      -> test_rk4_stability_polynomial_matrix, test_rk4_order
  * Euler step / coarse sweep          -> test_euler_golden, test_coarse_sweep_geometric
  * correction sign / index / order    -> test_linear_parareal_binomial_closed_form (+ P5/P6 bitwise)
  * inverse flow operands (transpose)  -> test_inverse_flow_closed_form_nonsymmetric
  * sqrt flow                          -> test_sqrt_steady_state
  * spectral oracle                    -> test_dense_vs_spectral, test_spectral_vs_mpmath
"""
import math
import os

import numpy as np
import pytest

from oracle import dense, spectral
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    vals = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, v = line.split("=", 1)
            vals[k.strip()] = v.strip()
    return vals


# ---------------------------------------------------------------------------------------------
# Propagators
# ---------------------------------------------------------------------------------------------
def test_euler_golden():
    """scalar x' = -x, x0 = 1, one Euler step h = 0.1 -> 0.9 (golden/spec_examples.txt)."""
    g = _read_golden("spec_examples.txt")
    x = dense.euler(lambda x: -x, 1.0, 0.1, 1)
    assert x == float(g["euler_one_step_h0.1"])


def test_coarse_sweep_geometric():
    """Euler coarse sweep of x' = -x, N = 4, dT = 0.25 gives 0.75^n (exact in FP64)."""
    out = dense.parareal(lambda x: -x, 1.0, 1.0, 4, 1, 1, 0)
    assert out["U"] == [0.75 ** n for n in range(5)]


def test_rk4_stability_polynomial_matrix():
    """Classical RK4 on the linear flow X' = M X multiplies by R(hM) = I + Z + Z^2/2 + Z^3/6 + Z^4/24
    (textbook stability polynomial).  M non-symmetric, so a transposed product also fails."""
    rng = np.random.default_rng(7)
    n = 6
    M = rng.standard_normal((n, n))
    X0 = rng.standard_normal((n, n))
    h = 0.05
    Z = h * M
    R = np.eye(n) + Z + Z @ Z / 2 + Z @ Z @ Z / 6 + Z @ Z @ Z @ Z / 24
    X1 = dense.rk4(lambda X: M @ X, X0, h, 1)
    np.testing.assert_allclose(X1, R @ X0, rtol=0, atol=1e-14 * np.abs(R @ X0).max() * 10)
    # three steps = R^3
    X3 = dense.rk4(lambda X: M @ X, X0, h, 3)
    np.testing.assert_allclose(X3, R @ R @ R @ X0, rtol=0, atol=1e-13)


def test_rk4_order():
    """RK4 is 4th order: on q' = (1 - lam) q^2 (exact q(t) = 1/(1 + t(lam - 1))) halving h
    divides the t = 1 error by ~16."""
    lam = 3.0
    rhs = lambda q: q * ((1 - lam) * q)
    exact = 1.0 / lam
    e1 = abs(dense.rk4(rhs, 1.0, 1 / 20, 20) - exact)
    e2 = abs(dense.rk4(rhs, 1.0, 1 / 40, 40) - exact)
    assert 14.0 < e1 / e2 < 18.0


def test_euler_order():
    """Forward Euler is 1st order on the same closed form."""
    lam = 3.0
    rhs = lambda q: q * ((1 - lam) * q)
    exact = 1.0 / lam
    e1 = abs(dense.euler(rhs, 1.0, 1 / 200, 200) - exact)
    e2 = abs(dense.euler(rhs, 1.0, 1 / 400, 400) - exact)
    assert 1.8 < e1 / e2 < 2.2


# ---------------------------------------------------------------------------------------------
# Algorithm 1 bookkeeping
# ---------------------------------------------------------------------------------------------
def test_linear_parareal_binomial_closed_form():
    """For a linear flow X' = M X the propagators are matrices G = R_E(h_G M)^{m_G},
    F = R_RK4(h_F M)^{m_F} (commuting), and classical parareal has the closed form
        U^k_n = sum_{j=0}^{min(k,n)} C(n, j) (F - G)^j G^{n-j} u0
    (standard linear parareal analysis, Gander & Vandewalle; the algorithm of).
    Pins the correction's sign, indices and the Step-0 sweep."""
    rng = np.random.default_rng(11)
    n = 5
    M = -np.eye(n) + 0.4 * rng.standard_normal((n, n))    # non-symmetric
    X0 = np.eye(n) + 0.1 * rng.standard_normal((n, n))
    T, N, mG, mF = 2.0, 6, 2, 5
    hG, hF = T / (N * mG), T / (N * mF)
    ZG, ZF = hG * M, hF * M
    RE = np.eye(n) + ZG
    RK = np.eye(n) + ZF + ZF @ ZF / 2 + ZF @ ZF @ ZF / 6 + ZF @ ZF @ ZF @ ZF / 24
    Gm = np.linalg.matrix_power(RE, mG)
    Fm = np.linalg.matrix_power(RK, mF)
    out = dense.parareal(lambda X: M @ X, X0, T, N, mG, mF, N, keep_history=True)
    for k, U in enumerate(out["history"]):
        for m in range(N + 1):
            ref = sum(math.comb(m, j) * np.linalg.matrix_power(Fm - Gm, j) @
                      np.linalg.matrix_power(Gm, m - j) for j in range(min(k, m) + 1)) @ X0
            np.testing.assert_allclose(U[m], ref, rtol=0, atol=1e-12)


def _small_inverse_case(n=10, seed=1):
    w = workloads.random_spd(n, seed)
    return w.A


def test_parareal_K_equals_N_is_sequential_fine_bitwise():
    """P:155-157 (Remark): after N sweeps parareal equals the sequential fine solution; with the
    correction evaluated as F + (Gnew - Gold) (R3) the equality is bitwise (P5)."""
    A = _small_inverse_case()
    rhs = dense.make_rhs(A, dense.FLOW_INVERSE)
    X0 = np.eye(A.shape[0])
    N = 5
    out = dense.parareal(rhs, X0, 1.0, N, 1, 6, N)
    seq = dense.sequential_fine(rhs, X0, 1.0, N, 6)
    for m in range(N + 1):
        assert np.array_equal(out["U"][m], seq[m])


def test_prefix_exactness_bitwise():
    """S:194/S:220 (P6): after k sweeps U^k_n equals the sequential fine solution for n <= k."""
    A = _small_inverse_case(8, 2)
    rhs = dense.make_rhs(A, dense.FLOW_INVERSE)
    X0 = np.eye(8)
    N = 6
    out = dense.parareal(rhs, X0, 1.0, N, 1, 4, N, keep_history=True)
    seq = dense.sequential_fine(rhs, X0, 1.0, N, 4)
    for k, U in enumerate(out["history"]):
        for m in range(min(k, N) + 1):
            assert np.array_equal(U[m], seq[m]), (k, m)
        if k < N:   # and strictly not yet converged beyond the prefix (the test is not vacuous)
            assert not np.array_equal(U[N], seq[N])


def test_skip_prefix_is_bitwise_identical():
    """R14: skipping F(U^k_n), n < k, and the identity corrections changes nothing bitwise."""
    A = _small_inverse_case(9, 3)
    a = dense.solve(A, dense.FLOW_INVERSE, 1.0, 6, 1, 5, 4, skip_prefix=False)
    b = dense.solve(A, dense.FLOW_INVERSE, 1.0, 6, 1, 5, 4, skip_prefix=True)
    assert np.array_equal(a["X"], b["X"])
    assert a["deltas"] == b["deltas"]


def test_identity_matrix_is_exact():
    """S:129, S:273 (P7): A = I gives F == 0 for the inverse flow and F(I) = 0 for the sqrt flow,
    so the result is exactly I."""
    n = 7
    for flow in (dense.FLOW_INVERSE, dense.FLOW_SQRT):
        out = dense.solve(np.eye(n), flow, 1.0, 4, 1, 3, 3)
        assert np.array_equal(out["X"], np.eye(n))


def test_single_slice():
    """S:197 (P7): N = 1 gives U^1_1 = F(u0) exactly."""
    A = _small_inverse_case(6, 4)
    rhs = dense.make_rhs(A, dense.FLOW_INVERSE)
    out = dense.parareal(rhs, np.eye(6), 1.0, 1, 2, 7, 1)
    assert np.array_equal(out["X"], dense.rk4(rhs, np.eye(6), 1.0 / 7, 7))


def test_zero_flow_constant():
    """x' = 0 keeps every iterate equal to u0."""
    out = dense.parareal(lambda x: 0.0 * x, 2.5, 1.0, 5, 1, 3, 3, keep_history=True)
    for U in out["history"]:
        assert U == [2.5] * 6


# ---------------------------------------------------------------------------------------------
# Flows against the matrix functions they define
# ---------------------------------------------------------------------------------------------
def test_inverse_flow_closed_form_nonsymmetric():
    """P:169-176 (eq. eqQ): Q(t) = (I + t(A - I))^{-1} solves dQ/dt = -Q (A - I) Q = Q (I - A) Q,
    Q(1) = A^{-1}.  A non-symmetric, so X (B X) with a transposed operand would fail.  The RK4
    sequential fine solution matches the closed form at every slice end T_n within the RK4 error."""
    n = 12
    A = workloads.random_nonsymmetric(n, 0)
    N, mF = 4, 100
    S = dense.sequential_fine(dense.make_rhs(A, dense.FLOW_INVERSE), np.eye(n), 1.0, N, mF)
    for m in range(N + 1):
        t = m / N
        Q = np.linalg.inv(np.eye(n) + t * (A - np.eye(n)))
        assert np.abs(S[m] - Q).max() < 1e-9 * np.abs(Q).max()
    assert dense.residual_inverse(A, S[N]) < 1e-9


def test_cfg0_inverse_and_P3_bound():
    """P:44/P:176 (P3): A X(1) ~ I.  BASELINE cfg[0] stops at a fixed K = 4 < N, so the bound is
    the parareal error at K plus the RK4 error: 1e-7; at K = N it is <= 1e-12."""
    w = workloads.config(0)
    r4 = dense.solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, 4)
    assert dense.residual_inverse(w.A, r4["X"]) < 1e-7
    rN = dense.solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.N)
    assert dense.residual_inverse(w.A, rN["X"]) < 1e-12
    assert np.abs(rN["X"] - np.linalg.inv(w.A)).max() < 1e-12


def test_sqrt_steady_state():
    """P:46-51 (eq. stat) with F(X) = A - X^2: the steady state X* = A^{1/2} (F(X*) = 0).  Small 2D
    Laplacian analogue of cfg[4]: ||A - X^2||_F/||A||_F <= 1e-10, X symmetric, and X equals
    V diag(sqrt(lam)) V^T (closed-form Kronecker sine eigenbasis) within 1e-10 (P4)."""
    m = 4
    A = workloads.laplacian_2d(m) + np.eye(m * m)
    V1, mu1 = workloads.laplacian_1d_eig(m)
    V = np.kron(V1, V1)
    lam = 1.0 + (mu1[:, None] + mu1[None, :]).reshape(-1)
    out = dense.solve(A, dense.FLOW_SQRT, 20.0, 64, 2, 32, 4, tol=1e-10, stop=dense.STOP_RESIDUAL)
    X = out["X"]
    assert out["converged"] and out["residuals"][-1] <= 1e-10
    assert np.abs(X - X.T).max() < 1e-13
    np.testing.assert_allclose(X, (V * np.sqrt(lam)) @ V.T, rtol=0, atol=1e-10)


def test_dense_vs_spectral():
    """P1: with X0 = I every iterate is a polynomial in A, so the dense iteration equals
    V diag(u^k_n(lam)) V^T with u the scalar iteration per eigenvalue."""
    w = workloads.random_spd(20, 5)
    d = dense.solve(w.A, dense.FLOW_INVERSE, 1.0, 6, 1, 10, 6, tol=1e-12, stop=dense.STOP_DELTA)
    s = spectral.solve(w.eigvals, dense.FLOW_INVERSE, 1.0, 6, 1, 10, 6, tol=1e-12, stop=dense.STOP_DELTA)
    Xs = spectral.reconstruct(w.eigvecs, s["X"])
    assert d["k_done"] == s["k_done"]
    assert dense.frob(d["X"] - Xs) / dense.frob(Xs) < 1e-13
    for a, b in zip(d["deltas"][:-1], s["deltas"][:-1]):
        assert abs(a - b) <= 1e-6 * b + 1e-14


def test_spectral_vs_mpmath():
    """P2: the FP64 scalar iteration matches a 50-digit mpmath recursion of the same algorithm to
    <= 1e-13 relative, and both match the closed form 1/lam at K = N within the RK4 error."""
    lams = np.array([0.5, 0.9, 1.3, 2.0, 2.5])
    N, mG, mF = 4, 1, 16
    s = spectral.solve(lams, dense.FLOW_INVERSE, 1.0, N, mG, mF, 3)
    for i, lam in enumerate(lams):
        x_mp, _ = spectral.mp_parareal_scalar(lam, dense.FLOW_INVERSE, 1, N, mG, mF, 3)
        assert abs(s["X"][i] - float(x_mp)) <= 1e-13 * abs(float(x_mp))
    sN = spectral.solve(lams, dense.FLOW_INVERSE, 1.0, N, mG, mF, N)
    np.testing.assert_allclose(sN["X"], 1.0 / lams, rtol=1e-6)


def test_mpmath_golden():
    """Stored 50-digit values (tests/golden/scalar_parareal_mp50.txt, written by
    tools/make_golden.py which calls only oracle/) still match the FP64 scalar oracle."""
    g = _read_golden("scalar_parareal_mp50.txt")
    for key, val in g.items():
        flow, lam, N, mG, mF, K = key.split(":")
        s = spectral.solve(np.array([float(lam)]), int(flow), 1.0 if int(flow) == 0 else 4.0,
                           int(N), int(mG), int(mF), int(K))
        assert abs(s["X"][0] - float(val)) <= 1e-13 * abs(float(val)), key


def test_diagonal_closed_form_cfg_spectra():
    """P2 closed form q(1) = 1/lam: sequential fine RK4 with each config's (N, m_F) reaches
    1/lam within the RK4 error (<= 1e-12 relative) over each config's spectral interval."""
    for (N, mF, lo, hi) in [(8, 64, 0.5, 1.5), (16, 128, 1.0, 2.0), (64, 256, 0.1, 10.0), (64, 128, 1.0, 3.2)]:
        lam = np.linspace(lo, hi, 9)
        s = spectral.solve(lam, dense.FLOW_INVERSE, 1.0, N, 1, mF, N)
        np.testing.assert_allclose(s["X"], 1.0 / lam, rtol=1e-12)


def test_exp_flow_against_expm():
    """Example 2: dQ/dt = A Q, Q(0) = I => Q(1) = exp(A).  The sequential fine RK4
    solution matches scipy's expm (the library definition) within the RK4 error, for a
    non-symmetric A; and parareal at K = N equals it bitwise (P5)."""
    import scipy.linalg
    n = 10
    A = workloads.random_nonsymmetric(n, 3, scale=1.0) - np.eye(n)
    N, mF = 5, 40
    rhs = dense.make_rhs(A, dense.FLOW_EXP)
    S = dense.sequential_fine(rhs, np.eye(n), 1.0, N, mF)
    E = scipy.linalg.expm(A)
    assert np.abs(S[N] - E).max() <= 1e-9 * np.abs(E).max()
    out = dense.solve(A, dense.FLOW_EXP, 1.0, N, 1, mF, N)
    assert np.array_equal(out["X"], S[N])
    # exp(A) exp(-A) = I
    Sm = dense.sequential_fine(dense.make_rhs(-A, dense.FLOW_EXP), np.eye(n), 1.0, N, mF)
    assert np.abs(S[N] @ Sm[N] - np.eye(n)).max() < 1e-9


def test_trig_flow_against_sinm_cosm():
    """Example 3, eq. (eqB) with X0 = 0: U(1) = (sin A; cos A).  Sequential fine RK4
    matches scipy's sinm/cosm (library definitions) within the RK4 error for a non-symmetric A, and
    sin^2 + cos^2 = I; parareal at K = N equals the sequential fine run bitwise; the spectral oracle
    (s' = lam c, c' = -lam s per eigenvalue) agrees with the dense one for a symmetric A."""
    import scipy.linalg
    n = 9
    A = workloads.random_nonsymmetric(n, 4, scale=1.0)
    N, mF = 5, 40
    S = dense.sequential_fine(dense.make_rhs(A, dense.FLOW_TRIG), dense.initial_state(n, dense.FLOW_TRIG),
                              1.0, N, mF)[N]
    assert S.shape == (2 * n, n)
    assert np.abs(S[:n] - scipy.linalg.sinm(A)).max() < 1e-9
    assert np.abs(S[n:] - scipy.linalg.cosm(A)).max() < 1e-9
    assert np.abs(S[:n] @ S[:n] + S[n:] @ S[n:] - np.eye(n)).max() < 1e-9
    out = dense.solve(A, dense.FLOW_TRIG, 1.0, N, 1, mF, N)
    assert np.array_equal(out["X"], S)
    w = workloads.random_spd(12, 8)
    d = dense.solve(w.A, dense.FLOW_TRIG, 1.0, 6, 2, 10, 3)
    s = spectral.solve(w.eigvals, dense.FLOW_TRIG, 1.0, 6, 2, 10, 3)
    ref = spectral.reconstruct(w.eigvecs, s["X"])
    assert dense.frob(d["X"] - ref) / dense.frob(ref) < 1e-13


def test_cosine_algorithm5():
    """Algorithm 5: m = min{m : 2^-m ||A||_inf <= 1} (golden: ||A||_inf = 5 -> m = 3,
    written out from the definition), A0 = 2^-m A, C0 = cos(A0) by parareal, C_{i+1} = 2C_i^2 - I.
    Against scipy's cosm within the RK4 error amplified by the m doublings."""
    import scipy.linalg
    C, m, out = dense.cosine_algorithm5(np.diag([5.0, -2.0, 1.0]), 4, 1, 20, 4)
    assert m == 3
    np.testing.assert_allclose(np.diag(C), np.cos([5.0, -2.0, 1.0]), rtol=0, atol=1e-9)
    n = 10
    A = 0.8 * workloads.random_nonsymmetric(n, 6, scale=2.0)
    C, m, out = dense.cosine_algorithm5(A, 6, 2, 30, 6)
    assert m >= 1
    assert np.abs(C - scipy.linalg.cosm(A)).max() < 1e-8


def test_accel_inverse_closed_forms():
    """Algorithm 8.  With E_k = A^{-1} - X_k and R = I - dt A the recursion gives
    E_k = R^{k-1} (R - k dt I) E_0 when u_0 = E_0 exactly (the paper's Fig. ACC_MAT_GRAD2 case),
    and E_k = R^k E_0 with no accelerator (u_0 = 0: forward Euler on dX/dt = I - AX)."""
    w = workloads.random_spd(8, 9)
    A = w.A / np.linalg.norm(w.A)          # rescaled by its Frobenius norm as in P:702
    Ainv = np.linalg.inv(A)
    n, dt, K = 8, 0.1, 25
    R = np.eye(n) - dt * A
    E0 = Ainv.copy()                        # X0 = 0
    Xs = accel = dense.accel_inverse(A, E0, dt, K)
    for k in (1, 5, 10, 25):
        Ek = np.linalg.matrix_power(R, k - 1) @ (R - k * dt * np.eye(n)) @ E0
        np.testing.assert_allclose(Ainv - Xs[k], Ek, rtol=0, atol=1e-11 * np.abs(Ainv).max())
    Xn = dense.accel_inverse(A, None, dt, K)
    for k in (1, 7, 25):
        np.testing.assert_allclose(Ainv - Xn[k], np.linalg.matrix_power(R, k) @ E0, rtol=0,
                                   atol=1e-11 * np.abs(Ainv).max())
    # the accelerator helps: at t = k dt = 1 (xi(t) = min(t-1, 0) e) the exact-e error is
    # -dt A R^9 E_0, far below the plain flow's R^10 E_0
    k1 = int(round(1 / dt))
    assert np.linalg.norm(Ainv - accel[k1]) < 0.2 * np.linalg.norm(Ainv - Xn[k1])


def test_global_qr_examples_and_orthonormality():
    """Algorithm 2: SPEC S:63-66 worked examples (diag(3,4) -> r_11 = 5; a dependent
    block 2 Z1 is eliminated), and on random blocks Q^T <> Q = I and Z_i in span(Q) (Proposition)."""
    Z1 = np.diag([3.0, 4.0])
    Q = []
    assert dense.global_qr([Z1], Q) == [0]
    np.testing.assert_allclose(Q[0], Z1 / 5.0, rtol=0, atol=1e-16)
    Q = []
    assert dense.global_qr([Z1, 2.0 * Z1], Q) == [0]
    rng = np.random.default_rng(3)
    Z = [rng.standard_normal((6, 2)) for _ in range(4)]
    Q = []
    dense.global_qr(Z, Q)
    G = np.array([[dense.frob_inner(a, b) for b in Q] for a in Q])
    np.testing.assert_allclose(G, np.eye(len(Q)), rtol=0, atol=1e-12)
    for Zi in Z:
        P = sum(dense.frob_inner(Zi, q) * q for q in Q)
        assert dense.frob(Zi - P) < 1e-12 * dense.frob(Zi)


def test_modified_parareal_saturated_basis_is_fine():
    """Algorithm 3: every iterate is a polynomial in A (X0 = I), so once S^k contains
    span{I, A, ..., A^{n-1}} the projection is the identity on the iterates and eq. (eq_update)
    reproduces the sequential fine propagation.  n = 3, N = 4: the Step-0 iterates I, G(I), ...
    already span it, so sweep 1 equals the sequential fine solution up to rounding."""
    n = 3
    A = workloads.random_nonsymmetric(n, 8, scale=1.0)
    out = dense.solve_modified(A, dense.FLOW_EXP, 1.0, 4, 1, 10, 1)
    seq = dense.solve_sequential_fine(A, dense.FLOW_EXP, 1.0, 4, 10)
    assert out["basis"] == n
    assert dense.frob(out["X"] - seq) <= 1e-12 * dense.frob(seq)


def test_modified_converges_faster_than_classical():
    """P:489-490 (Fig. "cos": "the modified parareal algorithm converges much faster"): on the trig
    block flow, the error against the sequential fine solution after k sweeps is never larger for
    Algorithm 3 than for Algorithm 1 (SPEC S:223 monotone dominance), and strictly smaller at k = 2."""
    n = 8
    w = workloads.random_spd(n, 12, lo=0.5, hi=3.0)
    N, mG, mF = 10, 1, 10
    seq = dense.solve_sequential_fine(w.A, dense.FLOW_TRIG, 1.0, N, mF)
    errs = []
    for k in (1, 2, 3):
        c = dense.solve(w.A, dense.FLOW_TRIG, 1.0, N, mG, mF, k)
        m = dense.solve_modified(w.A, dense.FLOW_TRIG, 1.0, N, mG, mF, k)
        errs.append((dense.frob(c["X"] - seq), dense.frob(m["X"] - seq)))
        assert errs[-1][1] <= errs[-1][0] * (1 + 1e-9) + 1e-14
    assert errs[1][1] < 0.5 * errs[1][0]
    # the trig states (p(A), q(A)) span at most 2n dimensions: once S^k holds them the update is the
    # fine propagation itself (rounding level), while classical parareal is still at ~1e-3
    assert errs[2][1] < 1e-11 * dense.frob(seq) and errs[2][0] > 1e-5 * dense.frob(seq)
    # R17: with a single Gram-Schmidt pass the same run loses orthogonality and diverges
    rhs = dense.make_rhs(w.A, dense.FLOW_TRIG)
    import oracle.dense as od
    orig = od.global_qr
    try:
        od.global_qr = lambda Z, Q, rank_tol=1e-12: orig(Z, Q, rank_tol, passes=1)
        one = od.modified_parareal(rhs, dense.initial_state(n, dense.FLOW_TRIG), 1.0, N, mG, mF, 3)
    finally:
        od.global_qr = orig
    assert dense.frob(one["X"] - seq) > 1e3 * errs[2][1]


def test_config_workloads_shapes():
    """workloads builds what BASELINE.json names (sizes, symmetry, spectra)."""
    for i in (0, 1, 2):
        w = workloads.config(i)
        assert w.A.shape == (w.n, w.n) and w.A.flags.c_contiguous
        assert np.array_equal(w.A, w.A.T)
        lam = np.linalg.eigvalsh(w.A)
        assert np.allclose(np.sort(lam), np.sort(w.eigvals), rtol=1e-12, atol=1e-12)
    assert workloads.config(1).n == 256 and workloads.config(2).n == 1024


# ---------------------------------------------------------------------------------------------
# Affine (linear inhomogeneous) flow and Algorithm 4 (§3 "The linear inhomogeneous case")
# ---------------------------------------------------------------------------------------------
def _affine_closed_form(A, Gsrc, U0, t):
    """u(t) = u0 + t phi(tA)(A u0 + g) (eq. eq1) for a MATRIX state, evaluated with the
    library's expm of the augmented generator M = [[A, A U0 + G], [0, 0]]:
    expm(tM) = [[e^{tA}, t phi(tA)(A U0 + G)], [0, I]]."""
    import scipy.linalg
    n = A.shape[0]
    M = np.zeros((2 * n, 2 * n))
    M[:n, :n] = A
    M[:n, n:] = A @ U0 + Gsrc
    return U0 + scipy.linalg.expm(t * M)[:n, n:]


def test_affine_flow_closed_form_nonsymmetric():
    """eq. (eq1) P:72-82 with a matrix state: the fine propagation of dU/dt = A U + G (A, G, U0
    non-symmetric and non-commuting, so a transposed or dropped term fails) reaches the closed form
    u0 + t phi(tA)(A u0 + g) within the RK4 truncation error; Euler within its first-order error."""
    n = 7
    A = workloads.random_nonsymmetric(n, 21, scale=1.0) - 1.5 * np.eye(n)
    rng = np.random.default_rng(21)
    Gs = rng.standard_normal((n, n))
    U0 = rng.standard_normal((n, n))
    ref = _affine_closed_form(A, Gs, U0, 1.0)
    rhs = dense.make_rhs(A, dense.FLOW_AFFINE, Gs)
    X = dense.rk4(rhs, U0, 1.0 / 64, 64)
    assert dense.frob(X - ref) <= 1e-8 * dense.frob(ref)
    Xe = dense.euler(rhs, U0, 1.0 / 4096, 4096)
    err = dense.frob(Xe - ref) / dense.frob(ref)
    assert 1e-6 < err < 1e-3
    # Example 5 is the instance (A, G) -> (-A, I), U0 = 0: X(t) -> A^{-1}
    w = workloads.random_spd(n, 22, lo=1.0, hi=2.0)
    Xs = dense.solve_sequential_fine(-w.A, dense.FLOW_AFFINE, 24.0, 8, 64, source=np.eye(n), X0=np.zeros((n, n)))
    assert dense.frob(Xs - np.linalg.inv(w.A)) <= 1e-9 * dense.frob(np.linalg.inv(w.A))


def test_affine_identity_of_the_fine_map():
    """for a linear fine propagator F(a X + b Y) = a (F(X) - F(0)) + b (F(Y) - F(0)) + F(0);
    the oracle's RK4 map on the affine flow satisfies it to rounding (an affine-ness bug, e.g. a
    source term applied twice per stage, breaks it at O(h))."""
    n = 6
    A = workloads.random_nonsymmetric(n, 23, scale=1.0)
    rng = np.random.default_rng(23)
    Gs, X, Y = (rng.standard_normal((n, n)) for _ in range(3))
    rhs = dense.make_rhs(A, dense.FLOW_AFFINE, Gs)
    F = lambda Z: dense.rk4(rhs, Z, 1.0 / 40, 10)
    a, b = 0.7, -1.9
    lhs = F(a * X + b * Y)
    F0 = F(np.zeros((n, n)))
    rhs_ = a * (F(X) - F0) + b * (F(Y) - F0) + F0
    assert dense.frob(lhs - rhs_) <= 1e-13 * dense.frob(lhs)
    # the coarse map is affine too, and G(0) = m_G steps of Euler from 0 = h G + ... (one step: h G)
    G1 = dense.euler(rhs, np.zeros((n, n)), 0.125, 1)
    assert np.array_equal(G1, 0.125 * Gs)


def test_algorithm4_zero_source_is_algorithm3_bitwise():
    """With G = 0, Step -1 gives F(0) = G(0) = 0 exactly and eq. (update2) reduces to eq. (eq_update)
    term by term: Algorithm 4 on the affine flow == Algorithm 3 on the exp flow, bitwise."""
    n = 5
    w = workloads.random_spd(n, 24, lo=0.5, hi=3.0)
    N, mG, mF, K = 6, 1, 8, 3
    m3 = dense.solve_modified(w.A, dense.FLOW_EXP, 1.0, N, mG, mF, K)
    m4 = dense.solve_modified(w.A, dense.FLOW_AFFINE, 1.0, N, mG, mF, K, source=np.zeros((n, n)))
    assert not np.any(m4["F0"]) and not np.any(m4["G0"])
    assert m3["basis"] == m4["basis"] and m3["k_done"] == m4["k_done"]
    for U3, U4 in zip(m3["U"], m4["U"]):
        assert np.array_equal(U3, U4)


def test_algorithm4_saturated_basis_is_fine_and_beats_classical():
    """Algorithm 4: once S^k spans every iterate, P_k = I on them and eq. (update2) is
    F(U) + G(0) - G(0) = F(U) -- the sequential fine solution (a dropped -G(0), or F(P U) without
    the affine correction of the Remark P:424-428, breaks this).  n = 2: every iterate of every
    propagator is r(A) W - C with W = U0 + A^{-1} G, C = A^{-1} G (Euler and RK4 share the fixed
    point -A^{-1} G), so all of them lie in span{W, A W, C} (dimension 3), which the Step-0 iterates
    already span: sweep 1 is the fine solution up to rounding -- far ahead of classical parareal;
    the closed form eq1 confirms the fine solution itself."""
    n = 2
    A = workloads.random_nonsymmetric(n, 25, scale=1.0) - np.eye(n)
    rng = np.random.default_rng(25)
    Gs = rng.standard_normal((n, n))
    U0 = rng.standard_normal((n, n))
    N, mG, mF = 4, 1, 16
    seq = dense.solve_sequential_fine(A, dense.FLOW_AFFINE, 1.0, N, mF, source=Gs, X0=U0)
    m = dense.solve_modified(A, dense.FLOW_AFFINE, 1.0, N, mG, mF, 1, source=Gs, X0=U0)
    assert m["basis"] == 3
    assert dense.frob(m["X"] - seq) <= 1e-12 * dense.frob(seq)
    c = dense.solve(A, dense.FLOW_AFFINE, 1.0, N, mG, mF, 1, source=Gs, X0=U0)
    assert dense.frob(c["X"] - seq) > 1e3 * dense.frob(m["X"] - seq)
    assert dense.frob(seq - _affine_closed_form(A, Gs, U0, 1.0)) <= 1e-7 * dense.frob(seq)
    # larger n, commuting data: monotone dominance over classical parareal
    n = 10
    w = workloads.random_spd(n, 26, lo=0.5, hi=2.0)
    N, mG, mF = 8, 1, 8
    src = np.eye(n)
    seq = dense.solve_sequential_fine(-w.A, dense.FLOW_AFFINE, 4.0, N, mF, source=src, X0=np.zeros((n, n)))
    for k in (1, 2, 3):
        c = dense.solve(-w.A, dense.FLOW_AFFINE, 4.0, N, mG, mF, k, source=src, X0=np.zeros((n, n)))
        m = dense.solve_modified(-w.A, dense.FLOW_AFFINE, 4.0, N, mG, mF, k, source=src, X0=np.zeros((n, n)))
        assert dense.frob(m["X"] - seq) <= dense.frob(c["X"] - seq) * (1 + 1e-9) + 1e-14


def test_affine_dense_vs_spectral():
    """The spectral oracle's affine recursion x' = lam x + gamma (P1 with a commuting source) against
    the dense oracle: Example 5's flow dX/dt = I - A X, X0 = 0, classical parareal."""
    w = workloads.random_spd(12, 27, lo=0.5, hi=2.0)
    N, mG, mF, K = 8, 2, 16, 4
    d = dense.solve(-w.A, dense.FLOW_AFFINE, 3.0, N, mG, mF, K, source=np.eye(12), X0=np.zeros((12, 12)))
    s = spectral.solve(-w.eigvals, dense.FLOW_AFFINE, 3.0, N, mG, mF, K, gamma=1.0, x0=0.0)
    X = spectral.reconstruct(w.eigvecs, s["X"])
    assert dense.frob(d["X"] - X) <= 1e-13 * dense.frob(X)
    np.testing.assert_allclose(d["deltas"], s["deltas"], rtol=1e-9)


def test_residual_definitions_closed_form():
    """a8 residuals on hand-computed non-symmetric 2 x 2 cases where
    ||A X - I|| != ||X A - I||: A = [[2, 1], [0, 1]], X = [[0, 0], [1, 0]] gives A X - I =
    [[0, 0], [1, -1]] (Frobenius sqrt 2, so ||A X - I||_F / sqrt(n) = 1) while X A - I =
    [[-1, 0], [2, 0]] (sqrt 5); a swapped product or a /n normalisation fails.  Square root:
    A = [[4, 1], [0, 9]], X = [[2, 0.2], [0, 3]] has X^2 = A exactly (residual 0) while the
    transposed square X X^T does not; X = 2 I gives A - X^2 = [[0, 1], [0, 5]], ||.||_F = sqrt 26,
    ||A||_F = sqrt 98."""
    A = np.array([[2.0, 1.0], [0.0, 1.0]])
    X = np.array([[0.0, 0.0], [1.0, 0.0]])
    assert dense.residual_inverse(A, X) == pytest.approx(1.0, rel=1e-15)
    assert dense.residual_inverse(A, X) != pytest.approx(math.sqrt(5.0) / math.sqrt(2.0), rel=1e-3)
    A = np.array([[4.0, 1.0], [0.0, 9.0]])
    assert dense.residual_sqrt(A, np.array([[2.0, 0.2], [0.0, 3.0]])) == 0.0
    assert dense.residual_sqrt(A, 2.0 * np.eye(2)) == pytest.approx(math.sqrt(26.0 / 98.0), rel=1e-15)


def test_max_slice_stop_rule_against_binomial_closed_form():
    """SPEC's stop rule (STOP_MAX_SLICE): stop at the first k with
    max_n ||U^k_n - U^{k-1}_n||_F <= tol max(1, ||U_0||_F).  The expected k comes from the binomial
    closed form of linear parareal (standard analysis, as test_linear_parareal_binomial_closed_form),
    not from the oracle's own iterates; the metric values too."""
    rng = np.random.default_rng(12)
    n = 4
    M = -np.eye(n) + 0.3 * rng.standard_normal((n, n))
    X0 = 2.0 * np.eye(n) + 0.1 * rng.standard_normal((n, n))
    T, N, mG, mF = 2.0, 8, 1, 6
    hG, hF = T / (N * mG), T / (N * mF)
    ZG, ZF = hG * M, hF * M
    Gm = np.linalg.matrix_power(np.eye(n) + ZG, mG)
    Fm = np.linalg.matrix_power(np.eye(n) + ZF + ZF @ ZF / 2 + ZF @ ZF @ ZF / 6 + ZF @ ZF @ ZF @ ZF / 24, mF)
    U = lambda k, m: sum(math.comb(m, j) * np.linalg.matrix_power(Fm - Gm, j) @ np.linalg.matrix_power(Gm, m - j)
                         for j in range(min(k, m) + 1)) @ X0
    scale = max(1.0, np.linalg.norm(X0))
    metric = [max(np.linalg.norm(U(k, m) - U(k - 1, m)) for m in range(N + 1)) / scale for k in range(1, N + 1)]
    tol = math.sqrt(metric[2] * metric[3])          # strictly between sweeps 3 and 4
    expect_k = next(k for k, v in enumerate(metric, start=1) if v <= tol)
    assert expect_k == 4
    out = dense.parareal(lambda X: M @ X, X0, T, N, mG, mF, N, tol, dense.STOP_MAX_SLICE)
    assert out["k_done"] == expect_k and out["converged"]
    np.testing.assert_allclose(out["deltas"], metric[:expect_k], rtol=1e-9)
