"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances:
  * whole solves: relative Frobenius error <= 1e-10 (BASELINE.json north star), in practice ~1e-14;
  * GEMM: ||C_gpu - C_ref||_F <= 2 n u || |A| |B| ||_F, u = 2^-53 (gamma_n bound applied to both
    sides);
  * element-wise stage updates: a few ulp (FMA contraction is the only difference);
  * bookkeeping (prefix exactness, K = N, logical-rank invariance, A = I): bitwise.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1505_07959_b200 as mf  # noqa: E402
import workloads  # noqa: E402
from oracle import dense, spectral  # noqa: E402

pytestmark = pytest.mark.gpu
U53 = 2.0 ** -53


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    mf.lib()
    yield


def _dev(a, ld=None):
    """Host array -> device tensor with leading dimension ld (padding zero), returns the n x n view."""
    n = a.shape[0]
    ld = ld or n
    t = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    t[:, :n] = torch.from_numpy(np.ascontiguousarray(a))
    return t[:, :n]


def relF(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


# ---------------------------------------------------------------------------------------------
# kernel level
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("n", [1, 8, 30, 64, 100, 129, 256, 500])
def test_dgemm_parity(n, tile):
    rng = np.random.default_rng(n * 10 + tile)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    ld = n + (n % 2) + (16 if n % 3 == 0 else 0)   # ragged leading dimensions too
    dA, dB = _dev(A, ld), _dev(B, ld)
    dD = _dev(np.zeros((n, n)), ld)
    mf.dgemm(dA, dB, out=dD, tile=tile)
    D = dD.cpu().numpy()
    ref = A @ B
    bound = 2 * n * U53 * np.linalg.norm(np.abs(A) @ np.abs(B))
    assert np.linalg.norm(D - ref) <= bound


@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("n", [300, 1100])
def test_dgemm_grouped_raster_ragged_bands(n, tile):
    """The persistent tile schedule walks bands of 8 tile rows (gemm.cuh tile_coords); these sizes
    leave a last band of fewer rows for every tile config (and ragged tiles inside it).  Every
    element must be produced exactly once: the output starts as NaN, so a tile never visited fails."""
    rng = np.random.default_rng(n + tile)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    dA, dB = _dev(A), _dev(B)
    dD = _dev(np.full((n, n), np.nan))
    mf.dgemm(dA, dB, out=dD, tile=tile)
    D = dD.cpu().numpy()
    assert np.isfinite(D).all()
    ref = A @ B
    assert np.all(np.abs(D - ref) <= 2 * n * U53 * (np.abs(A) @ np.abs(B)))


@pytest.mark.parametrize("n", [64, 200])
def test_dgemm_alpha_beta(n):
    rng = np.random.default_rng(5)
    A, B, C = (rng.standard_normal((n, n)) for _ in range(3))
    dD = mf.dgemm(_dev(A), _dev(B), C=_dev(C), alpha=-1.0, beta=1.0)
    ref = C - A @ B
    bound = 2 * (n + 1) * U53 * np.linalg.norm(np.abs(A) @ np.abs(B) + np.abs(C))
    assert np.linalg.norm(dD.cpu().numpy() - ref) <= bound


def test_dgemm_large_sampled():
    """n = 4096 (BASELINE cfg[3]/[4] size, the bench's tile config): sampled rows vs numpy."""
    n = 4096
    g = torch.Generator(device="cuda").manual_seed(0)
    dA = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    dB = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    dD = mf.dgemm(dA, dB)
    rows = [0, 1, 127, 128, 2047, 4000, 4095]
    A = dA[rows].cpu().numpy()
    B = dB.cpu().numpy()
    ref = A @ B
    got = dD[rows].cpu().numpy()
    bound = 2 * n * U53 * np.linalg.norm(np.abs(A) @ np.abs(B))
    assert np.linalg.norm(got - ref) <= bound


@pytest.mark.parametrize("stage", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [40, 256])
def test_rk_stage_parity(n, stage):
    rng = np.random.default_rng(stage)
    Y, W, X, S = (rng.standard_normal((n, n)) for _ in range(4))
    h = 1.0 / 64
    dX, dS, dYn = _dev(X), _dev(S), _dev(np.zeros((n, n)))
    mf.rk_stage(_dev(Y), _dev(W), dX, dS, dYn, stage, h)
    K = Y @ W
    tolK = 2 * n * U53 * np.abs(Y) @ np.abs(W)
    if stage == 4:
        refX = X + (h / 6) * (S + K)
        err = np.abs(dX.cpu().numpy() - refX)
        assert np.all(err <= (h / 6) * tolK + 4 * U53 * (np.abs(X) + (h / 6) * np.abs(S + K)))
    else:
        refS = K if stage == 1 else S + 2 * K
        c = h if stage == 3 else h / 2
        refY = X + c * K
        assert np.all(np.abs(dS.cpu().numpy() - refS) <= 2 * tolK + 4 * U53 * np.abs(refS))
        assert np.all(np.abs(dYn.cpu().numpy() - refY) <= c * tolK + 4 * U53 * (np.abs(X) + c * np.abs(K)))


@pytest.mark.parametrize("stage", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [300, 1030])
def test_rk_stage_staged_epilogue_bitwise(n, stage):
    """The 128 x 128 kernel stages the epilogue operands (C, X, S) through shared memory with
    cp.async; the per-element arithmetic and k order are those of the 64 x 64 kernel, so both tile
    configurations agree bitwise -- here at ragged n (partial tiles, partial 4-column groups) with the
    beta C term of the sqrt flow."""
    rng = np.random.default_rng(10 + stage)
    Y, W, X, S, C = (rng.standard_normal((n, n)) for _ in range(5))
    out = []
    for tile in (1, 2):
        dX, dS, dYn = _dev(X), _dev(S), _dev(np.zeros((n, n)))
        mf.rk_stage(_dev(Y), _dev(W), dX, dS, dYn, stage, 1.0 / 64, C=_dev(C), alpha=-1.0, beta=1.0, tile=tile)
        out.append((dX.cpu().numpy(), dS.cpu().numpy(), dYn.cpu().numpy()))
    for a, b in zip(*out):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("flow,n", [(0, 300), (1, 300), (2, 300), (0, 515)])
def test_staged_epilogue_solves_bitwise(flow, n):
    """Whole solves through every staged epilogue (RK stages, Step 0 Euler, the correction with its
    inline Gold) with 128 x 128 tiles agree bitwise with 64 x 64 tiles (no staging) at ragged n."""
    A = workloads.random_spd(n, 40 + n).A
    if flow == 1:
        A = A + np.eye(n)
    elif flow == 2:
        A = A - 1.5 * np.eye(n)
    res = [_solve_gpu(A, flow, 1.0, 4, 1, 3, 2, tile=t)[1:] for t in (1, 2)]
    assert np.array_equal(res[0][1], res[1][1])
    assert res[0][0]["deltas"] == res[1][0]["deltas"]


@pytest.mark.parametrize("n,N,K", [(3072, 2, 1), (4096, 3, 2)])
def test_staged_correction_large_n_bitwise(n, N, K):
    """Regression guard for the staged epilogue at the sizes where its persistent CTAs run many tiles
    (profiles/staged_epilogue_r02.md): whole sqrt-flow solves with 128 x 128 tiles (staged C / X / F,
    inline Gold) equal the unstaged 64 x 64 kernel bitwise, twice over.  The dropped early-issue
    variant (tools/experiments/gold_early_issue_r02.patch) fails exactly this comparison."""
    A = workloads.random_spd(n, 7).A + np.eye(n)
    ref = _solve_gpu(A, 1, 1.0, N, 1, 4, K, tile=1)[2]
    for _ in range(2):
        X = _solve_gpu(A, 1, 1.0, N, 1, 4, K, tile=2)[2]
        assert np.array_equal(X, ref)


def test_frobenius_parity():
    rng = np.random.default_rng(9)
    X, Y = rng.standard_normal((300, 300)), rng.standard_normal((300, 300))
    d, x = mf.frobenius(_dev(X), _dev(Y))
    assert abs(d - np.linalg.norm(X - Y)) <= 1e-13 * d
    assert abs(x - np.linalg.norm(X)) <= 1e-13 * x


# ---------------------------------------------------------------------------------------------
# solver level
# ---------------------------------------------------------------------------------------------
def _solve_gpu(A, flow, T, N, mG, mF, K, tol=0.0, stop=0, world=1, **opts):
    s = mf.Solver(A, flow, T, N, mG, mF, world=world)
    for k, v in opts.items():
        s.set_option(k, v)
    info = s.solve(K, tol, stop)
    X = s.result()
    return s, info, X


@pytest.mark.parametrize("n", [3, 40, 100])
def test_solver_small_vs_oracle(n):
    w = workloads.random_spd(n, n)
    N, mG, mF, K = 6, 1, 8, 3
    s, info, X = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, N, mG, mF, K)
    ref = dense.solve(w.A, dense.FLOW_INVERSE, 1.0, N, mG, mF, K)
    assert info["k_done"] == K
    assert relF(X, ref["X"]) <= 1e-12
    for k in range(K):
        assert abs(info["deltas"][k] - ref["deltas"][k]) <= 1e-6 * ref["deltas"][k] + 1e-15
    s.close()


def test_solver_sqrt_small_vs_oracle():
    m = 5
    A = workloads.laplacian_2d(m) + np.eye(m * m)
    N, mG, mF = 64, 2, 32
    s, info, X = _solve_gpu(A, mf.FLOW_SQRT, 20.0, N, mG, mF, 4, 1e-10, mf.STOP_RESIDUAL)
    ref = dense.solve(A, dense.FLOW_SQRT, 20.0, N, mG, mF, 4, 1e-10, dense.STOP_RESIDUAL)
    assert info["k_done"] == ref["k_done"] == 1
    assert relF(X, ref["X"]) <= 1e-12
    assert abs(info["residual0"] - ref["residual0"]) <= 1e-6 * ref["residual0"] + 1e-16
    assert s.residual() <= 1e-10


def test_coarse_only_K0():
    w = workloads.random_spd(24, 1)
    s, info, X = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, 5, 2, 4, 0)
    ref = dense.solve(w.A, dense.FLOW_INVERSE, 1.0, 5, 2, 4, 0)
    assert info["k_done"] == 0
    assert relF(X, ref["X"]) <= 1e-13


def test_prefix_exactness_and_K_equals_N_bitwise():
    """P5/P6: GPU U^k_n == GPU sequential fine for n <= k, bitwise; K = N exact."""
    w = workloads.random_spd(48, 2)
    N = 5
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 6)
    s.sequential_fine()
    seq = [s.slice(m) for m in range(N + 1)]
    for k in range(N + 1):
        info = s.solve(k)
        assert info["k_done"] == k
        for m in range(k + 1):
            assert np.array_equal(s.slice(m), seq[m]), (k, m)
    assert np.array_equal(s.result(), seq[N])
    # and the sequential fine GPU result matches the oracle's sequential fine run
    ref = dense.solve_sequential_fine(w.A, dense.FLOW_INVERSE, 1.0, N, 6)
    assert relF(seq[N], ref) <= 1e-13


@pytest.mark.parametrize("world", [2, 3, 4])
def test_logical_ranks_bitwise(world):
    """P9: the slice partition over ranks (contiguous blocks, boundary exchange) changes nothing."""
    w = workloads.random_spd(64, 3)
    N = 8
    _, i1, X1 = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 8, 16, 1e-12, mf.STOP_DELTA)
    _, iP, XP = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 8, 16, 1e-12, mf.STOP_DELTA, world=world)
    assert i1["k_done"] == iP["k_done"]
    assert np.array_equal(X1, XP)
    assert i1["deltas"] == iP["deltas"]


@pytest.mark.parametrize("overlap", [0, 1])
def test_overlap_and_batch_invariance(overlap):
    """Speculative overlap and the fine batch size do not change results (bitwise)."""
    w = workloads.random_spd(80, 4)
    _, ia, Xa = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, 7, 1, 6, 7, 1e-11, mf.STOP_DELTA, overlap=overlap)
    _, ib, Xb = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, 7, 1, 6, 7, 1e-11, mf.STOP_DELTA, overlap=1 - overlap,
                           fine_batch=2, tile=3)
    assert ia["k_done"] == ib["k_done"]
    assert np.array_equal(Xa, Xb)


@pytest.mark.parametrize("cs", [1, 2, 4])
def test_small_speculative_cancel_repeatable(cs):
    """K6/K6c under speculation: the next sweep's fine launch is queued before the stop test and is
    cancelled through the device stop flag when δ reaches tol; a cluster follows its rank-0 CTA's
    reading of the flag, so a flag raised while the clusters start cannot split one (a split
    cluster would hang on its exchange barrier).  Repeated solves must end, agree bitwise with the
    strictly phased run, and stop at the same k."""
    w = workloads.random_spd(32, 21)
    _, i0, X0 = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, 8, 1, 16, 8, 1e-9, mf.STOP_DELTA, overlap=0,
                           small_cluster=cs)
    assert 1 <= i0["k_done"] < 8
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, 8, 1, 16)
    s.set_option("overlap", 1)
    s.set_option("small_cluster", cs)
    for _ in range(20):
        info = s.solve(8, 1e-9, mf.STOP_DELTA)
        assert info["k_done"] == i0["k_done"]
        assert np.array_equal(s.result(), X0)
    s.close()


def test_identity_exact():
    """P7: A = I gives exactly I for both flows."""
    for flow in (mf.FLOW_INVERSE, mf.FLOW_SQRT):
        _, info, X = _solve_gpu(np.eye(33), flow, 1.0, 4, 1, 3, 3)
        assert np.array_equal(X, np.eye(33))


def test_single_slice():
    """N = 1 => U^1_1 = F(X0) = the sequential fine solution."""
    w = workloads.random_spd(20, 6)
    s, info, X = _solve_gpu(w.A, mf.FLOW_INVERSE, 1.0, 1, 2, 9, 1)
    ref = dense.solve_sequential_fine(w.A, dense.FLOW_INVERSE, 1.0, 1, 9)
    assert relF(X, ref) <= 1e-13


def test_nonsymmetric_inverse():
    """Non-symmetric A: catches a transposed operand anywhere on the GPU path."""
    n = 50
    A = workloads.random_nonsymmetric(n, 1)
    s, info, X = _solve_gpu(A, mf.FLOW_INVERSE, 1.0, 4, 1, 50, 4)
    ref = dense.solve(A, dense.FLOW_INVERSE, 1.0, 4, 1, 50, 4)
    assert relF(X, ref["X"]) <= 1e-12
    assert np.abs(X - np.linalg.inv(A)).max() <= 1e-8 * np.abs(np.linalg.inv(A)).max()


def test_nonfinite_reports_bad_slice():
    """a flow that blows up is reported as ENONFINITE naming the FIRST bad slice.  The expected
    slice comes from the oracle run on the same input (diagonal A: the scalar recursion
    q' = (1 - 40) q^2, whose Step-0 iterates stay finite but whose first fine sweep overflows)."""
    A = np.diag(np.full(16, 40.0))
    N, mG, mF = 4, 1, 4
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, N, mG, mF)
    with pytest.raises(mf.MfodeError) as e:
        s.solve(2, 1e-10, mf.STOP_DELTA)
    assert e.value.status == mf.ENONFINITE
    with np.errstate(all="ignore"):
        ref = spectral.solve(np.full(16, 40.0), dense.FLOW_INVERSE, 1.0, N, mG, mF, 2, keep_history=True)
    k_bad = next(k for k, d in enumerate(ref["deltas"], start=1) if not np.isfinite(d))
    expect = next(m for m, u in enumerate(ref["history"][k_bad]) if not np.all(np.isfinite(u)))
    info = e.value.info
    assert info is not None and info["k_done"] == k_bad
    assert info["bad_slice"] == expect and expect >= 1


def _fma(a, b, c):
    """Correctly rounded a*b + c (exact rational arithmetic, one rounding): the GPU's FMA."""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _gpu_order_scalar_parareal_inverse(lam, T, N, mG, mF, K):
    """The GPU kernels' arithmetic on one diagonal entry of the inverse flow, operation by operation
    (gemm.cuh / small.cuh / epilogue.cuh): B = 1 - lam (k_i_minus); each rhs K = fl(y fl(b y)) (the
    DMMA sums contain one non-zero product and exact zeros); RK stages Y = fma(c, K, X),
    S = K | fma(2, K, S), X = fma(h/6, S + K4, X); Euler g = fma(h, K, X); correction
    U = F + (g - Gold) (R3), prefix skipped (R14).  Returns U_N after K sweeps."""
    b = 1.0 - lam
    hF, hG = T / (N * mF), T / (N * mG)
    rhs = lambda y: y * (b * y)

    def F(x):
        for _ in range(mF):
            k = rhs(x)
            S = k
            y = _fma(0.5 * hF, k, x)
            k = rhs(y)
            S = _fma(2.0, k, S)
            y = _fma(0.5 * hF, k, x)
            k = rhs(y)
            S = _fma(2.0, k, S)
            y = _fma(hF, k, x)
            k = rhs(y)
            x = _fma(hF / 6.0, S + k, x)
        return x

    def G(x):
        for _ in range(mG):
            x = _fma(hG, rhs(x), x)
        return x

    U = [1.0]
    for n in range(N):
        U.append(G(U[n]))
    Gold = U[1:]
    for k in range(min(K, N)):
        Fk = {n: F(U[n]) for n in range(k, N)}
        V = list(U)
        for n in range(k, N):
            g = G(V[n])
            V[n + 1] = Fk[n] + (g - Gold[n])
            Gold[n] = g
        U = V
    return U[N]


@pytest.mark.parametrize("n,N,mG,mF,K", [(32, 8, 1, 64, 4), (200, 4, 2, 8, 2)])
def test_diagonal_A_matches_scalar_recursion(n, N, mG, mF, K):
    """SURVEY pin P2 (A(t)^{-1} = (1 + t(lam - 1))^{-1} per entry) on the CUDA path, both
    the K6 shared-memory kernels (n = 32) and the batched DMMA GEMMs (n = 200): off-diagonals stay
    exactly 0; each diagonal entry equals the FP64 scalar recursion in the kernels' operation order
    (<= 4 ulp; in practice bitwise), the 50-digit mpmath recursion to <= 1e-13, and at K = N the
    closed form 1/lam within the RK4 error."""
    rng = np.random.default_rng(n)
    lam = rng.uniform(0.5, 1.5, n)
    A = np.diag(lam)
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, N, mG, mF)
    s.solve(K)
    X = s.result()
    off = X - np.diag(np.diag(X))
    assert not np.any(off)
    d = np.diag(X)
    want = np.array([_gpu_order_scalar_parareal_inverse(float(l), 1.0, N, mG, mF, K) for l in lam])
    ulp = np.abs(d - want) / np.spacing(np.abs(want))
    assert ulp.max() <= 4, ulp.max()
    for i in range(0, n, max(1, n // 12)):
        u_mp, _ = spectral.mp_parareal_scalar(lam[i], dense.FLOW_INVERSE, 1, N, mG, mF, K)
        assert abs(d[i] - float(u_mp)) <= 1e-13 * abs(float(u_mp))
    s.solve(N)
    dN = np.diag(s.result())
    hF = 1.0 / (N * mF)
    assert np.max(np.abs(dN * lam - 1.0)) <= 0.1 * hF ** 4 + 1e-13   # RK4 truncation error O(h^4)


def test_invalid_arguments():
    with pytest.raises(mf.MfodeError) as e:
        mf.Solver(np.eye(4), 7, 1.0, 4, 1, 1)
    assert e.value.status == mf.EINVAL
    s = mf.Solver(np.eye(4), mf.FLOW_INVERSE, 1.0, 4, 1, 1)
    with pytest.raises(mf.MfodeError):
        s.solve(-1)
    with pytest.raises(mf.MfodeError):
        s.set_option("nope", 1)


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------------------------
def test_cfg0_full_vs_dense_oracle():
    w = workloads.config(0)
    s, info, X = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    ref = dense.solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert info["k_done"] == ref["k_done"] == 4
    assert relF(X, ref["X"]) <= 1e-10
    assert dense.residual_inverse(w.A, X) < 1e-7          # P3 bound at K = 4


def test_cfg1_full_vs_dense_oracle():
    w = workloads.config(1)
    s, info, X = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    ref = dense.solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-10
    sp = spectral.solve(w.eigvals, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert sp["k_done"] == info["k_done"]
    assert relF(X, spectral.reconstruct(w.eigvecs, sp["X"])) <= 1e-10
    assert s.residual() < 1e-10


@pytest.mark.slow
def test_cfg2_full_vs_spectral_oracle():
    w = workloads.config(2)
    s, info, X = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    sp = spectral.solve(w.eigvals, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert info["k_done"] == sp["k_done"]
    assert relF(X, spectral.reconstruct(w.eigvecs, sp["X"])) <= 1e-10


def test_cfg4_full_bench_workload_vs_spectral_oracle():
    """The bench workload (BASELINE cfg[4], n = 4096, N = 64) in the bench's launch configuration:
    the full output against the spectral oracle (Kronecker sine basis, exact in exact arithmetic)."""
    w = workloads.config(4)
    s, info, X = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    sp = spectral.solve(w.eigvals, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert info["k_done"] == sp["k_done"] == 1
    ref = spectral.reconstruct(w.eigvecs, sp["X"])
    assert relF(X, ref) <= 1e-10
    assert info["residual"] <= 1e-10
    assert abs(info["residual0"] - sp["residual0"]) <= 1e-3 * sp["residual0"] + 1e-15


@pytest.mark.parametrize("n", [5, 32, 48, 64])
@pytest.mark.parametrize("flow", [0, 1])
def test_small_kernels_bitwise_equal_gemm_path(n, flow):
    """K6 (whole propagation in one CTA's shared memory) uses the DMMA issue order, lane->k mapping
    and epilogue arithmetic of the launch-per-GEMM path, so the two agree bitwise; both match the oracle."""
    if flow == 0:
        w = workloads.random_spd(n, 10 + n)
        A, T, N, mG, mF = w.A, 1.0, 8, 1, 16
    else:
        m = int(round(math.sqrt(n)))
        A = workloads.laplacian_2d(m) + np.eye(m * m) if m * m == n else workloads.random_spd(n, 3).A + np.eye(n)
        T, N, mG, mF = 20.0, 64, 2, 32
    res = []
    for small in (1, 0):
        _, info, X = _solve_gpu(A, flow, T, N, mG, mF, 3, small=small)
        res.append((info, X))
    assert np.array_equal(res[0][1], res[1][1])
    assert res[0][0]["deltas"] == res[1][0]["deltas"]
    ref = dense.solve(A, flow, T, N, mG, mF, 3)
    assert relF(res[0][1], ref["X"]) <= 1e-12
    assert res[0][0]["gpu_launches"] < res[1][0]["gpu_launches"]


@pytest.mark.parametrize("n", [5, 17, 32, 33, 64])
@pytest.mark.parametrize("flow", [0, 1, 2])
def test_small_cluster_kernels_bitwise(n, flow):
    """K6c (one slice over a cluster of 2/4/8 CTAs, column-split, Y exchanged through DSMEM each
    stage) keeps each output element's DMMA sequence and epilogue arithmetic, so every cluster size
    agrees bitwise with the one-CTA kernel and with the launch-per-GEMM path; the solve matches the
    oracle.  Ragged n (5, 17, 33) leaves padded columns in some CTAs' column sets."""
    if flow == 1:
        A = workloads.random_spd(n, 5 + n).A + np.eye(n)
        T, N, mG, mF = 20.0, 16, 2, 16
    else:
        A = workloads.random_spd(n, 10 + n).A
        if flow == 2:
            A = A - 1.5 * np.eye(n)
        T, N, mG, mF = 1.0, 8, 1, 16
    sizes = [1, 2, 4] + ([8] if n > 32 else [])
    res = {}
    for cs in sizes:
        _, info, X = _solve_gpu(A, flow, T, N, mG, mF, 3, small_cluster=cs)
        res[cs] = (info, X)
    _, info0, X0 = _solve_gpu(A, flow, T, N, mG, mF, 3, small=0)
    for cs in sizes:
        assert np.array_equal(res[cs][1], X0), cs
        assert res[cs][0]["deltas"] == info0["deltas"], cs
    ref = dense.solve(A, flow, T, N, mG, mF, 3)
    assert relF(X0, ref["X"]) <= 1e-12


def test_small_cluster_option_validation():
    A = workloads.random_spd(32, 1).A
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, 4, 1, 4)
    with pytest.raises(mf.MfodeError):
        s.set_option("small_cluster", 8)    # n <= 32 has 32 columns: at most 4 CTAs of 8
    with pytest.raises(mf.MfodeError):
        s.set_option("small_cluster", 3)


@pytest.mark.parametrize("n", [40, 200])
def test_exp_flow_vs_oracle(n):
    """§8(f) f1: exp flow (Example 2) on the same kernels: GPU vs oracle and vs expm."""
    import scipy.linalg
    A = workloads.random_nonsymmetric(n, 5, scale=1.0) - np.eye(n)
    N, mG, mF, K = 8, 2, 16, 8
    s, info, X = _solve_gpu(A, mf.FLOW_EXP, 1.0, N, mG, mF, K, 1e-13, mf.STOP_DELTA)
    ref = dense.solve(A, dense.FLOW_EXP, 1.0, N, mG, mF, K, 1e-13, dense.STOP_DELTA)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-12
    E = scipy.linalg.expm(A)
    assert relF(X, E) <= 1e-8
    with pytest.raises(mf.MfodeError):
        s.residual()


@pytest.mark.parametrize("n", [24, 130])
def test_trig_flow_vs_oracle(n):
    """§8(f) f1: trig block flow (Example 3, eq. eqB, X0 = 0) -- the 2n x n state (sin; cos) runs as
    pairs of sub-matrices in one batched GEMM (K_X = A Y, K_Y = -A X)."""
    import scipy.linalg
    A = workloads.random_nonsymmetric(n, 7, scale=1.0)
    N, mG, mF = 6, 2, 20
    s = mf.Solver(A, mf.FLOW_TRIG, 1.0, N, mG, mF)
    info = s.solve(N, 1e-13, mf.STOP_DELTA)
    X = np.empty((2 * n, n))
    s.result(X)
    ref = dense.solve(A, dense.FLOW_TRIG, 1.0, N, mG, mF, N, 1e-13, dense.STOP_DELTA)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-12
    assert np.abs(X[:n] - scipy.linalg.sinm(A)).max() < 1e-8
    assert np.abs(X[n:] - scipy.linalg.cosm(A)).max() < 1e-8
    s3 = mf.Solver(A, mf.FLOW_TRIG, 1.0, N, mG, mF, world=3)
    i3 = s3.solve(N, 1e-13, mf.STOP_DELTA)
    X3 = np.empty((2 * n, n))
    s3.result(X3)
    assert np.array_equal(X, X3) and i3["k_done"] == info["k_done"]


def test_cosine_algorithm5_vs_oracle():
    """Algorithm 5 end to end through mfode_cosine vs the oracle's step-by-step version."""
    import scipy.linalg
    n = 60
    A = 0.8 * workloads.random_nonsymmetric(n, 6, scale=2.0)
    C, m, info = mf.cosine(A, 8, 2, 30, 8, 1e-13, mf.STOP_DELTA)
    Cref, mref, out = dense.cosine_algorithm5(A, 8, 2, 30, 8, 1e-13, dense.STOP_DELTA)
    assert m == mref and info["k_done"] == out["k_done"]
    assert relF(C, Cref) <= 1e-10
    assert np.abs(C - scipy.linalg.cosm(A)).max() < 1e-8


@pytest.mark.parametrize("n", [40, 150])
def test_accel_inverse_vs_oracle(n):
    """§8(f) f4: Algorithm 8 on the DMMA GEMM with the EPI_ACCEL epilogue vs the oracle's
    literal loop; with tol the residual ||AX - I||/sqrt(n) is reported."""
    w = workloads.random_spd(n, 11)
    A = w.A / np.linalg.norm(w.A)
    Ainv = np.linalg.inv(A)
    E0 = np.where(np.abs(Ainv) >= 0.01 * np.abs(Ainv).max(), Ainv, 0.0)   # thresholded at 1 %
    dt, K = 0.1, 40
    X, steps, res, status = mf.accel_inverse(A, E0, dt, K)
    ref = dense.accel_inverse(A, E0, dt, K)[K]
    assert steps == K
    assert relF(X, ref) <= 1e-12
    assert abs(res - dense.residual_inverse(A, ref)) <= 1e-9 * max(res, 1e-300) + 1e-14


@pytest.mark.parametrize("flow,n", [(mf.FLOW_TRIG, 8), (mf.FLOW_TRIG, 100), (mf.FLOW_EXP, 40)])
def test_modified_parareal_vs_oracle(flow, n):
    """§8(f) f2: Algorithm 3 on the GPU (Frobenius MGS x2, batched fine images of new
    basis blocks, sequential projected update) vs the oracle; both reach the sequential fine
    solution once the basis saturates, far ahead of classical parareal."""
    w = workloads.random_spd(n, 12, lo=0.5, hi=3.0)
    N, mG, mF, K = 10, 1, 10, 3
    s = mf.Solver(w.A, flow, 1.0, N, mG, mF)
    info = s.solve_modified(K)
    rows = 2 * n if flow == mf.FLOW_TRIG else n
    X = np.empty((rows, n))
    s.result(X)
    ref = dense.solve_modified(w.A, flow, 1.0, N, mG, mF, K)
    seq = dense.solve_sequential_fine(w.A, flow, 1.0, N, mF)
    assert info["k_done"] == K
    assert info["basis_size"] == ref["basis"]          # the same blocks kept (R16)
    assert relF(X, ref["X"]) <= 1e-10
    err_gpu = relF(X, seq)
    c = s.solve(K)
    Xc = np.empty((rows, n))
    s.result(Xc)
    assert err_gpu <= relF(Xc, seq) + 1e-14


@pytest.mark.parametrize("flow,n", [(mf.FLOW_INVERSE, 256), (mf.FLOW_INVERSE, 200), (mf.FLOW_SQRT, 196),
                                    (mf.FLOW_EXP, 130), (mf.FLOW_TRIG, 100)])
def test_symmetric_mode_vs_oracle(flow, n):
    """§8(f) f3(i): with A = A^T every iterate is a symmetric polynomial in A, so each GEMM computes
    only tiles with tile_m <= tile_n and mirrors them (half the flops).  The result is exactly
    symmetric and matches the oracle (full products) within the parity bar; the residual
    reduction counts mirrored entries twice."""
    if flow == mf.FLOW_SQRT:
        m = int(round(math.sqrt(n)))
        A = workloads.laplacian_2d(m) + np.eye(m * m)
        T, N, mG, mF, K, tol, stop = 20.0, 64, 2, 16, 4, 1e-10, mf.STOP_RESIDUAL
    else:
        A = workloads.random_spd(n, 20).A
        T, N, mG, mF, K, tol, stop = 1.0, 6, 1, 8, 6, 1e-11, mf.STOP_DELTA
    s = mf.Solver(A, flow, T, N, mG, mF)
    s.set_option("symmetric", 1)
    info = s.solve(K, tol, stop)
    rows = 2 * n if flow == mf.FLOW_TRIG else n
    X = np.empty((rows, n))
    s.result(X)
    ref = dense.solve(A, flow, T, N, mG, mF, K, tol, stop)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-10
    for b in range(rows // n):
        blk = X[b * n:(b + 1) * n]
        assert np.array_equal(blk, blk.T)
    if flow in (mf.FLOW_INVERSE, mf.FLOW_SQRT):
        r_sym = s.residual()
        r_ref = dense.flow_residual(A, flow)(X)
        assert abs(r_sym - r_ref) <= 1e-6 * r_ref + 1e-15


def test_symmetric_mode_rejects_nonsymmetric():
    A = workloads.random_nonsymmetric(80, 2)
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, 4, 1, 4)
    with pytest.raises(mf.MfodeError):
        s.set_option("symmetric", 1)


def test_small_kernels_logical_ranks_and_sequential():
    w = workloads.config(0)
    s1, i1, X1 = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, 8, 1e-13, mf.STOP_DELTA)
    s4, i4, X4 = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, 8, 1e-13, mf.STOP_DELTA, world=4)
    assert np.array_equal(X1, X4) and i1["k_done"] == i4["k_done"]
    s1.solve(w.N)
    XN = s1.result()
    s1.sequential_fine()
    assert np.array_equal(s1.result(), XN)     # P5 on the K6 path


def test_symmetric_mode_repeatable_inverse_n2048():
    """Regression (round 1): the DMMA consumers read each TMA-filled shared-memory stage with
    generic-proxy loads and released it early to the producer; without a proxy fence the TMA
    refill could overtake a pending load, corrupting one warp's 32 x 16 sub-tile in ~1-3 % of
    symmetric-mode launches (long mirrored epilogues made the producer wait at the stage).
    Repeated symmetric solves of the inverse flow at n = 2048 (TILE_64) must agree bitwise and
    match the full-product result at rounding level."""
    n = 2048
    rng = np.random.default_rng(3)
    G = rng.standard_normal((n, n))
    A = np.eye(n) + (G.T @ G) / (2 * n)
    A = (A + A.T) / 2
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, 4, 1, 4)
    s.set_option("tile", 2)
    s.solve(2)
    ref = s.result()
    s.set_option("symmetric", 1)
    outs = []
    for _ in range(6):
        s.solve(2)
        outs.append(s.result())
    for X in outs:
        assert np.array_equal(X, outs[0])
    assert relF(outs[0], ref) <= 1e-13


@pytest.mark.timeout(600)
def test_speculative_cancellation_never_hangs():
    """Regression (round 1): a speculative launch reads the stop flag the metric kernel sets on the
    coarse stream; when each thread read it on its own, a flip in mid-launch could cancel some warps
    of a CTA (or one CTA of a pair) and leave the rest waiting on barriers forever (seen as cfg[2]
    with K_max = 16 hanging after convergence at k = 8).  The decision is now CTA- (and pair-)
    uniform.  Many converging tolerance-stopped solves with speculation, DMMA and emulated GEMMs."""
    w = workloads.random_spd(1024, 9)
    for emu in (0, 16):
        s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, 16, 1, 3)
        s.set_option("emulation", emu)
        ks = set()
        for _ in range(8):
            info = s.solve(16, 1e-9, mf.STOP_DELTA)
            ks.add(info["k_done"])
        assert len(ks) == 1 and ks.pop() < 16
        s.close()


# ---------------------------------------------------------------------------------------------
# affine flow (eq. eq1) and Algorithm 4
# ---------------------------------------------------------------------------------------------
def _affine_case(n, seed):
    A = workloads.random_nonsymmetric(n, seed, scale=1.0) - np.eye(n)
    rng = np.random.default_rng(seed)
    return A, rng.standard_normal((n, n)), rng.standard_normal((n, n))


@pytest.mark.parametrize("n", [40, 150])
def test_affine_flow_classical_vs_oracle(n):
    """Classical parareal on dU/dt = A U + G with non-symmetric A, a non-commuting source G and a
    general U0 (a transposed operand or a dropped source fails): GPU vs the oracle, delta stop."""
    A, Gs, U0 = _affine_case(n, 31)
    N, mG, mF = 8, 2, 16
    s = mf.Solver(A, mf.FLOW_AFFINE, 1.0, N, mG, mF)
    s.set_affine(Gs, U0)
    info = s.solve(N, 1e-12, mf.STOP_DELTA)
    X = s.result()
    ref = dense.solve(A, dense.FLOW_AFFINE, 1.0, N, mG, mF, N, 1e-12, dense.STOP_DELTA, source=Gs, X0=U0)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-12
    s.sequential_fine()
    seq = dense.solve_sequential_fine(A, dense.FLOW_AFFINE, 1.0, N, mF, source=Gs, X0=U0)
    assert relF(s.result(), seq) <= 1e-13
    with pytest.raises(mf.MfodeError):
        s.residual()


@pytest.mark.parametrize("n", [12, 90])
def test_algorithm4_vs_oracle(n):
    """Algorithm 4 on the GPU (Step -1 F(0)/G(0), device Gram-Schmidt, batched fine images of the new
    blocks stored as F(Q_i) - F(0), eq. (update2)) against the oracle's literal Algorithm 4: the
    same kept blocks and the same iterate; and it is never behind classical parareal."""
    A, Gs, U0 = _affine_case(n, 32)
    N, mG, mF, K = 10, 1, 10, 3
    s = mf.Solver(A, mf.FLOW_AFFINE, 1.0, N, mG, mF)
    s.set_affine(Gs, U0)
    info = s.solve_modified(K)
    X = s.result()
    ref = dense.solve_modified(A, dense.FLOW_AFFINE, 1.0, N, mG, mF, K, source=Gs, X0=U0)
    assert info["k_done"] == K and info["basis_size"] == ref["basis"]
    assert relF(X, ref["X"]) <= 1e-10
    seq = dense.solve_sequential_fine(A, dense.FLOW_AFFINE, 1.0, N, mF, source=Gs, X0=U0)
    s.solve(K)
    assert relF(X, seq) <= relF(s.result(), seq) + 1e-14


def test_algorithm4_zero_source_equals_algorithm3():
    """With G = 0 Step -1 gives F(0) = G(0) = 0 and eq. (update2) is eq. (eq_update): the GPU's
    Algorithm 4 on the affine flow equals its Algorithm 3 on the exp flow (same kept blocks,
    rounding-level iterate)."""
    w = workloads.random_spd(30, 33, lo=0.5, hi=3.0)
    N, mG, mF, K = 8, 1, 8, 3
    s3 = mf.Solver(w.A, mf.FLOW_EXP, 1.0, N, mG, mF)
    i3 = s3.solve_modified(K)
    s4 = mf.Solver(w.A, mf.FLOW_AFFINE, 1.0, N, mG, mF)
    i4 = s4.solve_modified(K)
    assert i3["basis_size"] == i4["basis_size"]
    assert relF(s4.result(), s3.result()) <= 1e-14


def test_example5_steady_inverse_affine_vs_spectral():
    """Example 5's flow dX/dt = I - A X as the affine instance (A, G) -> (-A, I), X0 = 0,
    n = 256 (BASELINE cfg[1]'s matrix): classical and modified parareal vs the spectral oracle
    (x' = -lam x + 1, closed-form sine eigenbasis), and X(T) -> A^{-1}."""
    w = workloads.config(1)
    n = w.n
    T, N, mG, mF = 16.0, 16, 2, 32
    s = mf.Solver(-w.A, mf.FLOW_AFFINE, T, N, mG, mF)
    s.set_affine(np.eye(n), np.zeros((n, n)))
    info = s.solve(N, 1e-11, mf.STOP_DELTA)
    sp = spectral.solve(-w.eigvals, dense.FLOW_AFFINE, T, N, mG, mF, N, 1e-11, dense.STOP_DELTA, gamma=1.0, x0=0.0)
    assert info["k_done"] == sp["k_done"]
    ref = spectral.reconstruct(w.eigvecs, sp["X"])
    X = s.result()
    assert relF(X, ref) <= 1e-10
    assert relF(X, np.linalg.inv(w.A)) <= 1e-5     # e^{-lam_min T} with lam_min ~ 1: ~1e-7
    im = s.solve_modified(6)
    spm = dense.solve_modified(-w.A, dense.FLOW_AFFINE, T, N, mG, mF, 6, source=np.eye(n), X0=np.zeros((n, n)))
    # this spectrum puts several Gram-Schmidt candidates right at the R16 threshold (r_ii / ||Z_i||_F
    # = 1.1e-12, 9.5e-13 in the oracle), so CGS2 and MGS2 rounding may keep one block more or less;
    # such a block carries ~1e-12 of the iterate, far inside the parity bar
    assert abs(im["basis_size"] - spm["basis"]) <= 1
    assert relF(s.result(), spm["X"]) <= 1e-10


# ---------------------------------------------------------------------------------------------
# SPEC stop rule, per-phase timing
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("world", [1, 3])
def test_max_slice_stop_vs_oracle(world):
    """MFODE_STOP_MAX_SLICE: the max over every slice (all ranks) of the sweep's change,
    relative to max(1, ||U_0||_F): the same k_done and metric sequence as the oracle."""
    w = workloads.random_spd(70, 34)
    N, mG, mF = 9, 1, 8
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, N, mG, mF, world=world)
    info = s.solve(N, 1e-9, mf.STOP_MAX_SLICE)
    ref = dense.solve(w.A, dense.FLOW_INVERSE, 1.0, N, mG, mF, N, 1e-9, dense.STOP_MAX_SLICE)
    assert info["k_done"] == ref["k_done"] < N
    # the metric is a difference of nearly equal iterates: relative rounding ~ u ||U|| / ||dU||
    for g, r in zip(info["deltas"], ref["deltas"]):
        assert abs(g - r) <= 1e-6 * r + 1e-15
    assert relF(s.result(), ref["X"]) <= 1e-12


def test_phase_timings_reported():
    """mfode_solve_info carries per-phase device times (Step 0, correction busy time, boundary
    communication, stop tests); with logical ranks the boundary copies are timed as comm."""
    w = workloads.random_spd(512, 35)
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, 8, 1, 4, world=2)
    info = s.solve(4, 1e-12, mf.STOP_DELTA)
    for key in ("ms_coarse", "ms_correct", "ms_comm", "ms_metric"):
        assert info[key] > 0.0, (key, info)
    assert info["ms_coarse"] + info["ms_correct"] < 2 * info["ms_total"]
    s.set_option("phase_timing", 0)
    info0 = s.solve(4, 1e-12, mf.STOP_DELTA)
    assert info0["ms_correct"] == 0.0 and info0["k_done"] == info["k_done"]


def test_modified_parareal_phase_timings():
    """The modified parareal (Algorithm 3) reports its fine images (ms_fine: the sum of
    the fine-image spans) and its sequential projected update (ms_correct) as separate device
    times inside ms_total; timing off changes nothing in the result."""
    w = workloads.random_spd(256, 36, lo=0.5, hi=2.0)
    s = mf.Solver(w.A, mf.FLOW_EXP, 1.0, 8, 1, 8)
    s.solve_modified(1)
    info = s.solve_modified(3)
    X = s.result().copy()
    assert info["ms_fine"] > 0.0 and info["ms_correct"] > 0.0
    assert info["ms_fine"] + info["ms_correct"] <= info["ms_total"] * 1.001
    s.set_option("phase_timing", 0)
    info0 = s.solve_modified(3)
    assert info0["ms_correct"] == 0.0 and info0["basis_size"] == info["basis_size"]
    assert np.array_equal(s.result(), X)


@pytest.mark.timeout(900)
def test_cfg3_full_size_K1_vs_spectral_oracle():
    """BASELINE cfg[3] (the n = 4096 inverse flow of Example 1; BASELINE ties it to the
    8/16/32/64-slices-per-GPU split) at full size in the bench's launch configuration, fixed K = 1
    (Step 0 + one fine sweep of 64 slices x 128 RK4 steps + one correction), against the spectral
    oracle on the host eigendecomposition: elementwise relative Frobenius <= 1e-10."""
    w = workloads.config(3)
    s, info, X = _solve_gpu(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, 1)
    assert info["k_done"] == 1
    sp = spectral.solve(w.eigvals, w.flow, w.T, w.N, w.m_G, w.m_F, 1)
    ref = spectral.reconstruct(w.eigvecs, sp["X"])
    assert relF(X, ref) <= 1e-10
    assert abs(info["deltas"][0] - sp["deltas"][0]) <= 1e-6 * sp["deltas"][0]


# ---------------------------------------------------------------------------------------------
# K10: the fused one-launch fine propagator (fused.cuh)
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("flow,n", [(mf.FLOW_INVERSE, 100), (mf.FLOW_INVERSE, 256), (mf.FLOW_SQRT, 196),
                                    (mf.FLOW_EXP, 130), (mf.FLOW_AFFINE, 120), (mf.FLOW_INVERSE, 300),
                                    (mf.FLOW_INVERSE, 72)])
def test_fused_fine_kernel_bitwise_equal_gemm_path(flow, n):
    """K10 runs every RK4 phase of every slice of a sweep in one persistent launch (ticketed work
    items, per-slice phase counters); its main loop and epilogues are the launch-per-GEMM path's,
    so whole solves agree bitwise (ragged n: partial tiles in every phase), with far fewer launches;
    both match the oracle."""
    if flow == mf.FLOW_SQRT:
        m = int(round(math.sqrt(n)))
        A = workloads.laplacian_2d(m) + np.eye(m * m)
        T, N, mG, mF, K, tol, stop = 20.0, 64, 2, 8, 3, 0.0, mf.STOP_FIXED_K
    else:
        A = workloads.random_spd(n, 40).A if flow != mf.FLOW_AFFINE else _affine_case(n, 40)[0]
        T, N, mG, mF, K, tol, stop = 1.0, 7, 1, 6, 7, 1e-11, mf.STOP_DELTA
    outs = []
    for fused in (1, 0):
        s = mf.Solver(A, flow, T, N, mG, mF)
        if flow == mf.FLOW_AFFINE:
            _, Gs, U0 = _affine_case(n, 40)
            s.set_affine(Gs, U0)
        s.set_option("fused", fused)
        info = s.solve(K, tol, stop)
        outs.append((info, s.result()))
        s.close()
    (i1, X1), (i0, X0) = outs
    assert i1["k_done"] == i0["k_done"]
    assert np.array_equal(X1, X0)
    assert i1["deltas"] == i0["deltas"]
    assert i1["gpu_launches"] < i0["gpu_launches"]
    if flow == mf.FLOW_AFFINE:
        _, Gs, U0 = _affine_case(n, 40)
        ref = dense.solve(A, flow, T, N, mG, mF, K, tol, stop, source=Gs, X0=U0)
    else:
        ref = dense.solve(A, flow, T, N, mG, mF, K, tol, stop)
    assert relF(X1, ref["X"]) <= 1e-12


def test_fused_path_sequential_modified_and_ranks():
    """K10 under every caller: sequential fine (K = N bitwise, P5), logical ranks (P9), the modified
    parareal's batched fine images, and repeated tolerance solves (strictly phased: see solve_impl).  N = 24
    slices of n = 256 (384 tiles per phase) run the two-CTAs-per-SM configuration, the sequential
    runs (one slice) the 64 x 32 one."""
    w = workloads.random_spd(256, 41)
    N = 24
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 8)
    s.set_option("fused", 1)
    s.solve(N)
    XN = s.result()
    s.sequential_fine()
    assert np.array_equal(s.result(), XN)
    ks = {s.solve(N, 1e-9, mf.STOP_DELTA)["k_done"] for _ in range(6)}
    assert len(ks) == 1 and ks.pop() < N
    X1 = s.result()
    s3 = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 8, world=3)
    s3.set_option("fused", 1)
    s3.solve(N, 1e-9, mf.STOP_DELTA)
    assert np.array_equal(s3.result(), X1)
    se = mf.Solver(w.A, mf.FLOW_EXP, 1.0, N, 1, 8)
    ie1 = se.solve_modified(3)
    Xe1 = np.empty((256, 256))
    se.result(Xe1)
    se.set_option("fused", 0)
    ie0 = se.solve_modified(3)
    Xe0 = np.empty((256, 256))
    se.result(Xe0)
    assert ie1["basis_size"] == ie0["basis_size"] and np.array_equal(Xe1, Xe0)


def test_symmetry_check_on_device_is_exact():
    """The symmetric mode (f3(i)) needs A == A^T bitwise; the check runs on the device copy of A (a tile-pair
    kernel) for host and device inputs: one element off by one ulp, or a NaN, disables it."""
    w = workloads.random_spd(100, 50)
    A = w.A.copy()
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, 4, 1, 2)
    s.set_option("symmetric", 1)
    B = A.copy()
    B[3, 97] = np.nextafter(B[3, 97], 2.0)
    s.set_matrix(B)
    with pytest.raises(mf.MfodeError):
        s.set_option("symmetric", 1)
    s.set_matrix(A)
    s.set_option("symmetric", 1)
    C = A.copy()
    C[10, 10] = np.nan
    sd = mf.Solver(torch.from_numpy(C).cuda(), mf.FLOW_INVERSE, 1.0, 4, 1, 2)
    with pytest.raises(mf.MfodeError):
        sd.set_option("symmetric", 1)
    sd2 = mf.Solver(torch.from_numpy(A).cuda(), mf.FLOW_INVERSE, 1.0, 4, 1, 2)
    sd2.set_option("symmetric", 1)


@pytest.mark.parametrize("world,j", [(1, 3), (2, 5), (3, 2)])
def test_fault_injection_names_first_bad_slice(world, j):
    """Failure detection: the test hook poisons U^0_j after Step 0.  F(U^0_j) is then
    NaN, so the first correction sweep makes U^1_{j+1} non-finite while U^1_j (from slice j-1) stays
    finite: the solve must stop with ENONFINITE at k = 1 and name slice j + 1, on any rank layout."""
    w = workloads.random_spd(64, 60)
    N = 8
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 4, world=world)
    s.set_option("inject_nan_slice", j)
    with pytest.raises(mf.MfodeError) as e:
        s.solve(4, 1e-12, mf.STOP_DELTA)
    assert e.value.status == mf.ENONFINITE
    assert e.value.info["k_done"] == 1 and e.value.info["bad_slice"] == j + 1
    s.set_option("inject_nan_slice", 0)
    assert s.solve(4, 1e-12, mf.STOP_DELTA)["k_done"] >= 1      # the handle stays usable


def test_cta_share_bitwise_invariant():
    """Bounded persistence (process-wide option cta_share_us: how much of a launch each persistent CTA
    owns) changes the grid and tile-to-CTA assignment only, never an element's k order: bitwise equal."""
    w = workloads.random_spd(700, 61)
    outs = []
    try:
        for share in (2000, 60):
            s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, 6, 1, 4)
            s.set_option("cta_share_us", share)
            s.solve(3)
            outs.append(s.result())
            s.close()
    finally:
        s = mf.Solver(np.eye(4), mf.FLOW_INVERSE, 1.0, 2, 1, 1)
        s.set_option("cta_share_us", 2000)
    assert np.array_equal(outs[0], outs[1])
