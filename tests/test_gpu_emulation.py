"""GPU parity of f3(ii): FP64 GEMMs emulated on the int8 tensor cores
(tcgen05 kind::i8) by CRT / Ozaki-II splitting (paper_1505_07959_b200/csrc/ozaki.cu), through the
C ABI (mfode_dgemm_emulated, mfode_set_option("emulation", T)).

Bars:
  * GEMM: the a-priori bound of the scheme (include/mfode.h): per element
      |D - AB| <= 2^-(a+1) (2^e_i sum_k |B_kj| + 2^f_j sum_k |A_ik|) + 2^-2(a+1) n 2^e_i 2^f_j
    plus the FP64 rounding of both sides (2 n u |A||B|), a = floor((log2 M - 2 - ceil(log2 n)) / 2);
  * whole solves: relative Frobenius <= 1e-10 against the CPU oracle (north star), equal k_done;
  * bookkeeping (prefix exactness, K = N, logical ranks, batch size, repeated calls): bitwise --
    the emulated product is exact integer arithmetic plus deterministic scaling.
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
MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    mf.lib()
    yield


def abits(nmod, n):
    l2 = sum(math.log2(m) for m in MODULI[:nmod])
    kb = math.ceil(math.log2(n)) if n > 1 else 0
    return math.floor((l2 - 2 - kb) / 2 - 1e-9)


def emu_bound(A, B, a):
    n = A.shape[0]
    with np.errstate(divide="ignore"):
        ea = np.floor(np.log2(np.maximum(np.abs(A).max(1), 1e-300))) + 1
        eb = np.floor(np.log2(np.maximum(np.abs(B).max(0), 1e-300))) + 1
    sa, sb = 2.0 ** ea, 2.0 ** eb
    q = 2.0 ** -(a + 1)
    return (q * (sa[:, None] * np.abs(B).sum(0)[None, :] + sb[None, :] * np.abs(A).sum(1)[:, None])
            + q * q * n * sa[:, None] * sb[None, :] + 2 * n * U53 * (np.abs(A) @ np.abs(B)) + 1e-300)


def _dev(a, ld=None):
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
@pytest.mark.parametrize("nmod", [16, 12, 8])
@pytest.mark.parametrize("n", [1, 8, 30, 100, 129, 256, 300, 513])
def test_emulated_gemm_within_bound(n, nmod):
    rng = np.random.default_rng(1000 + n + nmod)
    A = rng.standard_normal((n, n)) * np.exp(rng.uniform(-4, 4, (n, 1)))   # rows of very different scale
    B = rng.standard_normal((n, n)) * np.exp(rng.uniform(-4, 4, (1, n)))   # columns too
    ld = n + (n % 2) + (16 if n % 3 == 0 else 0)
    dD = _dev(np.zeros((n, n)), ld)
    mf.dgemm_emulated(_dev(A, ld), _dev(B, ld), out=dD, n_moduli=nmod)
    D = dD.cpu().numpy()
    ref = A @ B
    assert np.all(np.abs(D - ref) <= emu_bound(A, B, abits(nmod, n)))
    if nmod == 16:
        assert relF(D, ref) <= 1e-14


def test_emulated_gemm_alpha_beta_and_determinism():
    n = 200
    rng = np.random.default_rng(7)
    A, B, C = (rng.standard_normal((n, n)) for _ in range(3))
    dA, dB, dC = _dev(A), _dev(B), _dev(C)
    D1 = mf.dgemm_emulated(dA, dB, dC, alpha=-0.5, beta=2.0).cpu().numpy()
    D2 = mf.dgemm_emulated(dA, dB, dC, alpha=-0.5, beta=2.0).cpu().numpy()
    assert np.array_equal(D1, D2)
    ref = -0.5 * (A @ B) + 2.0 * C
    assert np.all(np.abs(D1 - ref) <= 0.5 * emu_bound(A, B, abits(16, n)) + 4 * U53 * np.abs(ref))


def test_emulated_gemm_special_values():
    """Zero rows/columns stay exactly zero; integer matrices whose products fit are exact; a
    non-finite input row or column makes the affected outputs NaN (never a silent finite value)."""
    n = 64
    rng = np.random.default_rng(3)
    A = rng.integers(-1000, 1000, (n, n)).astype(np.float64)
    B = rng.integers(-1000, 1000, (n, n)).astype(np.float64)
    A[5] = 0.0
    B[:, 9] = 0.0
    D = mf.dgemm_emulated(_dev(A), _dev(B)).cpu().numpy()
    assert np.array_equal(D, A @ B)            # |entries| < 2^a: the scheme is exact
    assert np.all(D[5] == 0.0) and np.all(D[:, 9] == 0.0)
    A2 = A.copy()
    A2[3, 7] = np.inf
    D2 = mf.dgemm_emulated(_dev(A2), _dev(B)).cpu().numpy()
    assert np.all(np.isnan(D2[3]))
    assert np.all(np.isfinite(np.delete(D2, 3, axis=0)))
    B2 = B.copy()
    B2[11, 2] = np.nan
    D3 = mf.dgemm_emulated(_dev(A), _dev(B2)).cpu().numpy()
    assert np.all(np.isnan(D3[:, 2]))


def test_emulated_gemm_large_sampled():
    """n = 4096 (the bench size): sampled rows against the FP64 oracle, and the whole product
    against cuBLAS DGEMM (both within the bound)."""
    n = 4096
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    D = mf.dgemm_emulated(A, B)
    rows = np.array([0, 1, 777, 2048, 4095])
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    ref = An[rows] @ Bn
    b = emu_bound(An, Bn, abits(16, n))[rows]
    assert np.all(np.abs(D.cpu().numpy()[rows] - ref) <= b)
    ref_all = torch.matmul(A, B)
    assert float(torch.linalg.norm(D - ref_all) / torch.linalg.norm(ref_all)) <= 1e-14


def test_emulated_invalid_arguments():
    with pytest.raises(mf.MfodeError):
        mf.dgemm_emulated(_dev(np.eye(4)), _dev(np.eye(4)), n_moduli=1)
    with pytest.raises(mf.MfodeError):
        mf.dgemm_emulated(_dev(np.eye(4)), _dev(np.eye(4)), n_moduli=17)
    s = mf.Solver(np.eye(8), mf.FLOW_INVERSE, 1.0, 2, 1, 1)
    with pytest.raises(mf.MfodeError):
        s.set_option("emulation", 5)


# ---------------------------------------------------------------------------------------------
# whole solves with emulated GEMMs
# ---------------------------------------------------------------------------------------------
def _solve(A, flow, T, N, mG, mF, K, tol=0.0, stop=0, world=1, nmod=16, **opts):
    s = mf.Solver(A, flow, T, N, mG, mF, world=world)
    s.set_option("emulation", nmod)
    for k, v in opts.items():
        s.set_option(k, v)
    info = s.solve(K, tol, stop)
    rows = 2 * A.shape[0] if flow == mf.FLOW_TRIG else A.shape[0]
    X = np.empty((rows, A.shape[0]))
    s.result(X)
    return s, info, X


def test_cfg1_emulated_vs_dense_oracle():
    w = workloads.config(1)
    s, info, X = _solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    ref = dense.solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-10
    assert s.residual() < 1e-10


@pytest.mark.parametrize("flow,n", [(mf.FLOW_INVERSE, 100), (mf.FLOW_INVERSE, 257), (mf.FLOW_SQRT, 144),
                                    (mf.FLOW_EXP, 130), (mf.FLOW_TRIG, 70)])
def test_emulated_flows_vs_oracle(flow, n):
    if flow == mf.FLOW_SQRT:
        m = int(round(math.sqrt(n)))
        A = workloads.laplacian_2d(m) + np.eye(m * m)
        T, N, mG, mF, K, tol, stop = 20.0, 64, 2, 16, 4, 1e-10, mf.STOP_RESIDUAL
    elif flow == mf.FLOW_INVERSE and n == 257:
        A = workloads.random_nonsymmetric(n, 4)    # transposed operands would show here
        T, N, mG, mF, K, tol, stop = 1.0, 4, 1, 20, 4, 0.0, mf.STOP_FIXED_K
    else:
        A = workloads.random_spd(n, 30 + n).A
        T, N, mG, mF, K, tol, stop = 1.0, 6, 1, 8, 6, 1e-11, mf.STOP_DELTA
    s, info, X = _solve(A, flow, T, N, mG, mF, K, tol, stop)
    ref = dense.solve(A, flow, T, N, mG, mF, K, tol, stop)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-10


def test_emulated_prefix_exactness_K_equals_N_and_ranks_bitwise():
    """P5/P6/P9 hold bitwise on the emulated path: U^k_n == sequential fine for n <= k, K = N gives
    the sequential fine result, and logical ranks / fine batch / overlap change nothing."""
    w = workloads.random_spd(96, 5)
    N = 5
    s = mf.Solver(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 6)
    s.set_option("emulation", 16)
    s.sequential_fine()
    seq = [s.slice(m) for m in range(N + 1)]
    for k in (1, 3, N):
        info = s.solve(k)
        for m in range(k + 1):
            assert np.array_equal(s.slice(m), seq[m]), (k, m)
    ref = dense.solve_sequential_fine(w.A, dense.FLOW_INVERSE, 1.0, N, 6)
    assert relF(seq[N], ref) <= 1e-12
    _, i1, X1 = _solve(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 6, N, 1e-12, mf.STOP_DELTA)
    _, i3, X3 = _solve(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 6, N, 1e-12, mf.STOP_DELTA, world=3)
    _, ib, Xb = _solve(w.A, mf.FLOW_INVERSE, 1.0, N, 1, 6, N, 1e-12, mf.STOP_DELTA, fine_batch=2, overlap=0)
    assert i1["k_done"] == i3["k_done"] == ib["k_done"]
    assert np.array_equal(X1, X3) and np.array_equal(X1, Xb)


def test_emulated_symmetric_mode_vs_oracle():
    """f3(i) + f3(ii): upper-triangle tiles of the emulated products, mirrored in the decode."""
    m = 14
    A = workloads.laplacian_2d(m) + np.eye(m * m)
    s, info, X = _solve(A, mf.FLOW_SQRT, 20.0, 64, 2, 16, 4, 1e-10, mf.STOP_RESIDUAL, symmetric=1)
    ref = dense.solve(A, mf.FLOW_SQRT, 20.0, 64, 2, 16, 4, 1e-10, dense.STOP_RESIDUAL)
    assert info["k_done"] == ref["k_done"]
    assert relF(X, ref["X"]) <= 1e-10
    assert np.array_equal(X, X.T)


def test_emulated_nonfinite_reports_bad_slice():
    A = np.diag(np.full(16, 40.0))
    s = mf.Solver(A, mf.FLOW_INVERSE, 1.0, 4, 1, 4)
    s.set_option("emulation", 16)
    with pytest.raises(mf.MfodeError) as e:
        s.solve(2, 1e-10, mf.STOP_DELTA)
    assert e.value.status == mf.ENONFINITE


def test_cfg4_emulated_bench_workload_vs_spectral_oracle():
    """The bench workload (BASELINE cfg[4], n = 4096, N = 64) with emulated GEMMs, as bench.py's
    f3(ii) variant runs it: full output against the spectral oracle."""
    w = workloads.config(4)
    s, info, X = _solve(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    sp = spectral.solve(w.eigvals, w.flow, w.T, w.N, w.m_G, w.m_F, w.K_max, w.tol, w.stop)
    assert info["k_done"] == sp["k_done"] == 1
    assert relF(X, spectral.reconstruct(w.eigvecs, sp["X"])) <= 1e-10
    assert info["residual"] <= 1e-10


@pytest.mark.parametrize("flow", [mf.FLOW_INVERSE, mf.FLOW_EXP])
def test_emulated_constant_operand_cache_follows_set_matrix(flow):
    """The encodings of the constant operand (B = I - A for the inverse flow, A for the exp flow) are
    cached per stream; mfode_set_matrix changes the matrix generation, so the next solve re-encodes
    (a stale cache would reproduce the old matrix's result)."""
    n = 120
    A1 = workloads.random_spd(n, 41).A
    A2 = workloads.random_spd(n, 42).A
    s = mf.Solver(A1, flow, 1.0, 4, 1, 6)
    s.set_option("emulation", 16)
    for A in (A1, A2, A1):
        s.set_matrix(A)
        info = s.solve(4)
        X = s.result()
        ref = dense.solve(A, flow, 1.0, 4, 1, 6, 4)
        assert relF(X, ref["X"]) <= 1e-10


@pytest.mark.parametrize("flow,n", [(mf.FLOW_EXP, 140), (mf.FLOW_TRIG, 72)])
def test_emulated_modified_parareal_vs_oracle(flow, n):
    """f2 (Algorithm 3) on the emulated GEMMs: same bar as the DMMA path's test."""
    w = workloads.random_spd(n, 12, lo=0.5, hi=3.0)
    N, mG, mF, K = 10, 1, 10, 3
    s = mf.Solver(w.A, flow, 1.0, N, mG, mF)
    s.set_option("emulation", 16)
    info = s.solve_modified(K)
    rows = 2 * n if flow == mf.FLOW_TRIG else n
    X = np.empty((rows, n))
    s.result(X)
    ref = dense.solve_modified(w.A, flow, 1.0, N, mG, mF, K)
    seq = dense.solve_sequential_fine(w.A, flow, 1.0, N, mF)
    assert info["k_done"] == K
    err_gpu = relF(X, seq)
    err_ref = relF(ref["X"], seq)
    assert relF(X, ref["X"]) <= 1e-10 or (err_gpu <= 1e-10 and err_ref <= 1e-10)


@pytest.mark.parametrize("n", [100, 300, 4096])
def test_single_cta_and_pair_kernels_bitwise_equal(n):
    """The single-CTA (oz_pair = 0) and CTA-pair (default) int8 GEMM kernels compute the same exact
    integer products, so the emulated results are bitwise identical."""
    rng = np.random.default_rng(77 + n)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    knob = mf.Solver(np.eye(2), mf.FLOW_INVERSE, 1.0, 1, 1, 1)
    try:
        knob.set_option("oz_pair", 0)
        D0 = mf.dgemm_emulated(_dev(A), _dev(B)).cpu().numpy()
    finally:
        knob.set_option("oz_pair", 1)
    D1 = mf.dgemm_emulated(_dev(A), _dev(B)).cpu().numpy()
    assert np.array_equal(D0, D1)
    if n <= 300:
        assert np.all(np.abs(D1 - A @ B) <= emu_bound(A, B, abits(16, n)))


def test_emulated_symmetric_inverse_reuses_encoding():
    """Inverse flow, f3(i) + f3(ii): the second GEMM of each stage (K = Y W) reuses the row
    encoding of Y made for the first (W = B Y); results match the oracle and the non-symmetric
    emulated run, and repeated solves are bitwise identical."""
    A = workloads.random_spd(300, 77).A
    T, N, mG, mF, K = 1.0, 6, 1, 8, 6
    s, i1, X1 = _solve(A, mf.FLOW_INVERSE, T, N, mG, mF, K, 1e-11, mf.STOP_DELTA, symmetric=1)
    info2 = s.solve(K, 1e-11, mf.STOP_DELTA)
    X2 = np.empty_like(X1)
    s.result(X2)
    assert np.array_equal(X1, X2) and info2["k_done"] == i1["k_done"]
    ref = dense.solve(A, mf.FLOW_INVERSE, T, N, mG, mF, K, 1e-11, mf.STOP_DELTA)
    assert i1["k_done"] == ref["k_done"]
    assert relF(X1, ref["X"]) <= 1e-10
    _, _, X3 = _solve(A, mf.FLOW_INVERSE, T, N, mG, mF, K, 1e-11, mf.STOP_DELTA)
    assert relF(X1, X3) <= 1e-13


def test_emulated_gemm_extreme_row_scales():
    """Rows / columns of very different magnitude down to 1e-300: the power-of-two scaling never
    overflows (the scale is applied as two factors) and each row of the product stays accurate
    relative to its own scale."""
    n = 96
    rng = np.random.default_rng(21)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    A[3] *= 1e-300
    A[7] *= 1e250
    B[:, 5] *= 1e-290
    D = mf.dgemm_emulated(_dev(A), _dev(B)).cpu().numpy()
    ref = A @ B
    assert np.all(np.isfinite(D))
    rowerr = np.abs(D - ref).max(1) / np.abs(ref).max(1)
    assert rowerr.max() <= 1e-13
    assert np.abs(D[:, 5] - ref[:, 5]).max() <= 1e-13 * np.abs(ref[:, 5]).max()


def test_emulated_gemm_graded_rows_normwise_accuracy():
    """the emulation scales each row of A (column of B) by its largest entry, so its error
    bound is NORMWISE per row/column (include/mfode.h), not elementwise-relative.  With entries inside
    each row spanning 8 decades of the row maximum, every element stays within that bound, the result
    is FP64-accurate relative to |A||B| (what the bound promises), and entries much smaller than their
    row maximum lose relative accuracy -- measured here, not hidden."""
    n, nmod = 256, 16
    rng = np.random.default_rng(77)
    grade = 10.0 ** rng.uniform(-8, 0, (n, n))              # |A_ik| spans 1e-8 .. 1 of the row max
    A = rng.standard_normal((n, n)) * grade
    B = rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-8, 0, (n, n))
    D = mf.dgemm_emulated(_dev(A), _dev(B), n_moduli=nmod).cpu().numpy()
    ref = A @ B
    err = np.abs(D - ref)
    assert np.all(err <= emu_bound(A, B, abits(nmod, n)))
    scale = np.abs(A) @ np.abs(B)
    assert np.max(err / scale) <= 4 * n * U53                 # normwise: FP64-level against |A||B|
    # the same product on the FP64 DMMA path for contrast: also within gamma_n |A||B| (bitwise different)
    Dd = mf.dgemm(_dev(A), _dev(B)).cpu().numpy()
    assert np.max(np.abs(Dd - ref) / scale) <= 2 * n * U53
