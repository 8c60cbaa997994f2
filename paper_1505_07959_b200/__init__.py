"""Python binding of the mfode C-ABI library (include/mfode.h): argument marshalling only.

Every step of the parareal path runs in the CUDA library (libmfode.so, sm_100a).  There is no
CPU fallback: if the library is missing or cannot be loaded, every entry point raises.  PyTorch is
used by callers only for device memory, streams and process groups; this module accepts numpy
arrays (host) or torch CUDA tensors (device) and passes raw pointers.

Names follow the paper (Chehab & Petcu, arXiv 1505.07959): flows of P:44 (inverse) and P:46-51
(steady state / square root), classical parareal Algorithm 1.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmfode.so")

FLOW_INVERSE = 0
FLOW_SQRT = 1
FLOW_EXP = 2
FLOW_TRIG = 3      # state (sin, cos) stacked 2n x n (Example 3, eq. eqB)
FLOW_AFFINE = 4    # dU/dt = A U + G, U(0) = U0 (eq. eq1; Example 5 with (A, G) -> (-A, I))
STOP_FIXED_K = 0
STOP_DELTA = 1
STOP_RESIDUAL = 2
STOP_MAX_SLICE = 3  # max_n ||U^{k+1}_n - U^k_n||_F <= tol max(1, ||U_0||_F)
TILE_AUTO, TILE_128, TILE_64, TILE_32 = 0, 1, 2, 3

OK, NOT_CONVERGED, EINVAL, ENOMEM, ECUDA, ENCCL, ENONFINITE = 0, 1, -1, -2, -3, -4, -5
_STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL", -5: "ENONFINITE"}

EXPORTED = [
    "mfode_create", "mfode_create_device", "mfode_set_matrix", "mfode_parareal_solve", "mfode_sequential_fine",
    "mfode_residual", "mfode_get_result", "mfode_get_result_device", "mfode_get_slice", "mfode_set_option",
    "mfode_last_error", "mfode_destroy", "mfode_dgemm", "mfode_rk_stage", "mfode_frobenius", "mfode_partition",
    "mfode_kernel_launches", "mfode_last_global_error", "mfode_version", "mfode_cosine", "mfode_accel_inverse",
    "mfode_modified_parareal_solve", "mfode_dgemm_emulated", "mfode_release_workspace", "mfode_set_affine",
]


class MfodeError(RuntimeError):
    """A negative mfode_status.  ``info`` holds the solve's mfode_solve_info (as a dict) when the
    failing call filled one -- e.g. ``info["bad_slice"]`` for MFODE_ENONFINITE."""

    def __init__(self, status: int, msg: str, info: Optional[dict] = None):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.info = info


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("device", ctypes.c_int),
                ("nccl_uid", ctypes.c_void_p)]


class SolveInfo(ctypes.Structure):
    _fields_ = [("k_done", ctypes.c_int), ("bad_slice", ctypes.c_int), ("converged", ctypes.c_int),
                ("world", ctypes.c_int), ("last_delta", ctypes.c_double), ("residual", ctypes.c_double),
                ("residual0", ctypes.c_double), ("ms_total", ctypes.c_double), ("ms_fine", ctypes.c_double),
                ("fine_flops", ctypes.c_double), ("coarse_flops", ctypes.c_double), ("gpu_launches", ctypes.c_int),
                ("fine_kernel_launches", ctypes.c_int), ("fine_kernel_ms", ctypes.c_double),
                ("fine_kernel_flops", ctypes.c_double), ("deltas", ctypes.c_double * 64),
                ("basis_size", ctypes.c_int), ("ms_coarse", ctypes.c_double), ("ms_correct", ctypes.c_double),
                ("ms_comm", ctypes.c_double), ("ms_metric", ctypes.c_double)]

    def to_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "deltas"}
        d["deltas"] = [x for x in list(self.deltas)[: self.k_done]]
        return d


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmfode.so (raises if absent: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run python -m paper_1505_07959_b200.build "
                          "(there is no CPU fallback for the CUDA path)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, I, D, I64, V = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "mfode_create": (I, [ctypes.POINTER(P), P, I64, I, D, I, I, I, ctypes.POINTER(Dist)]),
        "mfode_create_device": (I, [ctypes.POINTER(P), P, I64, I, D, I, I, I, ctypes.POINTER(Dist), P]),
        "mfode_set_matrix": (I, [P, P]),
        "mfode_set_affine": (I, [P, P, P]),
        "mfode_parareal_solve": (I, [P, I, D, I, ctypes.POINTER(SolveInfo)]),
        "mfode_sequential_fine": (I, [P, ctypes.POINTER(SolveInfo)]),
        "mfode_residual": (I, [P, ctypes.POINTER(D)]),
        "mfode_get_result": (I, [P, P]),
        "mfode_get_result_device": (I, [P, P, P]),
        "mfode_get_slice": (I, [P, I, P]),
        "mfode_set_option": (I, [P, ctypes.c_char_p, I64]),
        "mfode_last_error": (ctypes.c_char_p, [P]),
        "mfode_destroy": (None, [P]),
        "mfode_dgemm": (I, [P, P, P, P, I64, I64, D, D, I, P]),
        "mfode_dgemm_emulated": (I, [P, P, P, P, I64, I64, D, D, I, P]),
        "mfode_release_workspace": (I, [P]),
        "mfode_rk_stage": (I, [P, P, P, D, D, P, P, P, I, D, I64, I64, I, P]),
        "mfode_frobenius": (I, [P, P, I64, I64, ctypes.POINTER(D), P]),
        "mfode_partition": (I, [I, I, I, ctypes.POINTER(I), ctypes.POINTER(I)]),
        "mfode_kernel_launches": (ctypes.c_int64, []),
        "mfode_last_global_error": (ctypes.c_char_p, []),
        "mfode_version": (ctypes.c_char_p, []),
        "mfode_cosine": (I, [P, I64, I, I, I, I, D, I, ctypes.POINTER(Dist), P, ctypes.POINTER(I),
                             ctypes.POINTER(SolveInfo)]),
        "mfode_accel_inverse": (I, [P, P, P, I64, D, I, D, I, P, ctypes.POINTER(I), ctypes.POINTER(D)]),
        "mfode_modified_parareal_solve": (I, [P, I, D, I, I, ctypes.POINTER(SolveInfo)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status: int, handle=None, info: Optional["SolveInfo"] = None) -> int:
    if status < 0:
        L = lib()
        msg = L.mfode_last_error(handle) if handle else L.mfode_last_global_error()
        raise MfodeError(status, (msg or b"").decode(), info.to_dict() if info is not None else None)
    return status


def _ptr(x) -> Optional[int]:
    """Raw pointer of a numpy array (host) or torch CUDA tensor (device), or None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _host_square(M, n: int, name: str, rows: Optional[int] = None) -> np.ndarray:
    """A C-contiguous float64 host copy of M with shape (rows or n, n), else ValueError (raw pointers
    cross the ABI: a wrong shape would make the library read or write past the buffer)."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    want = (rows if rows is not None else n, n)
    if M.shape != want:
        raise ValueError(f"{name} must have shape {want}, got {M.shape}")
    return M


def _host_out(out, shape, name: str) -> np.ndarray:
    """Validate (or allocate) a host output buffer written by the library."""
    if out is None:
        return np.empty(shape, dtype=np.float64)
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or not out.flags.c_contiguous \
            or not out.flags.writeable or out.shape != tuple(shape):
        raise ValueError(f"{name} must be a writable C-contiguous float64 array of shape {tuple(shape)}")
    return out


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


# ---------------------------------------------------------------------------------------------
# solver handle
# ---------------------------------------------------------------------------------------------
class Solver:
    """f(A) by classical parareal on dX/dt = F(X), X0 = I (mfode_create / mfode_parareal_solve)."""

    def __init__(self, A, flow: int, T: float, N: int, m_G: int, m_F: int, *, world: int = 1, rank: int = 0,
                 device: Optional[int] = None, nccl_uid: Optional[bytes] = None, stream=None):
        L = lib()
        self._h = ctypes.c_void_p()
        dist = None
        if device is None:
            device = 0
            try:
                import torch
                if torch.cuda.is_available():
                    device = torch.cuda.current_device()
            except ImportError:
                pass
        self._uid_buf = None
        if world > 1 or nccl_uid is not None or device != 0:
            uid_p = None
            if nccl_uid is not None:
                self._uid_buf = ctypes.create_string_buffer(bytes(nccl_uid), 128)
                uid_p = ctypes.cast(self._uid_buf, ctypes.c_void_p)
            dist = Dist(rank, world, device, uid_p)
        if isinstance(A, np.ndarray):
            A = np.ascontiguousarray(A, dtype=np.float64)
            if A.ndim != 2 or A.shape[0] != A.shape[1]:
                raise ValueError(f"A must be square, got shape {A.shape}")
            self.n = A.shape[0]
            st = L.mfode_create(ctypes.byref(self._h), A.ctypes.data, self.n, flow, T, N, m_G, m_F,
                                ctypes.byref(dist) if dist else None)
        else:   # torch CUDA tensor
            if not (getattr(A, "is_cuda", False) and str(A.dtype) == "torch.float64" and A.is_contiguous()
                    and A.dim() == 2 and A.shape[0] == A.shape[1]):
                raise ValueError("A must be a numpy array or a square, contiguous CUDA float64 tensor")
            self.n = A.shape[0]
            st = L.mfode_create_device(ctypes.byref(self._h), A.data_ptr(), self.n, flow, T, N, m_G, m_F,
                                       ctypes.byref(dist) if dist else None, _stream_ptr(stream))
        _check(st)
        self.flow, self.T, self.N, self.m_G, self.m_F, self.world = flow, T, N, m_G, m_F, world
        self.state_rows = 2 * self.n if flow == FLOW_TRIG else self.n   # the trig state is (sin; cos)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().mfode_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_matrix(self, A: np.ndarray):
        A = _host_square(A, self.n, "A")
        _check(lib().mfode_set_matrix(self._h, A.ctypes.data), self._h)

    def set_affine(self, G: Optional[np.ndarray] = None, U0: Optional[np.ndarray] = None):
        """FLOW_AFFINE: source G (None = 0) and initial state U0 (None = I) (mfode_set_affine)."""
        G = None if G is None else _host_square(G, self.n, "G")
        U0 = None if U0 is None else _host_square(U0, self.n, "U0")
        _check(lib().mfode_set_affine(self._h, _ptr(G), _ptr(U0)), self._h)

    def set_option(self, key: str, value: int):
        _check(lib().mfode_set_option(self._h, key.encode(), int(value)), self._h)

    def solve(self, K_max: int, tol: float = 0.0, stop: int = STOP_FIXED_K) -> dict:
        info = SolveInfo()
        st = _check(lib().mfode_parareal_solve(self._h, K_max, tol, stop, ctypes.byref(info)), self._h, info)
        d = info.to_dict()
        d["status"] = _STATUS[st]
        return d

    def solve_modified(self, K_max: int, tol: float = 0.0, stop: int = STOP_FIXED_K, max_basis: int = 0) -> dict:
        """Modified parareal: Algorithm 3 (exp, trig flows) or Algorithm 4 (affine flow)."""
        info = SolveInfo()
        st = _check(lib().mfode_modified_parareal_solve(self._h, K_max, tol, stop, max_basis, ctypes.byref(info)),
                    self._h, info)
        d = info.to_dict()
        d["status"] = _STATUS[st]
        return d

    def sequential_fine(self) -> dict:
        info = SolveInfo()
        _check(lib().mfode_sequential_fine(self._h, ctypes.byref(info)), self._h)
        return info.to_dict()

    def residual(self) -> float:
        r = ctypes.c_double()
        _check(lib().mfode_residual(self._h, ctypes.byref(r)), self._h)
        return r.value

    def result(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """U_N on the host: n x n, or 2n x n (sin; cos) for the trig flow."""
        out = _host_out(out, (self.state_rows, self.n), "out")
        _check(lib().mfode_get_result(self._h, out.ctypes.data), self._h)
        return out

    def result_device(self, out, stream=None):
        if not (getattr(out, "is_cuda", False) and str(out.dtype) == "torch.float64" and out.is_contiguous()
                and tuple(out.shape) == (self.state_rows, self.n)):
            raise ValueError(f"out must be a contiguous CUDA float64 tensor of shape {(self.state_rows, self.n)}")
        _check(lib().mfode_get_result_device(self._h, out.data_ptr(), _stream_ptr(stream)), self._h)
        return out

    def slice(self, n_index: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = _host_out(out, (self.state_rows, self.n), "out")
        _check(lib().mfode_get_slice(self._h, n_index, out.ctypes.data), self._h)
        return out


# ---------------------------------------------------------------------------------------------
# kernel-level entry points (torch CUDA float64 tensors, row-major, leading dimension = stride(0))
# ---------------------------------------------------------------------------------------------
def _square_operands(named: dict, ref_name: str):
    """Validate the device operands of a kernel-level call before raw pointers cross the ABI: every
    tensor must be CUDA float64 on one device, n x n, unit column stride, with the SAME row stride
    (the single leading dimension the C ABI takes) and 16-byte aligned.  Returns (n, ld)."""
    ref = named[ref_name]
    n = ref.shape[0]
    ld = ref.stride(0)
    for name, t in named.items():
        if t is None:
            continue
        if not getattr(t, "is_cuda", False):
            raise ValueError(f"{name} must be a CUDA tensor")
        if str(t.dtype) != "torch.float64":
            raise ValueError(f"{name} must be float64, got {t.dtype}")
        if t.device != ref.device:
            raise ValueError(f"{name} is on {t.device}, {ref_name} on {ref.device}")
        if t.dim() != 2 or tuple(t.shape) != (n, n):
            raise ValueError(f"{name} must be {n} x {n}, got {tuple(t.shape)}")
        if t.stride(1) != 1 or t.stride(0) != ld:
            raise ValueError(f"{name} must be row-major with row stride {ld} (got strides {t.stride()}); "
                             "transposed or differently padded views are not supported")
        if t.data_ptr() % 16 != 0:
            raise ValueError(f"{name} must be 16-byte aligned")
    if ld < n or (ld * 8) % 16 != 0:
        raise ValueError(f"row stride {ld} must be >= n = {n} and a multiple of 2 doubles")
    return n, ld

def dgemm(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, out=None, tile: int = TILE_AUTO, stream=None):
    """D = alpha A B + beta C on the B200 FP64 DMMA/TMA GEMM (mfode_dgemm)."""
    import torch
    if out is None:
        out = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, device=A.device)
    if beta != 0.0 and C is None:
        raise ValueError("C is required when beta != 0")
    n, ld = _square_operands({"A": A, "B": B, "C": C, "out": out}, "A")
    if out.data_ptr() in (A.data_ptr(), B.data_ptr()):
        raise ValueError("out must not alias A or B")
    _check(lib().mfode_dgemm(_ptr(A), _ptr(B), _ptr(C), _ptr(out), n, ld, alpha, beta, tile,
                             _stream_ptr(stream if stream is not None else torch.cuda.current_stream())))
    return out


def dgemm_emulated(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, out=None, n_moduli: int = 16,
                   stream=None):
    """D = alpha A B + beta C emulated on the int8 tensor cores (mfode_dgemm_emulated, f3(ii))."""
    import torch
    if out is None:
        out = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, device=A.device)
    if beta != 0.0 and C is None:
        raise ValueError("C is required when beta != 0")
    n, ld = _square_operands({"A": A, "B": B, "C": C, "out": out}, "A")
    if out.data_ptr() in (A.data_ptr(), B.data_ptr()):
        raise ValueError("out must not alias A or B")
    _check(lib().mfode_dgemm_emulated(_ptr(A), _ptr(B), _ptr(C), _ptr(out), n, ld, alpha, beta, n_moduli,
                                      _stream_ptr(stream if stream is not None else torch.cuda.current_stream())))
    return out


def release_workspace(stream=None):
    """Free the emulated-GEMM scratch cached for `stream` (mfode_release_workspace)."""
    import torch
    _check(lib().mfode_release_workspace(_stream_ptr(stream if stream is not None else torch.cuda.current_stream())))


def rk_stage(Yop, Bop, X, S, Ynext, stage: int, h: float, C=None, alpha: float = 1.0, beta: float = 0.0,
             tile: int = TILE_AUTO, stream=None):
    """One fused RK4 stage (mfode_rk_stage): K = alpha Yop Bop + beta C, then the stage update."""
    import torch
    if beta != 0.0 and C is None:
        raise ValueError("C is required when beta != 0")
    if stage < 4 and Ynext is None:
        raise ValueError("Ynext is required for stages 1-3")
    n, ld = _square_operands({"Yop": Yop, "Bop": Bop, "C": C, "X": X, "S": S, "Ynext": Ynext}, "X")
    _check(lib().mfode_rk_stage(_ptr(Yop), _ptr(Bop), _ptr(C), alpha, beta, _ptr(X), _ptr(S), _ptr(Ynext), stage,
                                h, n, ld, tile,
                                _stream_ptr(stream if stream is not None else torch.cuda.current_stream())))


def frobenius(X, Y=None, stream=None):
    """(||X - Y||_F, ||X||_F) by the library's deterministic reduction (mfode_frobenius)."""
    import torch
    out = (ctypes.c_double * 2)()
    n, ld = _square_operands({"X": X, "Y": Y}, "X")
    _check(lib().mfode_frobenius(_ptr(X), _ptr(Y), n, ld, out,
                                 _stream_ptr(stream if stream is not None else torch.cuda.current_stream())))
    return out[0], out[1]


def cosine(A: np.ndarray, N: int, m_G: int, m_F: int, K_max: int, tol: float = 0.0, stop: int = STOP_FIXED_K,
           world: int = 1):
    """Algorithm 5 through mfode_cosine: returns (cos(A), m, info)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    A = _host_square(A, n, "A")
    C = np.empty((n, n), dtype=np.float64)
    m = ctypes.c_int()
    info = SolveInfo()
    dist = Dist(0, world, 0, None) if world > 1 else None
    _check(lib().mfode_cosine(A.ctypes.data, n, N, m_G, m_F, K_max, tol, stop,
                              ctypes.byref(dist) if dist else None, C.ctypes.data, ctypes.byref(m),
                              ctypes.byref(info)))
    return C, m.value, info.to_dict()


def accel_inverse(A: np.ndarray, E0: Optional[np.ndarray], dt: float, max_steps: int, tol: float = 0.0,
                  check_every: int = 0, X0: Optional[np.ndarray] = None):
    """Algorithm 8 through mfode_accel_inverse: returns (X, steps, residual, status)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    A = _host_square(A, n, "A")
    X = np.empty((n, n), dtype=np.float64)
    E0 = None if E0 is None else _host_square(E0, n, "E0")
    X0 = None if X0 is None else _host_square(X0, n, "X0")
    steps, res = ctypes.c_int(), ctypes.c_double()
    st = _check(lib().mfode_accel_inverse(A.ctypes.data, _ptr(X0), _ptr(E0), n, dt, max_steps, tol, check_every,
                                          X.ctypes.data, ctypes.byref(steps), ctypes.byref(res)))
    return X, steps.value, res.value, _STATUS[st]


def partition(N: int, world: int, rank: int):
    """Host-only slice partition of the multi-rank driver: (first, count)."""
    f, c = ctypes.c_int(), ctypes.c_int()
    _check(lib().mfode_partition(N, world, rank, ctypes.byref(f), ctypes.byref(c)))
    return f.value, c.value


def kernel_launches() -> int:
    return int(lib().mfode_kernel_launches())


def version() -> str:
    return lib().mfode_version().decode()


def rk4_flops_per_step(n: int, flow: int) -> float:
    """Algorithmic flops of one RK4 step: 4 stages x (2 GEMMs inverse | 1 GEMM sqrt) x 2n^3."""
    return (16.0 if flow == FLOW_INVERSE else 8.0) * float(n) ** 3   # exp: 4 stages x 1 GEMM
