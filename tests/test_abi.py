"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mfode.h declares,
and the host-only logic (partition, argument validation before any CUDA call) behaves."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1505_07959_b200 as mf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mfode.h")).read()
    return sorted(set(re.findall(r"MFODE_API\s+[\w\s\*]*?\b(mfode_\w+)\s*\(", src)))


def test_library_builds_and_loads():
    from paper_1505_07959_b200 import build
    build.build(verbose=False)
    L = mf.lib()
    assert "sm_100a" in mf.version()


def test_exports_every_declared_symbol():
    L = mf.lib()
    names = _declared()
    assert len(names) >= 19
    for name in names:
        assert hasattr(L, name), name
    assert sorted(names) == sorted(mf.EXPORTED)


def test_partition_blocks():
    for N in (1, 7, 16, 64):
        for world in range(1, min(N, 8) + 1):
            covered = []
            sizes = []
            for r in range(world):
                f, c = mf.partition(N, world, r)
                covered.extend(range(f, f + c))
                sizes.append(c)
            assert covered == list(range(N))
            assert max(sizes) - min(sizes) <= 1
            assert sizes == sorted(sizes, reverse=True)


def test_partition_invalid():
    with pytest.raises(mf.MfodeError):
        mf.partition(4, 5, 0) if False else mf.partition(0, 1, 0)
    with pytest.raises(mf.MfodeError):
        mf.partition(8, 2, 2)


def test_create_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call, so it is checkable on a CPU box."""
    L = mf.lib()
    h = ctypes.c_void_p()
    A = np.eye(4)
    assert L.mfode_create(ctypes.byref(h), None, 4, 0, 1.0, 4, 1, 1, None) == mf.EINVAL
    assert L.mfode_create(ctypes.byref(h), A.ctypes.data, 0, 0, 1.0, 4, 1, 1, None) == mf.EINVAL
    assert L.mfode_create(ctypes.byref(h), A.ctypes.data, 4, 9, 1.0, 4, 1, 1, None) == mf.EINVAL
    assert L.mfode_create(ctypes.byref(h), A.ctypes.data, 4, 0, -1.0, 4, 1, 1, None) == mf.EINVAL
    assert L.mfode_create(ctypes.byref(h), A.ctypes.data, 4, 0, 1.0, 0, 1, 1, None) == mf.EINVAL
    assert L.mfode_create(ctypes.byref(h), A.ctypes.data, 4, 0, 1.0, 4, 0, 1, None) == mf.EINVAL
    d = mf.Dist(0, 9, 0, None)
    assert L.mfode_create(ctypes.byref(h), A.ctypes.data, 4, 0, 1.0, 4, 1, 1, ctypes.byref(d)) == mf.EINVAL
    assert b"world" in L.mfode_last_global_error()
    assert L.mfode_parareal_solve(None, 1, 0.0, 0, None) == mf.EINVAL
    assert L.mfode_dgemm(None, None, None, None, 4, 4, 1.0, 0.0, 0, None) == mf.EINVAL
    # f3(ii) emulated GEMM: NULL operands, moduli count and size limits are checked before any CUDA call
    x = ctypes.c_void_p(1)
    assert L.mfode_dgemm_emulated(None, None, None, None, 4, 4, 1.0, 0.0, 16, None) == mf.EINVAL
    assert L.mfode_dgemm_emulated(x, x, None, x, 4, 4, 1.0, 0.0, 1, None) == mf.EINVAL
    assert L.mfode_dgemm_emulated(x, x, None, x, 4, 4, 1.0, 0.0, 17, None) == mf.EINVAL
    assert L.mfode_dgemm_emulated(x, x, None, x, 40000, 40000, 1.0, 0.0, 16, None) == mf.EINVAL
    assert L.mfode_dgemm_emulated(x, x, None, x, 4, 3, 1.0, 0.0, 16, None) == mf.EINVAL


def test_no_oracle_import_in_product_path():
    """The product path never touches oracle/ (and the oracle never touches the product path)."""
    pkg = os.path.join(ROOT, "paper_1505_07959_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                code = re.sub(r'"""[\s\S]*?"""|#.*|//.*', "", txt)   # drop docstrings / comments
                assert "import oracle" not in code and "from oracle" not in code, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            code = re.sub(r'"""[\s\S]*?"""|#.*', "", open(os.path.join(ROOT, "oracle", f)).read())
            assert "paper_1505_07959_b200" not in code and "mfode" not in code, f


def test_affine_and_stop_rule_argument_checks_without_gpu():
    L = mf.lib()
    assert L.mfode_set_affine(None, None, None) == mf.EINVAL
    assert L.mfode_modified_parareal_solve(None, 1, 0.0, 0, 0, None) == mf.EINVAL
    assert mf.FLOW_AFFINE == 4 and mf.STOP_MAX_SLICE == 3
    src = open(os.path.join(ROOT, "include", "mfode.h")).read()
    assert "MFODE_FLOW_AFFINE = 4" in src and "MFODE_STOP_MAX_SLICE = 3" in src


def test_kernel_wrappers_validate_operands_before_the_abi():
    """a transposed view, a wrong dtype, a non-square or a host tensor must be
    rejected by the binding -- the C ABI takes one leading dimension for every operand and TMA would
    otherwise read past a smaller allocation."""
    torch = pytest.importorskip("torch")
    A = torch.zeros((8, 8), dtype=torch.float64)
    with pytest.raises(ValueError, match="CUDA"):
        mf.dgemm(A, A)
    with pytest.raises(ValueError, match="CUDA"):
        mf.frobenius(A)
    with pytest.raises(ValueError):
        mf.rk_stage(A, A, A, A, None, 1, 0.1)
    with pytest.raises(ValueError, match="beta"):
        mf.dgemm_emulated(A, A, beta=1.0)


def test_host_buffers_validated_before_the_abi():
    """Host arrays that the library reads or writes through raw pointers are shape-checked in the
    binding (a smaller buffer would be overrun): result / slice outputs (2n x n for the trig flow),
    set_matrix / set_affine / accel_inverse inputs."""
    with pytest.raises(ValueError):
        mf._host_out(np.empty((3, 4)), (4, 4), "out")
    with pytest.raises(ValueError):
        mf._host_out(np.empty((4, 4), dtype=np.float32), (4, 4), "out")
    with pytest.raises(ValueError):
        mf._host_out(np.empty((8, 4))[::2], (4, 4), "out")          # not contiguous
    assert mf._host_out(None, (8, 4), "out").shape == (8, 4)
    with pytest.raises(ValueError):
        mf._host_square(np.eye(3), 4, "A")
    with pytest.raises(ValueError):
        mf.accel_inverse(np.eye(4), np.eye(3), 0.1, 2)             # E0 of the wrong size, no GPU call made
