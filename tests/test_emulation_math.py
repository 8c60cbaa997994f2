"""CPU checks of the arithmetic behind f3(ii), the int8-tensor-core FP64 emulation
(paper_1505_07959_b200/csrc/ozaki.cu), written independently in exact Python
integers: the moduli are pairwise coprime, the operand width a leaves the CRT margin
k 2^(2a) < M/4, the bias-split residue formula equals x mod m, the pair CRT and the group CRT
reconstruct the exact integer product, and the quotient estimate from 0.32 fixed-point weights
is exact within the margin.  No GPU needed."""
import math
import random

import numpy as np
import pytest

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def abits(nmod, k):
    l2 = sum(math.log2(m) for m in MODULI[:nmod])
    kb = math.ceil(math.log2(k)) if k > 1 else 0
    return min(60, math.floor((l2 - 2 - kb) / 2 - 1e-9))


def test_moduli_pairwise_coprime_and_fit_uint8():
    for i, a in enumerate(MODULI):
        assert 2 <= a <= 256
        for b in MODULI[i + 1:]:
            assert math.gcd(a, b) == 1


@pytest.mark.parametrize("nmod", [8, 12, 14, 16])
@pytest.mark.parametrize("k", [1, 2, 100, 4096, 32768])
def test_crt_margin(nmod, k):
    a = abits(nmod, k)
    M = math.prod(MODULI[:nmod])
    assert a >= 8 or nmod == 8
    if a >= 8:
        assert k * (2 ** a) ** 2 < M // 4          # |C'| < M/4: the signed CRT representative is exact
        assert k * 255 * 255 < 2 ** 31             # int32 accumulation of uint8 residue products


def test_bias_split_residue():
    rng = random.Random(1)
    for m in MODULI:
        c1, c2 = (1 << 20) % m, (1 << 40) % m
        nb = m - (1 << 61) % m
        for _ in range(500):
            x = rng.randint(-(1 << 60), 1 << 60)
            xb = x + (1 << 61)
            u0, u1, u2 = xb & 0xFFFFF, (xb >> 20) & 0xFFFFF, xb >> 40
            s = u2 * c2 + u1 * c1 + u0 + nb
            assert s < 2 ** 31
            assert s % m == x % m


def _pair_weights(nmod):
    M = math.prod(MODULI[:nmod])
    groups = [MODULI[i] * (MODULI[i + 1] if i + 1 < nmod else 1) for i in range(0, nmod, 2)]
    W = [(M // P) * pow(M // P, -1, P) for P in groups]
    return M, groups, W


@pytest.mark.parametrize("nmod", [12, 15, 16])
def test_exact_product_reconstruction(nmod):
    """Random integer matrices of the encoded width: residue products per modulus, pair CRT (as the
    GEMM epilogue), group CRT with 32-bit limbs mod 2^128 and the fixed-point quotient (as the
    decode) reproduce the exact integer product."""
    rng = np.random.default_rng(nmod)
    k = 64
    a = abits(nmod, k)
    M, groups, W = _pair_weights(nmod)
    A = [[int(v) for v in row] for row in rng.integers(-(2 ** a), 2 ** a, (3, k), dtype=np.int64)]
    B = [[int(v) for v in row] for row in rng.integers(-(2 ** a), 2 ** a, (k, 3), dtype=np.int64)]
    pwq = [math.floor(w * 2 ** 32 / M) for w in W]
    for i in range(3):
        for j in range(3):
            exact = sum(A[i][t] * B[t][j] for t in range(k))
            res = []
            for m in MODULI[:nmod]:
                acc = sum((A[i][t] % m) * (B[t][j] % m) for t in range(k))   # uint8 x uint8 -> int32
                assert acc < 2 ** 31
                res.append(acc % m)
            rho = []
            for g in range(0, nmod, 2):                                         # epilogue pair CRT
                if g + 1 < nmod:
                    ma, mb = MODULI[g], MODULI[g + 1]
                    ra, rb = res[g], res[g + 1]
                    rho.append(ra + ma * (((rb + 2 * mb - ra) % mb) * pow(ma, -1, mb) % mb))
                else:
                    rho.append(res[g])
            S = sum(r * w for r, w in zip(rho, W)) % 2 ** 128                    # limbs, wrapping
            q = (sum(r * p for r, p in zip(rho, pwq)) + 2 ** 31) >> 32           # fixed-point quotient
            c = (S - q * M) % 2 ** 128
            if c >= 2 ** 127:
                c -= 2 ** 128
            assert c == exact
