"""Direct tests of the tcgen05 GEMM engines (3xTF32) on plain matrices."""
import ctypes as C

import numpy as np
import pytest

import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import check, lib

pytestmark = pytest.mark.gpu


def fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def run(mode, rows, K, N, variant=0, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((rows, K)).astype(np.float32)
    Y = rng.standard_normal((K, N) if mode == 0 else (rows, N)).astype(np.float32)
    out = np.zeros((rows, N) if mode == 0 else (K, N), np.float32)
    check(lib().hmtl_selftest_gemm(mode, variant, rows, K, N, fp(X), fp(Y), fp(out)))
    ref = X.astype(np.float64) @ Y if mode == 0 else X.astype(np.float64).T @ Y
    return np.linalg.norm(out - ref) / np.linalg.norm(ref)


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    if lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("rows,K,N", [(300, 128, 128), (1000, 256, 128), (257, 128, 256), (64, 32, 32)])
def test_row_gemm_3xtf32(rows, K, N):
    assert run(0, rows, K, N) < 1e-5  # 3xTF32 + TMEM accumulation ~1e-6


@pytest.mark.parametrize("rows,M,N", [(1000, 128, 128), (333, 256, 128), (96, 32, 32), (500, 128, 256)])
def test_reduce_gemm_3xtf32(rows, M, N):
    assert run(1, rows, M, N) < 1e-5


@pytest.mark.parametrize("rows,M,N", [(1000, 128, 128), (77, 128, 64), (3509, 128, 128), (999, 64, 96), (333, 96, 32)])
def test_reduce_gemm_tma_operands(rows, M, N):
    """TMA operand path (tc_red_tma_kernel: MN-major 128B_BASE32B tiles, in-place hi/lo
    split, partial last chunk zeroed) against FP64 and bit-equal to the register path."""
    assert run(1, rows, M, N, variant=1) < 1e-5
    rng = np.random.default_rng(3)
    X = rng.standard_normal((rows, M)).astype(np.float32)
    Y = rng.standard_normal((rows, N)).astype(np.float32)
    a, b = np.zeros((M, N), np.float32), np.zeros((M, N), np.float32)
    check(lib().hmtl_selftest_gemm(1, 0, rows, M, N, fp(X), fp(Y), fp(a)))
    check(lib().hmtl_selftest_gemm(1, 1, rows, M, N, fp(X), fp(Y), fp(b)))
    assert np.array_equal(a, b)
