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
