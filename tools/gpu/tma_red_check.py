# TMA reduce GEMM vs numpy (debug: variant bits select descriptor hypotheses)
import ctypes as C
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_21788_b200._lib import lib
rng = np.random.default_rng(0)
for rows, K, N in ((256, 128, 128), (1000, 128, 128), (77, 128, 64), (3509, 128, 128), (999, 64, 96), (333, 96, 32)):
    X = rng.standard_normal((rows, K)).astype(np.float32)
    Y = rng.standard_normal((rows, N)).astype(np.float32)
    ref = X.astype(np.float64).T @ Y.astype(np.float64)
    for v in (0, 1):
        Cm = np.zeros((K, N), np.float32)
        fp = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))
        rc = lib().hmtl_selftest_gemm(1, v, rows, K, N, fp(X), fp(Y), fp(Cm))
        err = np.abs(Cm - ref).max() / np.abs(ref).max()
        print(rows, K, N, "variant", v, "rc", rc, "maxrel %.3e" % err, lib().hmtl_last_error().decode() if rc else "", flush=True)
