"""Ingress probe, single SM vs both SMs of a TPC (2-CTA clusters)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21788_b200._lib import check, lib
f = lib().hmtl_selftest_ingress
def run(mode, grid, stride, total, chunk, depth):
    v = C.c_float()
    check(f(mode, grid, stride, total, chunk, depth, C.byref(v)))
    return v.value
for grid in (2, 56, 148):
    for cl in (0, 10):
        print(f"grid {grid:3d} {'cluster2' if cl else 'single  '}: bulk32K d4 {run(cl + 0, grid, 1 << 20, 262144, 32768, 4):6.1f}"
              f"  bulk16K d4 {run(cl + 0, grid, 1 << 20, 262144, 16384, 4):6.1f}  cp.async128K {run(cl + 2, grid, 1 << 20, 131072, 16, 1):6.1f}"
              f"  tma16K d4 {run(cl + 3, grid, 0, 131072, 16384, 4):6.1f}")
