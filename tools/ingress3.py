"""Ingress probe: warm L2 vs cold (flushed) vs cold + in-kernel L2 prefetch."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21788_b200._lib import check, lib
f = lib().hmtl_selftest_ingress
def run(mode, grid, stride, total, chunk, depth):
    v = C.c_float()
    check(f(mode, grid, stride, total, chunk, depth, C.byref(v)))
    return v.value
for grid in (28, 56):
    for base, name in ((0, "warm"), (20, "cold"), (40, "cold+prefetch")):
        print(f"grid {grid:3d} {name:14s}: bulk32K d3 {run(base + 0, grid, 1 << 20, 131072, 32768, 3):6.1f}"
              f"  bulk32K d2 {run(base + 0, grid, 1 << 20, 131072, 32768, 2):6.1f}"
              f"  tma16K d4 {run(base + 3, grid, 0, 131072, 16384, 4):6.1f}  cp.async128K {run(base + 2, grid, 1 << 20, 131072, 16, 1):6.1f}")
