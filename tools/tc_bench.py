"""Time the tcgen05 engines on plain matrices (and ablations): achieved TFLOP/s."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21788_b200._lib import check, lib
cases = [(0, 56704, 128, 128), (0, 4 * 56704, 128, 128), (0, 56704, 128, 256), (0, 3509, 256, 128),
         (1, 56704, 128, 128), (1, 4 * 56704, 128, 128), (1, 3509, 256, 128)]
for dbg in (0, 1, 2, 3):
    for mode, rows, K, N in cases:
        if dbg and mode == 1: continue
        ms = C.c_float()
        check(lib().hmtl_selftest_time(mode | (dbg << 4), rows, K, N, 20, C.byref(ms)))
        fl = 2.0 * rows * K * N
        by = 4.0 * (rows * K + rows * N)
        print(f"dbg {dbg} mode {mode} rows {rows} K {K} N {N}: {ms.value*1e3:.1f} us  {fl/ms.value/1e9:.1f} TF/s (x3 {3*fl/ms.value/1e9:.1f})  {by/ms.value/1e6:.0f} GB/s")
