"""Tensor-pipe issue-rate probe: SM clocks per M=128 x N MMA (one K step) for
tf32 / bf16, operands in smem (SS) or A in TMEM (TS).  Floor: 128*N/256 clk."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21788_b200._lib import check, lib
names = {0: "tf32 SS", 1: "tf32 TS", 2: "bf16 SS", 3: "bf16 TS", 4: "tf32 SS warp-issue"}
for v in (0, 4):
    for N in (64, 128, 256):
        c = C.c_float()
        check(lib().hmtl_selftest_mma_rate(v, N, 4096, C.byref(c)))
        print(f"{names[v]} N={N:3d}: {c.value:7.1f} clk/MMA (floor {128 * N / 256:.0f})")
