"""Shared-memory ingress probe (hmtl_selftest_ingress): bytes per SM clock moved into
shared memory by bulk copies, from global (distinct or shared source) and from a
2-CTA cluster peer.  Engine design input for the node-row chain."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21788_b200._lib import check, lib
f = lib().hmtl_selftest_ingress
def run(mode, grid, stride, total, chunk, depth):
    v = C.c_float()
    check(f(mode, grid, stride, total, chunk, depth, C.byref(v)))
    return v.value
print("mode0 global->smem: grid, stride, chunk KB, depth -> B/clk per SM")
for grid in (1, 56, 148):
    for stride in (1 << 20,):
        for chunk, depth in ((16384, 4), (32768, 4), (65536, 2), (8192, 8)):
            print(f"  grid {grid:3d} {'shared ' if stride == 0 else 'distinct'} chunk {chunk // 1024:2d} KB depth {depth:2d}: "
                  f"{run(0, grid, stride, 262144, chunk, depth):6.1f}")
print("mode2 cp.async, 256 threads, all in flight; mode3 tensor TMA 16 KB boxes")
for grid in (1, 56, 148):
    for total in (65536, 131072):
        print(f"  grid {grid:3d} total {total // 1024} KB: cp.async {run(2, grid, 1 << 20, total, 16, 1):6.1f}  "
              + "  ".join(f"tma d{d} {run(3, grid, 0, total, 16384, d):6.1f}" for d in (2, 4, 8)))
print("mode1 peer smem push (both ways): grid, total KB, chunk KB -> B/clk per SM")
for grid in (2, 56, 148):
    for total, chunk in ((65536, 4096), (65536, 8192), (65536, 16384), (32768, 4096)):
        print(f"  grid {grid:3d} total {total // 1024} KB chunk {chunk // 1024} KB: {run(1, grid, 0, total, chunk, 16):6.1f}")
