"""CTA-pair (cta_group::2) accumulator layout probe: which TMEM lane of which CTA
holds accumulator row r (D[r][n] = r + 1 + 1024 (n + 1))."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_21788_b200._lib import check, lib
for M, N in ((128, 64), (128, 128), (256, 64), (256, 128)):
    out = np.zeros((4, 128, 32), np.float32)
    check(lib().hmtl_selftest_pair_layout(M, N, out.ctypes.data_as(C.POINTER(C.c_float))))
    print(f"M={M} N={N}")
    for cta in range(2):
        rows = []
        for lane in range(128):
            v = out[cta, lane]
            r = int(round(v[0] - 1024)) - 1 if v[0] else -1
            ok = v[0] == 0 or all(abs(v[c] - (r + 1 + 1024 * (c + 1))) < 0.5 for c in range(32))
            rows.append((r, ok))
        print(f"  cta {cta}: lane->row", [r for r, _ in rows], "consistent cols" if all(o for _, o in rows) else "COLUMN MISMATCH")
        if not all(o for _, o in rows):
            for lane in (0, 1, 16, 32, 64):
                print("    lane", lane, out[cta, lane, :8].tolist())

# .16x256b shape: thread t, value 4j + {0,1,2,3} = (lane t/4 | t/4 + 8, column 8j + 2(t%4) + {0,1})
M, N = 256, 64
out = np.zeros((4, 128, 32), np.float32)
check(lib().hmtl_selftest_pair_layout(M, N, out.ctypes.data_as(C.POINTER(C.c_float))))
acc = out[:2]
w = out[2:].reshape(-1)
bad = 0
for cta in range(2):
    for warp in range(4):
        for h in range(2):
            for t in range(32):
                for j in range(4):
                    for e in range(4):
                        lane = 32 * warp + 16 * h + t // 4 + (8 if e >= 2 else 0)
                        col = 8 * j + 2 * (t % 4) + (e & 1)
                        got = w[((cta * 4 + warp) * 2 + h) * 512 + t * 16 + 4 * j + e]
                        bad += got != acc[cta, lane, col]
print("16x256b layout as assumed" if bad == 0 else f"16x256b layout MISMATCH ({bad} values)")
