"""Phase timestamps of the fused node-chain kernel (last launch of an eager step).
HMTL_CHAIN_STAMPS=1 python tools/chain_stamps.py"""
import ctypes as C, os, sys
os.environ.setdefault("HMTL_CHAIN_STAMPS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import bench
import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import check, lib
heads, batches, _ = bench.rank_batches(0, 1)
caps = P.Caps.for_samples(batches[0])
m = P.ModelT(P.ModelHyper(**bench.HYPER), 7, heads, caps=caps)
cfg = P.TrainConfig(use_graph=os.environ.get("STAMPS_GRAPH") == "1")
for i in range(3):
    m.train_step(batches[0], cfg)
NC = 256
buf = (C.c_longlong * (NC * 32))()
check(lib().hmtl_debug_chain_stamps(m.ctx, buf, NC * 32))
names = {0: "setup", 1: "prod_done", 2: "mma0_start", 3: "mma0_issued", 4: "mma1_start", 5: "mma1_issued",
         6: "mma2_start", 7: "mma2_issued", 8: "epi0_start", 9: "epi0_end", 10: "epi1_start", 11: "epi1_end",
         12: "epi2_start", 13: "epi2_end", 26: "a_conv0", 27: "a_conv3", 28: "mma_a0", 29: "mma_a7", 31: "exit"}
for g in range(3):  # first slab of epilogue warp 0: TMEM read, outputs formed, X chunk published
    names.update({14 + 4 * g: f"e{g}_tmem", 15 + 4 * g: f"e{g}_formed", 16 + 4 * g: f"e{g}_published"})
for cta in [int(x) for x in os.environ.get("CTAS", "0,13,27").split(",")]:
    row = buf[cta * 32:(cta + 1) * 32]
    print(f"CTA {cta}: " + "  ".join(f"{names.get(i, 'b%d' % (i - 14))}={row[i] / 1.9e3:.2f}us" for i in range(32) if row[i]))
ctas = [c for c in range(NC) if buf[c * 32 + 31]]
print(f"{len(ctas)} CTAs; per-stamp median / max over CTAs (us):")
import statistics
for i in range(32):
    v = [buf[c * 32 + i] / 1.9e3 for c in ctas if buf[c * 32 + i]]
    if v:
        print(f"  {names.get(i, 'b%d' % (i - 14)):12s} med {statistics.median(v):7.2f}  max {max(v):7.2f}")
