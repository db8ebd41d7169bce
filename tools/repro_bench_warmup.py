"""Repro harness: bench.py's setup + warmup steps, reporting the failing step (if any)."""
import ctypes as C, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import bench
import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import check, lib

heads, batches, share = bench.rank_batches(0, 1)
caps = P.Caps.for_samples(batches[0])
for b in batches[1:]:
    caps = caps.union(P.Caps.for_samples(b))
model = P.ModelT(P.ModelHyper(**bench.HYPER), 7, heads, caps=caps, device=0)
slots = []
for b in batches:
    sl = C.c_int()
    check(lib().hmtl_pool_add(model.ctx, C.byref(b.as_c()), C.byref(sl)))
    slots.append(sl.value)
cfg = P.TrainConfig(use_graph=os.environ.get("EAGER", "0") != "1")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sync = os.environ.get("SYNC", "1") == "1"
for i in range(n):
    try:
        check(lib().hmtl_pool_bind(model.ctx, slots[i % len(slots)], None))
        check(lib().hmtl_train_step(model.ctx, C.byref(cfg.c()), None))
        if sync:
            L = C.c_float()
            check(lib().hmtl_read_loss(model.ctx, C.byref(L)))
    except Exception as e:
        print(f"FAIL at step {i}: {e}", flush=True)
        sys.exit(1)
print("ok", n, flush=True)
