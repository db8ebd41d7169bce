"""Per-rank step time of the bench workload at world size W, emulated on one GPU
(no NCCL): each rank's batch and heads from bench.rank_batches.
python tools/rank_cost.py [W ...]"""
import ctypes as C, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch
import bench
import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import check, lib

for W in [int(x) for x in sys.argv[1:]] or [8]:
    for r in range(W):
        heads, batches, share = bench.rank_batches(r, W)
        caps = P.Caps.for_samples(batches[0])
        for b in batches[1:]:
            caps = caps.union(P.Caps.for_samples(b))
        m = P.ModelT(P.ModelHyper(**bench.HYPER), 7, heads, caps=caps)
        slots = []
        for b in batches:
            sl = C.c_int()
            check(lib().hmtl_pool_add(m.ctx, C.byref(b.as_c()), C.byref(sl)))
            slots.append(sl.value)
        cfg = P.TrainConfig(use_graph=True)
        def step(i):
            check(lib().hmtl_pool_bind(m.ctx, slots[i % len(slots)], None))
            check(lib().hmtl_train_step(m.ctx, C.byref(cfg.c()), None))
        for i in range(5):
            step(i)
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ext = torch.cuda.ExternalStream(lib().hmtl_ctx_stream(m.ctx))
        a.record(ext)
        for i in range(20):
            step(i)
        b_.record(ext)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b_) / 20
        b0 = batches[0]
        E = C.c_int()
        check(lib().hmtl_batch_edges(m.ctx, C.byref(E), None, None, None))
        print(f"W={W} rank {r} heads {heads}: G={b0.G} N={b0.N} E={E.value}  {ms:.4f} ms/step", flush=True)
        m.close()
