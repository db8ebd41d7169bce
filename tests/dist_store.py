"""Sharded sample store over NCCL (DataStore, src/datastore.cpp:99-248).

Launched by tests/test_dist.py as
  torchrun --nproc-per-node P tests/dist_store.py <out.npz>
Every rank generates the same synthetic datasets, keeps only its make_partition
shard in HBM (hmtl_store_create_sharded) and fetches three steps of its epoch
plan (base and taskpar modes); remote samples arrive by NCCL send/recv.  Each
fetched batch is checked against the same plan rows bound from a replicated
store (hmtl_store_bind): the forward predictions must be bit-identical.  Rank 0
writes the per-rank verdicts and the number of remote samples exchanged.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

COUNTS = (30, 20, 20, 8, 6)
B_LOCAL = 4


def run(out):
    import paper_2506_21788_b200 as P
    from paper_2506_21788_b200 import data
    from paper_2506_21788_b200._lib import check, lib

    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    specs = data.default5_specs()
    parts = {k: data.generate_dataset(specs[k], 1234 + k, count=c) for k, c in enumerate(COUNTS)}
    counts = {k: c for k, c in enumerate(COUNTS)}
    pool = P.Samples.concat([parts[k] for k in range(5)])
    result = {}
    for mode in ("base", "taskpar"):
        # taskpar: dataset k served by the ranks of its head group (general placement)
        members = {k: sorted({k % world, (k + 1) % world}) if k in (0, 3) else [k % world] for k in range(5)}
        part = P.make_partition(counts, world, mode, members if mode == "taskpar" else None)
        owned = [k for k in range(5) if mode == "base" or rank in members[k]]
        shard = []
        for k in range(5):
            cnt, serving, ranges = part[k]
            if rank in serving:
                lo, hi = ranges[serving.index(rank)]
                shard.append(parts[k].take(range(lo, hi)))
        shard = P.Samples.concat(shard)
        hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
        m = P.ModelT(hp, 7, owned, caps=P.Caps(64, 4096, 1 << 20), device=local)
        uid = P.comm_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, 0)
        m.comm_init(bytes(t.tolist()), world, rank)
        st = P.SampleStore.sharded(m, shard, part)
        full = P.SampleStore(pool, device=local)
        plans = [P.epoch_plan(mode, counts, world, 99, B_LOCAL, r, members if mode == "taskpar" else None)
                 for r in range(world)]
        ok, remote = True, 0
        for s in range(3):
            ds = np.stack([p[1][s * B_LOCAL:(s + 1) * B_LOCAL] for p in plans])
            ix = np.stack([p[2][s * B_LOCAL:(s + 1) * B_LOCAL] for p in plans])
            for d, i in zip(ds[rank], ix[rank]):
                cnt, serving, ranges = part[int(d)]
                owner = next(r for r, (lo, hi) in zip(serving, ranges) if lo <= i < hi)
                remote += owner != rank
            st.fetch(m, ds, ix)
            check(lib().hmtl_build_batch(m.ctx, None))
            a = m.forward(None)
            full.bind(m, ds[rank], ix[rank])
            check(lib().hmtl_build_batch(m.ctx, None))
            b = m.forward(None)
            ok &= bool(np.array_equal(a.energy_per_atom, b.energy_per_atom) and np.array_equal(a.forces, b.forces))
        result[f"{mode}_ok"] = np.array(ok)
        result[f"{mode}_remote"] = np.array(remote)
        st.close(), full.close(), m.close()
    objs = [None] * world
    dist.all_gather_object(objs, result)
    if rank == 0:
        np.savez(out, **{f"r{r}_{k}": v for r, d in enumerate(objs) for k, v in d.items()})


if __name__ == "__main__":
    dist.init_process_group("gloo")
    try:
        run(sys.argv[1])
    finally:
        dist.destroy_process_group()
