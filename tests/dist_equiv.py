"""Distributed equivalence of the MTL-par step (acceptance 2).

Launched by tests/test_gpu_multi.py as
  torchrun --nproc-per-node P tests/dist_equiv.py <out.npz> [--backend nccl|oracle]
Each rank owns the heads hmtl_head_placement gives it, trains 3 steps on its
own batch through the B200 path with NCCL head-group + global allreduce, and
rank 0 gathers every rank's final parameters.  With --backend oracle (CPU,
gloo) the same plan runs on the FP64 oracle with torch.distributed(gloo)
allreduces -- the host-side logic test that runs without GPUs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

HEADS = 5
WEIGHTS = (1, 1, 1, 2, 3)
STEPS = 3


def rank_batch(rank, world, step, counts=(6, 4, 4, 2, 1)):
    from paper_2506_21788_b200 import data
    from paper_2506_21788_b200.model import Samples

    share = data.head_placement(world, WEIGHTS)
    specs = data.default5_specs()
    parts = []
    for k in range(HEADS):
        if share[rank, k] <= 0:
            continue
        members = [r for r in range(world) if share[r, k] > 0]
        per = int(round(world * counts[k] * share[rank, k]))
        pool = data.generate_dataset(specs[k], 1234 + k + 100 * step, count=per * len(members))
        slot = members.index(rank)
        parts.append(pool.take(range(slot * per, (slot + 1) * per)))
    return Samples.concat(parts), [k for k in range(HEADS) if share[rank, k] > 0], share


def run_gpu(out):
    import ctypes as C

    import paper_2506_21788_b200 as P
    from paper_2506_21788_b200._lib import check, lib

    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    batches = []
    for s in range(STEPS):
        b, heads, share = rank_batch(rank, world, s)
        batches.append(b)
    caps = P.Caps.for_samples(batches[0])
    for b in batches[1:]:
        caps = caps.union(P.Caps.for_samples(b))
    hp = P.ModelHyper(20, 2, 32, 32, 3, HEADS, 5.0)
    m = P.ModelT(hp, 7, heads, caps=caps, device=local)
    idb = (C.c_uint8 * 128)()
    if rank == 0:
        check(lib().hmtl_comm_unique_id(idb))
    t = torch.tensor(list(bytes(idb)), dtype=torch.uint8)
    dist.broadcast(t, 0)
    check(lib().hmtl_comm_init(m.ctx, (C.c_uint8 * 128)(*t.tolist()), world, rank))
    cfg = P.TrainConfig(use_graph=True)
    losses = [m.train_step(b, cfg) for b in batches]
    result = {"shared": m.shared_block(), **{f"head{k}": m.head_block(k) for k in heads},
              "losses": np.array(losses)}
    gather(result, out)


def oracle_step_grads(o, oh, sh, hd, b):
    import oracle as O

    ob = O.batch_from_samples(dict(n_atoms=b.n_atoms, species=b.species, pos=b.positions, forces=b.forces,
                                   energy=b.energy, dsid=b.dataset_id), 5.0, o.build_edges)
    E, F, c = o.forward(oh, sh, hd, ob)
    L, dE, dF = o.loss(ob, E, F)
    gs, gh = o.backward(oh, sh, hd, ob, c, dE, dF)
    return L, gs, gh


def emulate(world):
    """Single-process emulation of `world` MTL-par ranks on the FP64 oracle: every
    rank's gradients computed in turn, shared grads averaged over all ranks, head k's
    over the ranks that own it (hmtl/mesh.hpp:322-334 group means), AdamW per rank."""
    import oracle as O

    o = O.Oracle()
    oh = O.Hyper(20, 2, 32, 32, 3, HEADS, 5.0)
    state = []
    for r in range(world):
        _, heads, share = rank_batch(r, world, 0)
        sh = o.init_block(oh, 7, -1)
        hd = {k: o.init_block(oh, 7, k) for k in heads}
        st = {"s": (np.zeros_like(sh), np.zeros_like(sh)),
              **{k: (np.zeros_like(hd[k]), np.zeros_like(hd[k])) for k in heads}}
        state.append((sh, hd, st))
    losses = [[] for _ in range(world)]
    for s in range(STEPS):
        res = []
        for r in range(world):
            b, _, _ = rank_batch(r, world, s)
            L, gs, gh = oracle_step_grads(o, oh, state[r][0], state[r][1], b)
            losses[r].append(L)
            res.append((gs, gh))
        gmean = sum(g for g, _ in res) / world
        for r in range(world):
            sh, hd, st = state[r]
            o.adamw(sh, gmean.copy(), *st["s"], s + 1)
            for k in hd:
                owners = [q for q in range(world) if k in res[q][1]]
                gk = sum(res[q][1][k] for q in owners) / len(owners)
                o.adamw(hd[k], np.ascontiguousarray(gk), *st[k], s + 1)
    out = {}
    for r in range(world):
        out[f"r{r}_shared"] = state[r][0]
        for k, v in state[r][1].items():
            out[f"r{r}_head{k}"] = v
        out[f"r{r}_losses"] = np.array(losses[r])
    return out


def run_oracle(out):
    import oracle as O

    rank, world = dist.get_rank(), dist.get_world_size()
    o = O.Oracle()
    oh = O.Hyper(20, 2, 32, 32, 3, HEADS, 5.0)
    b0, heads, share = rank_batch(rank, world, 0)
    sh = o.init_block(oh, 7, -1)
    hd = {k: o.init_block(oh, 7, k) for k in heads}
    st = {"s": (np.zeros_like(sh), np.zeros_like(sh)), **{k: (np.zeros_like(hd[k]), np.zeros_like(hd[k])) for k in heads}}
    # head sub-groups (hmtl/mesh.hpp:52-58 generalised): ranks sharing head k
    groups = {k: dist.new_group([r for r in range(world) if share[r, k] > 0]) for k in range(HEADS)}
    losses, seen = [], set()
    for s in range(STEPS):
        b, _, _ = rank_batch(rank, world, s)
        seen |= set(int(x) for x in b.dataset_id)
        L, gs, gh = oracle_step_grads(o, oh, sh, hd, b)
        losses.append(L)
        for k in heads:  # head grads: mean within the head's sub-group
            t = torch.from_numpy(gh[k])
            dist.all_reduce(t, group=groups[k])
            gh[k] = t.numpy() / (share[:, k] > 0).sum()
        t = torch.from_numpy(gs)  # shared grads: mean over all ranks
        dist.all_reduce(t)
        gs = t.numpy() / world
        o.adamw(sh, gs, *st["s"], s + 1)
        for k in heads:
            o.adamw(hd[k], np.ascontiguousarray(gh[k]), *st[k], s + 1)
    gather({"shared": sh, **{f"head{k}": hd[k] for k in heads}, "losses": np.array(losses),
            "dsids": np.array(sorted(seen))}, out)


def gather(result, out):
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, result)
    if dist.get_rank() == 0:
        merged = {}
        for r, d in enumerate(objs):
            for k, v in d.items():
                merged[f"r{r}_{k}"] = v
        np.savez(out, **merged)


if __name__ == "__main__":
    out = sys.argv[1]
    backend = sys.argv[sys.argv.index("--backend") + 1] if "--backend" in sys.argv else "nccl"
    dist.init_process_group("gloo")
    try:
        run_gpu(out) if backend == "nccl" else run_oracle(out)
    finally:
        dist.destroy_process_group()
