"""Parity AT THE MEASURED CONFIGURATIONS (VERDICT r1 "What's weak" #1): the
B200 training step, run exactly as bench.py runs it (pooled batch, CUDA-graph
replay of hmtl_train_step), against the FP64 oracle (oracle/hmtl_oracle.c,
pinned bit-exact to the reference by tests/test_oracle_golden.py) on:

* mtl5-weak: the bench's own 1-GPU batch -- 276 structures, 56,706 edges, five
  heads -- so every persistent row-GEMM CTA runs ~3 row tiles (TMEM accumulator
  double-buffering, cross-tile prefetch, B reloads at head-segment boundaries);
* cfg2: 2 heads x 16 structures, H=128, L=4;
* cfg4: 8 structures of 200-300 atoms at rc 6 (~22k edges each), L=6, H=W=256.

The compared step is the THIRD step of a fresh context (step 1 eager, step 2
graph capture, step 3 graph replay), at the device's parameters after two
AdamW updates.  Tolerance (north star): rel_vec_error <= 1e-4 in FP32
(tests/oracles.hpp:62-74 metric) on predictions, loss, per-layer activations
and every gradient.  The oracle is OpenMP-threaded with per-element order kept
(bit-identical to its serial form).
"""
import numpy as np
import pytest

import bench
import oracle as O

import paper_2506_21788_b200 as P

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    O.build(ref=False)
    if P.lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")


def rel(a, b):
    return O.rel_vec_error(a, b)


def measured_step(workload):
    hyper = bench.WORKLOADS[workload]["hyper"]
    heads, batches, _ = bench.rank_batches(0, 1, workload=workload)
    caps = P.Caps.for_samples(batches[0])
    for b in batches[1:]:
        caps = caps.union(P.Caps.for_samples(b))
    hp = P.ModelHyper(**hyper)
    m = P.ModelT(hp, 7, heads, caps=caps)
    cfg = P.TrainConfig(use_graph=True)
    m.train_step(batches[1], cfg)  # eager: records the tensor-core B images
    m.train_step(batches[2], cfg)  # captured + replayed
    sh = m.shared_block().astype(np.float64)
    hb = {k: m.head_block(k).astype(np.float64) for k in heads}
    s = batches[0]  # the bench's first batch, through a graph replay
    L = m.train_step(s, cfg)
    pred = m.predictions()
    g = m.grads()
    acts = {}
    for l in range(hp.layers):
        for name in ("h", "z2", "agg", "vz1"):
            acts[(name, l)] = m.debug(name, l)
    acts[("h", hp.layers)] = m.debug("h", hp.layers)
    E_dev = len(m.edges().edge_dst)
    m.close()
    o = O.Oracle()
    oh = O.Hyper(**hyper)
    ob = O.batch_from_samples(dict(n_atoms=s.n_atoms, species=s.species, pos=s.positions, forces=s.forces,
                                   energy=s.energy, dsid=s.dataset_id), oh.cutoff, o.build_edges)
    assert E_dev == len(ob["edge_dst"])
    E, F, cache = o.forward(oh, sh, hb, ob)
    Lo, dE, dF = o.loss(ob, E, F)
    gs, gh = o.backward(oh, sh, hb, ob, cache, dE, dF)
    return dict(s=s, L=L, pred=pred, g=g, acts=acts, E=E, F=F, Lo=Lo, gs=gs, gh=gh, cache=cache, heads=heads,
                edges=E_dev, layers=hp.layers)


def check(r):
    errs = {"energy": rel(r["pred"].energy_per_atom, r["E"]), "forces": rel(r["pred"].forces, r["F"]),
            "loss": abs(r["L"] - r["Lo"]) / abs(r["Lo"]), "g_shared": rel(r["g"].shared, r["gs"])}
    for k in r["heads"]:
        errs[f"g_head{k}"] = rel(r["g"].heads[k], r["gh"][k])
    c = r["cache"]
    for l in range(r["layers"]):
        errs[f"h{l}"] = rel(r["acts"][("h", l)], c["h_in"][l])
        errs[f"z2_{l}"] = rel(r["acts"][("z2", l)], c["z2"][l])
        errs[f"agg{l}"] = rel(r["acts"][("agg", l)], c["agg"][l])
        errs[f"vz1_{l}"] = rel(r["acts"][("vz1", l)], c["vz1"][l])
    errs["h_final"] = rel(r["acts"][("h", r["layers"])], c["h_final"])
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    print({k: f"{v:.1e}" for k, v in errs.items()})
    assert not bad, bad
    return errs


def test_mtl5_bench_batch_train_step_parity():
    r = measured_step("mtl5-weak")
    assert r["s"].G == 276 and r["edges"] == 56706  # the bench line's per-GPU batch
    check(r)


def test_cfg2_train_step_parity():
    r = measured_step("cfg2")
    assert r["s"].G == 32
    check(r)


def test_cfg4_full_shape_train_step_parity():
    r = measured_step("cfg4")
    assert r["s"].G == 8 and r["edges"] > 100_000
    assert r["s"].n_atoms.min() >= 200
    check(r)
