"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists):   python tests/golden/make_golden.py

It builds oracle/_ref/libhmtl_ref.so (oracle/Makefile compiles the reference
sources in place) and records, with fixed seeds (model seed 7 and friends,
generator seeds 1234+k as in SURVEY.md 8(c)):

  nbr_kat.npz        edge sets of adversarial neighbour-list cases and of each
                     default5 source (hmtl/graph.hpp:46-83)
  dataset5.npz       first samples of each default5_specs() source
                     (src/dataset.cpp:106-161, 213-239)
  model_tiny.npz     tiny_hyper-style model (L2 H8, 2 heads), mixed batch: params,
                     full forward cache, predictions, SPEC-loss upstreams, grads (FP64)
  model_med.npz      L3 H32 W32, 3 heads, 12 structures from three sources: FP64
                     predictions/grads/h_final plus the reference's own FP32
                     (ModelT<float>) outputs = the FP32 noise floor
  train_ref.npz      5 steps of the reference CPU trainer (ModelT<float> + SPEC loss/AdamW)
  hmtd_ds{0,3}.bin   HMTD sample files written by the reference (src/sample_io.cpp:104-120)
                     and hmtd.npz, their samples (`python make_golden.py hmtd`)
  ckpt_ref.hmtp      save_checkpoint (src/model_io.cpp:62-84) of FP32-representable
                     blocks (L2 H16 W16, 3 heads) + ckpt.npz (`python make_golden.py ckpt`)
  epoch_plan.npz     shuffle_epoch (src/datastore.cpp:47-97) per-rank plans, base and
                     taskpar, several meshes/seeds (`python make_golden.py epoch_plan`)

The fixtures are small (< 2 MB total) and are committed; tests never read
/root/reference at run time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402


def concat(parts):
    out = {}
    for k in ("n_atoms", "species", "pos", "forces", "energy", "dsid"):
        out[k] = np.concatenate([p[k] for p in parts])
    return out


def main():
    O.build(ref=True)
    ref = O.Ref()
    specs = [ref.default5_spec(i) for i in range(5)]

    # ---------------------------------------------------------------- nbr KATs
    kat = {}
    # atoms exactly at the cutoff: d^2 == 25 exactly -> inclusive (graph.hpp:71)
    cases = {
        "at_rc_x": [[0, 0, 0], [5, 0, 0]],
        "at_rc_345": [[0, 0, 0], [3, 4, 0]],
        "just_out": [[0, 0, 0], [5.000000000000001, 0, 0]],
        "single": [[1.0, 2.0, 3.0]],
        "two_close": [[0.3, -0.2, 0.1], [1.4, 0.8, -0.5]],
        "line": [[float(i) * 2.5, 0, 0] for i in range(7)],
    }
    ns, ps = [], []
    for name, p in cases.items():
        ns.append(len(p))
        ps.extend(p)
    n = np.array(ns, np.int32)
    pos = np.array(ps, np.float64)
    go, eo, dst, src = ref.build_edges(n, pos, 5.0)
    kat.update(kat_n=n, kat_pos=pos, kat_go=go, kat_eo=eo, kat_dst=dst, kat_src=src)
    for k, sp in enumerate(specs):
        s = ref.generate(sp, 1234 + k, count=12)
        go, eo, dst, src = ref.build_edges(s["n_atoms"], s["pos"], 5.0)
        kat.update({f"src{k}_n": s["n_atoms"], f"src{k}_pos": s["pos"], f"src{k}_eo": eo, f"src{k}_dst": dst,
                    f"src{k}_src": src})
    # cfg4-like large cell, rc 6
    sp4 = dict(specs[3])
    sp4.update(n_min=200, n_max=300, count=2)
    s = ref.generate(sp4, 99, count=2)
    go, eo, dst, src = ref.build_edges(s["n_atoms"], s["pos"], 6.0)
    kat.update(big_n=s["n_atoms"], big_pos=s["pos"], big_eo=eo, big_dst=dst, big_src=src)
    np.savez_compressed(os.path.join(HERE, "nbr_kat.npz"), **kat)

    # ---------------------------------------------------------------- dataset
    ds = {}
    for k, sp in enumerate(specs):
        s = ref.generate(sp, 1234 + k, count=6)
        for key, v in s.items():
            ds[f"src{k}_{key}"] = v
        ds[f"spec{k}_elements"] = np.array(sp["elements"], np.uint8)
        ds[f"spec{k}_params"] = np.array([sp["n_min"], sp["n_max"], sp["alpha"], sp["sigma"]], np.float64)
        ds[f"spec{k}_mu"] = np.array(sp["mu"], np.float64)
    # a cfg1 spec: elements {0,1,2,3}, n in [18,22], alpha 1, sigma .01
    c1 = dict(dataset_id=0, elements=[0, 1, 2, 3], n_min=18, n_max=22, alpha=1.0, sigma=0.01, mu=[0.0] * 20)
    s = ref.generate(c1, 1234, count=4)
    for key, v in s.items():
        ds[f"cfg1_{key}"] = v
    np.savez_compressed(os.path.join(HERE, "dataset5.npz"), **ds)

    # ---------------------------------------------------------------- model tiny
    def model_case(h, parts, owned, seed, with_cache, fname, extra_float=False):
        s = concat(parts)
        go, eo, dst, src = ref.build_edges(s["n_atoms"], s["pos"], h.cutoff)
        b = dict(s)
        b.update(graph_offset=go, edge_offset=eo, edge_dst=dst, edge_src=src)
        m = O.RefModel(ref, h, seed, owned, dbl=True)
        sh = m.block(-1)
        hd = {k: m.block(k) for k in owned}
        r0 = m.run(b, len(dst), cache=False)
        # SPEC loss upstreams computed with the FP64 oracle restatement of SPEC.md:383-391
        L, dE, dF = O.Oracle().loss(b, r0["energy"], r0["forces"])
        r = m.run(b, len(dst), dE, dF, cache=with_cache)
        out = dict(hyper=np.array([h.n_species, h.layers, h.hidden, h.head_width, h.head_depth, h.n_heads], np.int32),
                   cutoff=np.float64(h.cutoff), owned=np.array(owned, np.int32), seed=np.int64(seed),
                   shared=sh, energy=r["energy"], forces=r["forces"], loss=np.float64(L), dE=dE, dF=dF,
                   g_shared=r["g_shared"], **{f"head{k}": hd[k] for k in owned},
                   **{f"g_head{k}": r["g_heads"][k] for k in owned},
                   **{f"in_{k}": v for k, v in b.items()})
        if with_cache:
            out.update({f"cache_{k}": v for k, v in r["cache"].items()})
        else:
            rc = m.run(b, len(dst), cache=True)
            out["cache_h_final"] = rc["cache"]["h_final"]
            out["cache_s"] = rc["cache"]["s"]
        if extra_float:
            mf = O.RefModel(ref, h, seed, owned, dbl=False)
            rf = mf.run(b, len(dst), dE, dF, cache=True)
            out.update(f32_energy=rf["energy"], f32_forces=rf["forces"], f32_g_shared=rf["g_shared"],
                       f32_h_final=rf["cache"]["h_final"], **{f"f32_g_head{k}": rf["g_heads"][k] for k in owned})
        np.savez_compressed(os.path.join(HERE, fname), **out)

    tiny = O.Hyper(n_species=20, layers=2, hidden=8, head_width=8, head_depth=3, n_heads=2, cutoff=5.0)
    p0 = ref.generate(specs[0], 1234, count=3)
    p1 = ref.generate(dict(specs[1], dataset_id=1), 1235, count=3)
    model_case(tiny, [p0, p1], [0, 1], 7, True, "model_tiny.npz")

    med = O.Hyper(n_species=20, layers=3, hidden=32, head_width=32, head_depth=3, n_heads=5, cutoff=5.0)
    q0 = ref.generate(specs[0], 1234, count=5)
    q2 = ref.generate(specs[2], 1236, count=4)
    q3 = ref.generate(specs[3], 1237, count=3)
    model_case(med, [q0, q2, q3], [0, 2, 3], 7, False, "model_med.npz", extra_float=True)

    # ---------------------------------------------------------------- trainer
    h = O.Hyper(n_species=20, layers=2, hidden=16, head_width=16, head_depth=3, n_heads=2, cutoff=5.0)
    t0 = ref.generate(specs[0], 1234, count=6)
    t1 = ref.generate(dict(specs[1], dataset_id=1), 1235, count=6)
    s = concat([t0, t1])
    m = O.RefModel(ref, h, 7, [0, 1], dbl=False)
    tr = O.RefTrainer(ref, m)
    losses = [tr.step(s, threads=3) for _ in range(5)]
    np.savez_compressed(os.path.join(HERE, "train_ref.npz"), losses=np.array(losses), shared_after=m.block(-1),
                        head0_after=m.block(0), head1_after=m.block(1),
                        hyper=np.array([20, 2, 16, 16, 3, 2], np.int32), **s)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


EPOCH_CASES = [  # (counts, n_groups, replicas, mode, seed, b_local)
    ({0: 37, 1: 25, 2: 41, 3: 12, 4: 9}, 5, 1, 1, 11, 2),
    ({0: 37, 1: 25, 2: 41, 3: 12, 4: 9}, 5, 2, 1, 12, 1),
    ({0: 100, 1: 60}, 2, 3, 1, 13, 4),
    ({0: 37, 1: 25, 2: 41, 3: 12, 4: 9}, 1, 4, 0, 14, 3),
    ({0: 20, 3: 17}, 2, 2, 0, 15, 2),
    ({2: 50}, 1, 1, 0, 16, 5),
]


def epoch_plans():
    O.build(ref=True)
    ref = O.Ref()
    out = {}
    for i, (counts, ng, rep, mode, seed, b) in enumerate(EPOCH_CASES):
        for r in range(ng * rep):
            steps, ds, ix = ref.shuffle_epoch(counts, ng, rep, mode, seed, b, r)
            out[f"c{i}_r{r}_ds"], out[f"c{i}_r{r}_idx"], out[f"c{i}_r{r}_steps"] = ds, ix, np.array(steps)
    np.savez_compressed(os.path.join(HERE, "epoch_plan.npz"), **out)


def partitions():
    """make_partition (src/datastore.cpp:25-45) of the reference for every EPOCH_CASES mesh."""
    O.build(ref=True)
    ref = O.Ref()
    out = {}
    for i, (counts, ng, rep, mode, seed, b) in enumerate(EPOCH_CASES):
        part = ref.make_partition(counts, ng, rep, mode)
        for d, rows in part.items():
            out[f"c{i}_d{d}"] = np.array(rows, np.int64).reshape(-1, 3)
    np.savez_compressed(os.path.join(HERE, "partition.npz"), **out)


def hmtd_files():
    O.build(ref=True)
    ref = O.Ref()
    out = {}
    for k, cnt in ((0, 8), (3, 4)):
        spec = ref.default5_spec(k)
        s = ref.generate(spec, 4321 + k, count=cnt)
        ref.write_samples(os.path.join(HERE, f"hmtd_ds{k}.bin"), k, 1, s)
        for key, v in s.items():
            out[f"ds{k}_{key}"] = v
    np.savez_compressed(os.path.join(HERE, "hmtd.npz"), **out)


def ckpt_files():
    O.build(ref=True)
    ref = O.Ref()
    h = O.Hyper(n_species=20, layers=2, hidden=16, head_width=16, head_depth=3, n_heads=3, cutoff=5.0)
    m = O.RefModel(ref, h, 11, [0, 1, 2], dbl=True)
    out = {}
    for which in (-1, 0, 1, 2):
        b = m.block(which).astype(np.float32).astype(np.float64)  # FP32-representable blocks
        m.set_block(which, b)
        out["shared" if which < 0 else f"head{which}"] = b.astype(np.float32)
    m.save_checkpoint(os.path.join(HERE, "ckpt_ref.hmtp"))
    out["hyper"] = np.array([20, 2, 16, 16, 3, 3], np.int32)
    np.savez_compressed(os.path.join(HERE, "ckpt.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["ckpt"]:
        ckpt_files()
    elif sys.argv[1:] == ["epoch_plan"]:
        epoch_plans()
    elif sys.argv[1:] == ["partition"]:
        partitions()
    elif sys.argv[1:] == ["hmtd"]:
        hmtd_files()
    else:
        main()
