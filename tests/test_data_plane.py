"""Data plane on the hot path's input side: the epoch plan
(shuffle_epoch, src/datastore.cpp:47-97) and the device-resident sample store
that assembles each step's batch in HBM (DataStore, hmtl/datastore.hpp:77-115).

The plan is host C++ behind the C ABI (no GPU needed) and must equal the
reference's own shuffle_epoch item for item (tests/golden/epoch_plan.npz, made
by tests/golden/make_golden.py from the unmodified reference)."""
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data

sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN)))
from golden.make_golden import EPOCH_CASES  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()


def mesh_members(counts, n_groups, replicas):
    return {k: list(range(k * replicas, (k + 1) * replicas)) for k in counts}


@pytest.mark.parametrize("case", range(len(EPOCH_CASES)))
def test_epoch_plan_matches_reference(case):
    g = np.load(os.path.join(GOLDEN, "epoch_plan.npz"))
    counts, ng, rep, mode, seed, b = EPOCH_CASES[case]
    members = mesh_members(counts, ng, rep) if mode == 1 else None
    for r in range(ng * rep):
        steps, ds, ix = P.epoch_plan("taskpar" if mode == 1 else "base", counts, ng * rep, seed, b, r, members)
        assert steps == int(g[f"c{case}_r{r}_steps"])
        assert np.array_equal(ds, g[f"c{case}_r{r}_ds"]), (case, r)
        assert np.array_equal(ix, g[f"c{case}_r{r}_idx"]), (case, r)


@pytest.mark.parametrize("case", range(len(EPOCH_CASES)))
def test_partition_matches_reference(case):
    """make_partition / balanced_split (src/datastore.cpp:11-45) vs the reference's own
    (tests/golden/partition.npz): serving ranks and shard ranges per dataset."""
    g = np.load(os.path.join(GOLDEN, "partition.npz"))
    counts, ng, rep, mode, seed, b = EPOCH_CASES[case]
    members = mesh_members(counts, ng, rep) if mode == 1 else None
    part = P.make_partition(counts, ng * rep, "taskpar" if mode == 1 else "base", members)
    for d, (cnt, serving, ranges) in part.items():
        mine = np.array([(r, lo, hi) for r, (lo, hi) in zip(serving, ranges)], np.int64)
        assert np.array_equal(mine, g[f"c{case}_d{d}"]), (case, d)
        assert cnt == counts[d] and ranges[0][0] == 0 and ranges[-1][1] == cnt


def test_shard_range_errors():
    with pytest.raises(P.HmtlError):
        P.shard_range(10, 0, 0)
    with pytest.raises(P.HmtlError):
        P.shard_range(10, 3, 3)
    assert [P.shard_range(10, 4, i) for i in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]


def test_taskpar_routing_and_coverage_general_placement():
    """Placement groups of different sizes (5 heads on 8 ranks, shares {1,1,1,2,3}):
    every rank draws only its group's dataset, replicas get disjoint samples,
    and all groups take the same number of steps."""
    share = data.head_placement(8, (1, 1, 1, 2, 3))
    members = {k: [r for r in range(8) if share[r, k] > 0] for k in range(5)}
    counts = {0: 400, 1: 300, 2: 350, 3: 500, 4: 600}
    plans = [P.epoch_plan("taskpar", counts, 8, 99, 4, r, members) for r in range(8)]
    assert len({p[0] for p in plans}) == 1
    for k, grp in members.items():
        seen = set()
        for r in grp:
            steps, ds, ix = plans[r]
            assert set(ds.tolist()) <= {k}
            items = set(ix.tolist())
            assert not (seen & items)
            seen |= items
    for r in range(8):
        assert set(plans[r][1].tolist()) <= {k for k, grp in members.items() if r in grp}


def test_epoch_plan_errors():
    with pytest.raises(P.HmtlError):
        P.epoch_plan("base", {0: 10}, 1, 1, 0, 0)
    with pytest.raises(P.HmtlError):
        P.epoch_plan("taskpar", {0: 10, 1: 5}, 2, 1, 1, 0, {0: [0]})  # dataset 1 without a sub-group


@pytest.mark.gpu
def test_store_batch_equals_host_batch():
    """A plan's batch gathered on the device from the HBM pool is the batch the
    host would pack: same edges, and a train step gives a bit-identical loss."""
    specs = data.default5_specs()
    parts = [data.generate_dataset(sp, 1234 + k, count=c) for k, (sp, c) in enumerate(zip(specs, (30, 20, 20, 8, 6)))]
    pool = P.Samples.concat(parts)
    store = P.SampleStore(pool)
    counts = store.counts()
    assert counts == {k: c for k, c in enumerate((30, 20, 20, 8, 6))}
    steps, ds, ix = P.epoch_plan("base", counts, 1, 5, 8, 0)
    assert steps == 10
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    offs = {k: np.cumsum([0] + [p.G for p in parts])[k] for k in range(5)}
    cfg = P.TrainConfig(use_graph=False)
    for s in range(3):
        d, i = ds[s * 8:(s + 1) * 8], ix[s * 8:(s + 1) * 8]
        host = pool.take([int(offs[int(a)] + int(b)) for a, b in zip(d, i)])
        caps = P.Caps.for_samples(host)
        m1 = P.ModelT(hp, 7, range(5), caps=caps)
        m2 = P.ModelT(hp, 7, range(5), caps=caps)
        store.bind(m1, d, i)
        L1 = m1.train_step(None, cfg)
        L2 = m2.train_step(host, cfg)
        assert L1 == L2, (s, L1, L2)
        assert np.array_equal(m1.shared_block(), m2.shared_block())
        m1.close()
        m2.close()
    with pytest.raises(P.HmtlError):
        store.bind(P.ModelT(hp, 7, [0], caps=P.Caps(64, 4096, 1 << 20)), np.array([1], np.uint8), np.array([0], np.uint64))
    with pytest.raises(P.HmtlError):
        store.bind(P.ModelT(hp, 7, [0], caps=P.Caps(64, 4096, 1 << 20)), np.array([0], np.uint8), np.array([30], np.uint64))
    store.close()


def hmtd_samples(k):
    g = np.load(os.path.join(GOLDEN, "hmtd.npz"))
    return P.Samples(g[f"ds{k}_n_atoms"], g[f"ds{k}_species"], g[f"ds{k}_pos"], g[f"ds{k}_forces"],
                     g[f"ds{k}_energy"], g[f"ds{k}_dsid"])


@pytest.mark.parametrize("k", [0, 3])
def test_hmtd_writer_byte_identical_to_reference(k, tmp_path):
    """Our writer reproduces the reference's write_sample_file byte for byte
    (fixture files written by the unmodified reference)."""
    ref_bytes = open(os.path.join(GOLDEN, f"hmtd_ds{k}.bin"), "rb").read()
    out = str(tmp_path / f"x{k}.bin")
    P.hmtd_write(out, k, 1, hmtd_samples(k))
    assert open(out, "rb").read() == ref_bytes
    assert P.hmtd_header(out) == (k, 1, len(hmtd_samples(k).n_atoms))


def test_hmtd_header_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(P.HmtlError):
        P.hmtd_header(str(bad))
    with pytest.raises(P.HmtlError):
        P.hmtd_header(str(tmp_path / "missing.bin"))


@pytest.mark.gpu
def test_store_from_hmtd_matches_reference_samples(tmp_path):
    """Reference-written HMTD files -> GPU CRC check + parse -> device batch: a
    train step on it equals the step on the same samples uploaded from the host."""
    files = [os.path.join(GOLDEN, f"hmtd_ds{k}.bin") for k in (0, 3)]
    store = P.SampleStore.from_hmtd(files)
    assert store.counts() == {0: 8, 3: 4}
    host = P.Samples.concat([hmtd_samples(0), hmtd_samples(3)])
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    caps = P.Caps.for_samples(host)
    cfg = P.TrainConfig(use_graph=False)
    m1, m2 = P.ModelT(hp, 7, [0, 3], caps=caps), P.ModelT(hp, 7, [0, 3], caps=caps)
    store.bind(m1, np.array([0] * 8 + [3] * 4, np.uint8), np.array(list(range(8)) + list(range(4)), np.uint64))
    assert m1.train_step(None, cfg) == m2.train_step(host, cfg)
    assert np.array_equal(m1.head_block(3), m2.head_block(3))
    m1.close(), m2.close(), store.close()
    # a flipped byte inside a record -> the GPU CRC check rejects the file (io)
    raw = bytearray(open(files[1], "rb").read())
    raw[18 + 40] ^= 0x10
    bad = tmp_path / "bad.bin"
    bad.write_bytes(bytes(raw))
    with pytest.raises(P.HmtlError, match="CRC"):
        P.SampleStore.from_hmtd([files[0], str(bad)])
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(bytes(raw[:-7]))
    with pytest.raises(P.HmtlError, match="truncated"):
        P.SampleStore.from_hmtd([str(trunc)])


@pytest.mark.gpu
def test_align_energies_matches_reference(tmp_path):
    """align_energies (src/dataset.cpp:263-356) on the GPU vs the reference's
    own (oracle/_ref): per-element offsets (NaN pattern exact, values to 1e-9), aligned labels
    to 1e-10, structures byte-identical, output headers aligned = 1; planted offsets recovered."""
    import oracle as O

    O.build(ref=True)
    ref = O.Ref()
    files = []
    for k, planted in ((0, None), (1, {0: 1.25, 1: -0.75}), (3, {2: 0.5})):
        spec = ref.default5_spec(k)
        if planted:
            mu = list(spec["mu"])
            for e, v in planted.items():
                mu[e] += v
            spec = dict(spec, mu=mu)
        s = ref.generate(spec, 500 + k, count=60 + 10 * k)
        f = str(tmp_path / f"in{k}.hmtd")
        ref.write_samples(f, k, 0, s)
        files.append(f)
    out_r = [str(tmp_path / f"ref{k}.hmtd") for k in range(3)]
    out_g = [str(tmp_path / f"gpu{k}.hmtd") for k in range(3)]
    off_r, sk_r = ref.align_energies(files, 0, out_r)
    off_g, sk_g = P.align_energies(files, 0, out_g)
    assert sorted(off_r) == sorted(off_g) and sk_r == sk_g
    for d in off_r:
        a, b = off_r[d], off_g[d]
        assert np.array_equal(np.isnan(a), np.isnan(b)), d
        m = ~np.isnan(a)
        assert np.all(np.abs(a[m] - b[m]) <= 1e-9 * np.maximum(1.0, np.abs(a[m]))), d
    for fr, fg in zip(out_r, out_g):
        assert P.hmtd_header(fg)[1] == 1
        sr, sg = P.SampleStore.from_hmtd([fr]).download(), P.SampleStore.from_hmtd([fg]).download()
        assert np.array_equal(sr.n_atoms, sg.n_atoms) and np.array_equal(sr.species, sg.species)
        assert np.array_equal(sr.positions, sg.positions) and np.array_equal(sr.forces, sg.forces)
        assert np.max(np.abs(sr.energy - sg.energy)) < 1e-10
    with pytest.raises(P.HmtlError):
        P.align_energies(files[:1], 0, out_g[:1])  # need at least two datasets
    with pytest.raises(P.HmtlError):
        P.align_energies(files[1:], 0, out_g[1:])  # reference dataset not among inputs
