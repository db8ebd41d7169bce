"""Parity of the B200 path (through the C ABI) against the FP64 oracle, which is
itself pinned bit-exact to the reference (tests/test_oracle_golden.py).

Tolerances: integer/index work (edge sets) bit-exact; FP32 activations,
predictions and gradients norm-wise rel_vec_error <= 1e-4
(tests/oracles.hpp:62-74 metric of the reference; north star "rel 1e-4 in FP32").
"""
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN

import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data
from paper_2506_21788_b200.model import Samples

pytestmark = pytest.mark.gpu
TOL = 1e-4


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def hyper_pair(hv, cutoff=5.0):
    hp = P.ModelHyper(int(hv[0]), int(hv[1]), int(hv[2]), int(hv[3]), int(hv[4]), int(hv[5]), cutoff)
    return hp, O.Hyper(hp.n_species, hp.layers, hp.hidden, hp.head_width, hp.head_depth, hp.n_heads, cutoff)


def samples_of(g, prefix="in_"):
    return Samples(g[prefix + "n_atoms"], g[prefix + "species"], g[prefix + "pos"], g[prefix + "forces"],
                   g[prefix + "energy"], g[prefix + "dsid"])


def oracle_batch(o, s: Samples, cutoff):
    b = dict(n_atoms=s.n_atoms, species=s.species, pos=s.positions, forces=s.forces, energy=s.energy,
             dsid=s.dataset_id)
    return O.batch_from_samples(b, cutoff, o.build_edges)


def rel(a, b):
    return O.rel_vec_error(a, b)


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    O.build(ref=False)
    if P.lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def orc():
    return O.Oracle()


# ------------------------------------------------------------------ nbr list
def test_neighbour_list_bit_exact_vs_reference_fixtures():
    g = golden("nbr_kat.npz")
    hp = P.ModelHyper(n_heads=1)
    m = P.ModelT(hp, 7, [0])
    cases = [("kat", 5.0, "kat_n", "kat_pos", "kat_eo", "kat_dst", "kat_src")]
    cases += [(f"src{k}", 5.0, f"src{k}_n", f"src{k}_pos", f"src{k}_eo", f"src{k}_dst", f"src{k}_src") for k in range(5)]
    for name, rc, kn, kp, keo, kd, ks in cases:
        n = g[kn]
        s = Samples(n, np.zeros(n.sum(), np.uint8), g[kp], np.zeros_like(g[kp]), np.zeros(len(n)),
                    np.zeros(len(n), np.uint8))
        b = m.build_batch(s)
        assert np.array_equal(b.edge_dst, g[kd]), name
        assert np.array_equal(b.edge_src, g[ks]), name
        assert np.array_equal(b.edge_offset, g[keo]), name
    # cfg4-like cells at rc 6
    hp6 = P.ModelHyper(n_heads=1, cutoff=6.0)
    m6 = P.ModelT(hp6, 7, [0])
    n = g["big_n"]
    s = Samples(n, np.zeros(n.sum(), np.uint8), g["big_pos"], np.zeros_like(g["big_pos"]), np.zeros(len(n)),
                np.zeros(len(n), np.uint8))
    b = m6.build_batch(s)
    assert np.array_equal(b.edge_dst, g["big_dst"]) and np.array_equal(b.edge_src, g["big_src"])


def test_at_cutoff_pairs_inclusive():
    hp = P.ModelHyper(n_heads=1)
    m = P.ModelT(hp, 7, [0])
    pos = np.array([[0, 0, 0], [5, 0, 0], [0, 0, 0], [3, 4, 0], [0, 0, 0], [5.000000000000001, 0, 0]], float)
    s = Samples([2, 2, 2], np.zeros(6, np.uint8), pos, np.zeros_like(pos), np.zeros(3), np.zeros(3, np.uint8))
    b = m.build_batch(s)
    assert list(np.diff(b.edge_offset)) == [2, 2, 0]


# ------------------------------------------------------------------ model
def run_both(orc, hp, oh, s: Samples, owned, seed=7, upstream="loss"):
    m = P.ModelT(hp, seed, owned)
    sh = orc.init_block(oh, seed, -1)
    heads = {k: orc.init_block(oh, seed, k) for k in owned}
    b = oracle_batch(orc, s, hp.cutoff)
    E, F, cache = orc.forward(oh, sh, heads, b)
    L, dE, dF = orc.loss(b, E, F)
    pred = m.forward(s)
    return m, dict(sh=sh, heads=heads, b=b, E=E, F=F, cache=cache, L=L, dE=dE, dF=dF), pred


@pytest.mark.parametrize("case", ["model_tiny.npz", "model_med.npz"])
def test_forward_backward_parity_golden_cases(orc, case):
    g = golden(case)
    hp, oh = hyper_pair(g["hyper"])
    owned = [int(k) for k in g["owned"]]
    s = samples_of(g)
    m, r, pred = run_both(orc, hp, oh, s, owned)
    # reference predictions are the fixture itself
    assert rel(pred.energy_per_atom, g["energy"]) < TOL
    assert rel(pred.forces, g["forces"]) < TOL
    L = m.loss()
    assert abs(L - g["loss"]) / abs(g["loss"]) < TOL
    assert rel(m.debug("dE"), g["dE"]) < TOL and rel(m.debug("dF"), g["dF"]) < TOL
    gb = m.backward(None, None)  # device upstreams of the SPEC loss
    assert rel(gb.shared, g["g_shared"]) < TOL
    for k in owned:
        assert rel(gb.heads[k], g[f"g_head{k}"]) < TOL, k


def test_per_layer_activations_parity(orc):
    """ForwardCacheT parity points (hmtl/model.hpp:117-151), layer by layer."""
    g = golden("model_tiny.npz")
    hp, oh = hyper_pair(g["hyper"])
    owned = [int(k) for k in g["owned"]]
    s = samples_of(g)
    m, r, pred = run_both(orc, hp, oh, s, owned)
    c = r["cache"]
    N, E, G = s.N, len(r["b"]["edge_dst"]), s.G
    H, W = hp.hidden, hp.head_width
    for l in range(hp.layers):
        assert rel(m.debug("h", l), c["h_in"][l]) < TOL, ("h_in", l)
        assert rel(m.debug("z1", l), c["z1"][l]) < TOL, ("z1", l)
        assert rel(m.debug("z2", l), c["z2"][l]) < TOL, ("z2", l)
        assert rel(m.debug("agg", l), c["agg"][l]) < TOL, ("agg", l)
        assert rel(m.debug("vz1", l), c["vz1"][l]) < TOL, ("vz1", l)
    assert rel(m.debug("h", hp.layers), c["h_final"]) < TOL
    assert rel(m.debug("pooled"), c["pooled"]) < TOL
    for i in range(hp.head_depth):
        w = W if i < hp.head_depth - 1 else 1
        assert rel(m.debug("ez", i).reshape(G, W)[:, :w], c["ez"][i][:, :w]) < TOL, ("ez", i)
    for i in range(1, hp.head_depth - 1):
        assert rel(m.debug("zf", i), c["fz"][i]) < TOL, ("zf", i)
    assert rel(m.debug("s"), c["s"]) < TOL


def five_source_batch(counts=(6, 5, 5, 3, 2), seed=1234):
    specs = data.default5_specs()
    return Samples.concat([data.generate_dataset(sp, seed + k, count=c) for k, (sp, c) in enumerate(zip(specs, counts))])


@pytest.mark.parametrize("H,W,L,D", [(64, 64, 3, 3), (32, 48, 2, 4), (128, 128, 4, 3), (16, 16, 1, 2)])
def test_parity_five_heads_shapes(orc, H, W, L, D):
    s = five_source_batch()
    hp = P.ModelHyper(20, L, H, W, D, 5, 5.0)
    oh = O.Hyper(20, L, H, W, D, 5, 5.0)
    owned = [0, 1, 2, 3, 4]
    m, r, pred = run_both(orc, hp, oh, s, owned)
    assert rel(pred.energy_per_atom, r["E"]) < TOL
    assert rel(pred.forces, r["F"]) < TOL
    gb = m.backward(r["dE"], r["dF"])
    gs, gh = orc.backward(oh, r["sh"], r["heads"], r["b"], r["cache"], r["dE"], r["dF"])
    assert rel(gb.shared, gs) < TOL
    for k in owned:
        assert rel(gb.heads[k], gh[k]) < TOL, k


def test_taskpar_rank_owns_subset_and_rejects_foreign(orc):
    s = five_source_batch()
    sel = [i for i in range(s.G) if s.dataset_id[i] in (1, 3)]
    sub = s.take(sel)
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    oh = O.Hyper(20, 2, 32, 32, 3, 5, 5.0)
    m, r, pred = run_both(orc, hp, oh, sub, [1, 3])
    assert rel(pred.forces, r["F"]) < TOL
    gb = m.backward(r["dE"], r["dF"])
    gs, gh = orc.backward(oh, r["sh"], r["heads"], r["b"], r["cache"], r["dE"], r["dF"])
    assert rel(gb.shared, gs) < TOL and rel(gb.heads[3], gh[3]) < TOL
    with pytest.raises(P.HmtlError) as ei:
        m.forward(s)  # contains datasets 0,2,4 -> unowned (hmtl/model.hpp:345-347)
    assert ei.value.code == 1


def test_empty_graph_rejected():
    m = P.ModelT(P.ModelHyper(), 5, [0])
    s = Samples([2, 0], np.zeros(2, np.uint8), np.zeros((2, 3)), np.zeros((2, 3)), np.zeros(2), np.zeros(2, np.uint8))
    with pytest.raises(P.HmtlError) as ei:
        m.forward(s)
    assert ei.value.code == 1


def test_single_node_no_edges(orc):
    hp = P.ModelHyper(layers=2, hidden=8, head_width=8)
    m = P.ModelT(hp, 5, [0])
    s = Samples([1], [3], [[1.0, 2.0, 3.0]], [[0, 0, 0]], [0.0], [0])
    p1 = m.forward(s)
    assert p1.forces[0, 0] == 0.0 and np.isfinite(p1.energy_per_atom[0])
    s2 = Samples([1], [3], [[-4.0, 0.5, 9.0]], [[0, 0, 0]], [0.0], [0])
    p2 = m.forward(s2)
    assert p2.energy_per_atom[0] == p1.energy_per_atom[0]


def test_two_atom_antisymmetry_bit_exact():
    hp = P.ModelHyper(layers=2, hidden=8, head_width=8)
    m = P.ModelT(hp, 9, [0])
    s = Samples([2], [2, 4], [[0.3, -0.2, 0.1], [1.4, 0.8, -0.5]], np.zeros((2, 3)), [0.0], [0])
    p = m.forward(s)
    assert np.array_equal(p.forces[0], -p.forces[1])


def test_zero_upstream_zero_grads():
    hp = P.ModelHyper(layers=2, hidden=8, head_width=8)
    m = P.ModelT(hp, 3, [0])
    s = five_source_batch((4, 0, 0, 0, 0))
    m.forward(s)
    g = m.backward(np.zeros(s.G), np.zeros((s.N, 3)))
    assert not g.shared.any() and not g.heads[0].any()


def test_head_isolation():
    s = five_source_batch((3, 3, 0, 0, 0))
    hp = P.ModelHyper(layers=2, hidden=8, head_width=8, n_heads=2)
    m = P.ModelT(hp, 43, [0, 1])
    p1 = m.forward(s)
    m.set_head_block(1, m.head_block(1) + 0.05)
    p2 = m.forward(s)
    d = s.dataset_id
    assert np.array_equal(p1.energy_per_atom[d == 0], p2.energy_per_atom[d == 0])
    assert np.all(p1.energy_per_atom[d == 1] != p2.energy_per_atom[d == 1])


def test_rigid_motion_invariance():
    rng = np.random.default_rng(77)
    hp = P.ModelHyper(layers=2, hidden=16, head_width=16)
    m = P.ModelT(hp, 31, [0])
    base = five_source_batch((6, 0, 0, 0, 0))
    for trial in range(5):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        t = rng.uniform(-5, 5, 3)
        p1 = m.forward(base)
        rot = Samples(base.n_atoms, base.species, base.positions @ q.T + t, base.forces, base.energy, base.dataset_id)
        p2 = m.forward(rot)
        assert rel(p2.energy_per_atom, p1.energy_per_atom) < 1e-4
        assert rel(p2.forces, p1.forces @ q.T) < 1e-4


def test_determinism_bitwise():
    s = five_source_batch()
    hp = P.ModelHyper(20, 3, 64, 64, 3, 5, 5.0)
    outs = []
    for _ in range(2):
        m = P.ModelT(hp, 7, range(5))
        p = m.forward(s)
        m.loss()
        g = m.backward()
        outs.append((p.energy_per_atom.copy(), p.forces.copy(), g.shared.copy()))
        m.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("order", ["interleaved", "reversed"])
def test_parity_batch_not_grouped_by_head(orc, order):
    """Graphs not grouped by head (head-sorted permutations in use: permuted row sets,
    register-operand weight gradients) -- the grouped case takes identity row sets and
    TMA operands; both must match the oracle."""
    s = five_source_batch()
    idx = np.arange(s.G)
    idx = idx[::-1] if order == "reversed" else np.argsort(idx % 5, kind="stable")[::-1].copy()
    rng = np.random.default_rng(5)
    if order == "interleaved":
        rng.shuffle(idx)
    u = s.take(idx.tolist())
    hp = P.ModelHyper(20, 2, 128, 128, 3, 5, 5.0)
    oh = O.Hyper(20, 2, 128, 128, 3, 5, 5.0)
    m, r, pred = run_both(orc, hp, oh, u, [0, 1, 2, 3, 4])
    assert rel(pred.energy_per_atom, r["E"]) < TOL and rel(pred.forces, r["F"]) < TOL
    gb = m.backward(r["dE"], r["dF"])
    gs, gh = orc.backward(oh, r["sh"], r["heads"], r["b"], r["cache"], r["dE"], r["dF"])
    assert rel(gb.shared, gs) < TOL
    for k in range(5):
        assert rel(gb.heads[k], gh[k]) < TOL, k
