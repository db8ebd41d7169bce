"""Error semantics of the device training step (the reference throws before any
update: hmtl/model.hpp:341-347 unowned/empty, :483-486 non-finite; build_batch
contract hmtl/graph.hpp:56) and capacity growth that keeps training state.

A step whose batch trips a device error bit must raise the reference's error
when its result is read AND leave parameters, AdamW m/v and the step counter
untouched; an edge-capacity overflow must not read or write past the
capacity-sized buffers (the run below would fault otherwise) and the next valid
step must train normally.
"""
import numpy as np
import pytest

import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data
from paper_2506_21788_b200.model import Samples

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    if P.lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")


def batch(counts, seed=1234):
    specs = data.default5_specs()
    return Samples.concat([data.generate_dataset(sp, seed + k, count=c) for k, (sp, c) in enumerate(zip(specs, counts)) if c])


def state(m):
    return [m.shared_block()] + [m.head_block(k) for k in m.owned]


def same(a, b):
    return all(np.array_equal(x, y, equal_nan=True) for x, y in zip(a, b))


@pytest.mark.parametrize("use_graph", [False, True])
def test_non_finite_prediction_raises_and_skips_update(use_graph):
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    s = batch((3, 2, 2, 1, 1))
    m = P.ModelT(hp, 7, range(5), caps=P.Caps.for_samples(s))
    cfg = P.TrainConfig(use_graph=use_graph)
    m.train_step(s, cfg)
    m.train_step(s, cfg)  # (graph mode: captured and replayed from here on)
    hb = m.head_block(2)
    bad = hb.copy()
    bad[-1] = np.nan  # force.b2 of head 2 -> every force of head-2 graphs is NaN
    m.set_head_block(2, bad)
    before = state(m)
    with pytest.raises(P.HmtlError) as ei:
        m.train_step(s, cfg)
    assert ei.value.code == 1 and "non-finite" in str(ei.value)
    assert same(state(m), before)  # parameters untouched (no AdamW, no decay)
    # repair the head: training resumes with the step counter where it was
    m.set_head_block(2, hb)
    L = m.train_step(s, cfg)
    ref = P.ModelT(hp, 7, range(5), caps=P.Caps.for_samples(s))
    for _ in range(3):
        Lr = ref.train_step(s, P.TrainConfig(use_graph=use_graph))
    assert np.isfinite(L) and abs(L - Lr) <= 1e-6 * abs(Lr)
    for a, b in zip(state(m), state(ref)):
        assert np.array_equal(a, b)


def test_pbc_edge_overflow_raises_without_out_of_bounds():
    hp = P.ModelHyper(20, 2, 32, 32, 3, 1, 5.0)
    rng = np.random.default_rng(3)
    n = np.array([4, 4], np.int32)
    pos = rng.uniform(0.0, 2.0, size=(8, 3))
    s = Samples(n, np.zeros(8, np.uint8), pos, np.zeros((8, 3)), np.zeros(2), np.zeros(2, np.uint8))
    cells = np.tile(np.eye(3) * 2.0, (2, 1, 1))  # 2 A cubic cells at rc 5: ~130 images per atom
    m = P.ModelT(hp, 7, [0], caps=P.Caps(4, 16, 64))
    m.reserve = lambda *a, **k: None  # keep the deliberately small edge capacity
    before = state(m)
    m.upload_pbc(s, cells)
    with pytest.raises(P.HmtlError) as ei:
        m.train_step(None, P.TrainConfig(use_graph=False))
    assert ei.value.code == 1 and "edge capacity" in str(ei.value)
    assert same(state(m), before)
    # an open-boundary batch that fits trains normally afterwards (error bits reset per step)
    ok = Samples(np.array([3], np.int32), np.zeros(3, np.uint8), np.array([[0, 0, 0], [1.2, 0, 0], [0, 1.3, 0]], float),
                 np.zeros((3, 3)), np.zeros(1), np.zeros(1, np.uint8))
    L = m.train_step(ok, P.TrainConfig(use_graph=False))
    assert np.isfinite(L) and not same(state(m), before)


def test_reserve_keeps_adamw_state_and_step():
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    small, big = batch((2, 1, 1, 1, 0), 5), batch((6, 5, 4, 3, 2), 6)
    cfg = P.TrainConfig(use_graph=True)
    grown = P.ModelT(hp, 7, range(5), caps=P.Caps.for_samples(small))
    wide = P.ModelT(hp, 7, range(5), caps=P.Caps.for_samples(small).union(P.Caps.for_samples(big)))
    La = [grown.train_step(x, cfg) for x in (small, small, big, small)]  # big forces a reserve
    Lb = [wide.train_step(x, cfg) for x in (small, small, big, small)]
    assert grown.caps.covers(big)
    np.testing.assert_allclose(La, Lb, rtol=1e-5)
    for a, b in zip(state(grown), state(wide)):
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)


def test_nbr_build_standalone_matches_model_path():
    """hmtl_nbr_build (no model context, any dataset ids) == the step's edge set."""
    s = batch((3, 2, 2, 1, 1))
    ids = s.dataset_id.copy()
    ids[:] = np.arange(s.G) % 40  # more than 16 distinct ids: the old C++ build_batch truncated them
    s40 = Samples(s.n_atoms, s.species, s.positions, s.forces, s.energy, ids.astype(np.uint8))
    e = P.nbr_build(s40, 5.0)
    m = P.ModelT(P.ModelHyper(n_heads=5), 7, range(5))
    b = m.build_batch(s)
    assert np.array_equal(e["edge_dst"], b.edge_dst) and np.array_equal(e["edge_src"], b.edge_src)
    assert np.array_equal(e["edge_offset"], b.edge_offset)
    # rev is the reverse edge, row_ptr the dst-major CSR
    assert np.array_equal(e["edge_src"][e["rev"]], e["edge_dst"]) and np.array_equal(e["edge_dst"][e["rev"]], e["edge_src"])
    assert np.array_equal(np.repeat(np.arange(s.N), np.diff(e["row_ptr"])), e["edge_dst"])
