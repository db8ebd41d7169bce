"""CPU-only checks of the product library's host side (no GPU needed):
the C ABI loads and exports every declared symbol, layouts/init/generator
match the reference fixtures, placement and census formulas."""
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, ROOT

import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data
from paper_2506_21788_b200._lib import HmtlError, lib


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hmtl_b200.h")).read()
    declared = set(re.findall(r"\b(hmtl_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 30
    L = lib()
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert L.hmtl_abi_version() == 1


def test_layouts_match_reference_restatement(oracle):
    for hp in (P.ModelHyper(layers=2, hidden=8, head_width=8, n_heads=2),
               P.ModelHyper(layers=4, hidden=128, head_width=128, head_depth=3, n_heads=5),
               P.ModelHyper(layers=3, hidden=16, head_width=24, head_depth=4, n_heads=1)):
        h = O.Hyper(hp.n_species, hp.layers, hp.hidden, hp.head_width, hp.head_depth, hp.n_heads, hp.cutoff)
        assert P.shared_layout(hp) == oracle.layout(h, True)
        assert P.head_layout(hp) == oracle.layout(h, False)


def test_init_matches_reference_params():
    g = dict(np.load(os.path.join(GOLDEN, "model_med.npz")))
    hv = g["hyper"]
    hp = P.ModelHyper(int(hv[0]), int(hv[1]), int(hv[2]), int(hv[3]), int(hv[4]), int(hv[5]))
    import ctypes as C
    out = np.zeros(len(g["shared"]), np.float32)
    assert lib().hmtl_init_block(C.byref(hp.c()), int(g["seed"]), -1, out.ctypes.data_as(C.POINTER(C.c_float))) == 0
    np.testing.assert_array_equal(out, g["shared"].astype(np.float32))  # static_cast<float>(double draw)
    for k in g["owned"]:
        out = np.zeros(len(g[f"head{k}"]), np.float32)
        lib().hmtl_init_block(C.byref(hp.c()), int(g["seed"]), int(k), out.ctypes.data_as(C.POINTER(C.c_float)))
        np.testing.assert_array_equal(out, g[f"head{k}"].astype(np.float32))


def test_generator_bit_identical_to_reference():
    g = dict(np.load(os.path.join(GOLDEN, "dataset5.npz")))
    specs = data.default5_specs()
    for k, s in enumerate(specs):
        assert s.elements == list(g[f"spec{k}_elements"])
        assert [s.n_min, s.n_max, s.alpha, s.sigma] == list(g[f"spec{k}_params"])
        assert np.array_equal(s.mu, g[f"spec{k}_mu"])
        x = data.generate_dataset(s, 1234 + k, count=6)
        for f, key in (("n_atoms", "n_atoms"), ("species", "species"), ("positions", "pos"), ("forces", "forces"),
                       ("energy", "energy"), ("dataset_id", "dsid")):
            assert np.array_equal(getattr(x, f), g[f"src{k}_{key}"]), (k, f)
    c1 = data.DatasetSpec(0, [0, 1, 2, 3], 18, 22, 1.0, 0.01)
    x = data.generate_dataset(c1, 1234, count=4)
    assert np.array_equal(x.positions, g["cfg1_pos"]) and np.array_equal(x.energy, g["cfg1_energy"])


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
def test_head_placement_balanced(world):
    w = np.array([1, 1, 1, 2, 3], float)
    share = data.head_placement(world, w)
    assert np.allclose(share.sum(axis=0), 1.0)  # every head fully served
    load = share @ w
    assert np.allclose(load, w.sum() / world)  # equal work per rank
    for k in range(5):  # equal split within each head sub-group
        s = share[:, k][share[:, k] > 0]
        assert np.allclose(s, s[0])


def test_head_placement_matches_survey_maps():
    """P=8 -> GPUs-per-head {1,1,1,2,3}; P=2 -> heads-per-GPU {3,2}."""
    s8 = data.head_placement(8, [1, 1, 1, 2, 3])
    assert list((s8 > 0).sum(axis=0)) == [1, 1, 1, 2, 3]
    s2 = data.head_placement(2, [1, 1, 1, 2, 3])
    assert sorted((s2 > 0).sum(axis=1)) == [2, 3]


def test_regime_and_footprint_census():
    assert P.classify_regime(1000000, 1000, 2) == 1
    assert P.classify_regime(1000, 1000000, 5) == 2
    assert P.classify_regime(10000, 2000, 5) == 3
    assert P.memory_footprint(1000, 200, 5, "base") == 2000
    assert P.memory_footprint(1000, 200, 5, "taskpar") == 1200
    hp = P.ModelHyper.paper_preset(5)
    sl, hl = P.shared_layout(hp), P.head_layout(hp)
    ps = sl[-1][3] + sl[-1][1] * sl[-1][2]
    ph = hl[-1][3] + hl[-1][1] * hl[-1][2]
    assert (ps, ph) == (18033584, 3126615)
    assert P.classify_regime(ps, ph, 5) == 3


def test_no_cpu_fallback_without_device():
    if lib().hmtl_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(HmtlError) as ei:
        P.ModelT(P.ModelHyper(), 7, [0])
    assert ei.value.code == 6 and "no CPU fallback" in str(ei.value)
