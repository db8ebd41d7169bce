"""Pin the FP64 C restatement (oracle/hmtl_oracle.c) against fixtures that the
unmodified reference produced (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def hyper_of(g):
    h = g["hyper"]
    return O.Hyper(int(h[0]), int(h[1]), int(h[2]), int(h[3]), int(h[4]), int(h[5]), float(g.get("cutoff", 5.0)))


def test_neighbour_list_kats_bit_exact(oracle):
    g = load("nbr_kat.npz")
    go, eo, dst, src = oracle.build_edges(g["kat_n"], g["kat_pos"], 5.0)
    assert np.array_equal(dst, g["kat_dst"]) and np.array_equal(src, g["kat_src"])
    assert np.array_equal(eo, g["kat_eo"])
    # the two at-cutoff pairs (d^2 == 25 exactly) are inclusive (graph.hpp:71); 5+1ulp is not
    assert list(np.diff(g["kat_eo"])[:3]) == [2, 2, 0]
    for k in range(5):
        go, eo, dst, src = oracle.build_edges(g[f"src{k}_n"], g[f"src{k}_pos"], 5.0)
        assert np.array_equal(dst, g[f"src{k}_dst"]) and np.array_equal(src, g[f"src{k}_src"])
        assert np.array_equal(eo, g[f"src{k}_eo"])
    go, eo, dst, src = oracle.build_edges(g["big_n"], g["big_pos"], 6.0)
    assert np.array_equal(dst, g["big_dst"]) and np.array_equal(src, g["big_src"])


def test_empty_graph_rejected(oracle):
    with pytest.raises(ValueError):
        oracle.build_edges(np.array([2, 0], np.int32), np.zeros((2, 3)), 5.0)


def _batch(g):
    return {k[3:]: v for k, v in g.items() if k.startswith("in_")}


@pytest.mark.parametrize("name", ["model_tiny.npz", "model_med.npz"])
def test_params_forward_backward_match_reference(oracle, name):
    g = load(name)
    h = hyper_of(g)
    owned = [int(k) for k in g["owned"]]
    sh = oracle.init_block(h, int(g["seed"]), -1)
    assert np.array_equal(sh, g["shared"])  # init_block_, model.hpp:211-225
    heads = {k: oracle.init_block(h, int(g["seed"]), k) for k in owned}
    for k in owned:
        assert np.array_equal(heads[k], g[f"head{k}"])
    b = _batch(g)
    E, F, c = oracle.forward(h, sh, heads, b)
    np.testing.assert_array_equal(E, g["energy"])
    np.testing.assert_array_equal(F, g["forces"])
    for key in O.CACHE_KEYS:
        if f"cache_{key}" in g:
            np.testing.assert_array_equal(c[key], g[f"cache_{key}"], err_msg=key)
    L, dE, dF = oracle.loss(b, E, F)
    assert L == g["loss"]
    gs, gh = oracle.backward(h, sh, heads, b, c, dE, dF)
    np.testing.assert_array_equal(gs, g["g_shared"])
    for k in owned:
        np.testing.assert_array_equal(gh[k], g[f"g_head{k}"])


def test_reference_fp32_noise_floor_documented():
    """ModelT<float> vs ModelT<double>: the floor any FP32 path sits on."""
    g = load("model_med.npz")
    assert O.rel_vec_error(g["f32_energy"], g["energy"]) < 1e-5
    assert O.rel_vec_error(g["f32_forces"], g["forces"]) < 1e-5
    assert O.rel_vec_error(g["f32_g_shared"], g["g_shared"]) < 1e-4


def test_fd_gradient_three_atom_graph(oracle):
    """Mirror of tests/test_model.cpp:334-357 on the restatement."""
    h = O.Hyper(layers=2, hidden=8, head_width=8, head_depth=3, n_heads=1)
    rng = np.random.default_rng(15)
    b = dict(n_atoms=np.array([3], np.int32), species=rng.integers(0, 20, 3).astype(np.uint8),
             pos=rng.uniform(0, 3.5, (3, 3)), forces=np.zeros((3, 3)), energy=np.zeros(1), dsid=np.zeros(1, np.uint8))
    b = O.batch_from_samples(b, 5.0, oracle.build_edges)
    sh = oracle.init_block(h, 29, -1)
    hd = {0: oracle.init_block(h, 29, 0)}
    we = rng.uniform(-1, 1, 1)
    wf = rng.uniform(-1, 1, 9)
    E, F, c = oracle.forward(h, sh, hd, b)
    gs, gh = oracle.backward(h, sh, hd, b, c, we, wf)

    def readout(shv, hv):
        E, F, _ = oracle.forward(h, shv, {0: hv}, b, cache=False)
        return float(we @ E + wf @ F.ravel())

    eps = 1e-6
    fd = np.zeros_like(sh)
    for i in range(sh.size):
        p, m = sh.copy(), sh.copy()
        p[i] += eps
        m[i] -= eps
        fd[i] = (readout(p, hd[0]) - readout(m, hd[0])) / (2 * eps)
    assert O.rel_vec_error(gs, fd) < 1e-6
    fdh = np.zeros_like(hd[0])
    for i in range(fdh.size):
        p, m = hd[0].copy(), hd[0].copy()
        p[i] += eps
        m[i] -= eps
        fdh[i] = (readout(sh, p) - readout(sh, m)) / (2 * eps)
    assert O.rel_vec_error(gh[0], fdh) < 1e-6


def test_adamw_scalar_kat(oracle):
    """SPEC.md:410-418 example: t=1, g=1, lr=1e-3, wd=0 -> step ~ -1e-3."""
    p = np.array([0.5])
    g = np.array([1.0])
    m = np.zeros(1)
    v = np.zeros(1)
    oracle.adamw(p, g, m, v, 1, lr=1e-3, wd=0.0)
    assert abs((p[0] - 0.5) - (-1e-3 / (1 + 1e-8))) < 1e-15
    p2 = np.array([0.5]); m2 = np.zeros(1); v2 = np.zeros(1)
    oracle.adamw(p2, np.zeros(1), m2, v2, 1, wd=0.0)
    assert p2[0] == 0.5


def test_trainer_restatement_tracks_reference_trainer(oracle):
    """5 steps of the FP64 restated trainer vs the reference-based CPU trainer (FP32)."""
    g = load("train_ref.npz")
    h = hyper_of(g)
    sh = oracle.init_block(h, 7, -1)
    hd = {k: oracle.init_block(h, 7, k) for k in (0, 1)}
    b = O.batch_from_samples({k: g[k] for k in ("n_atoms", "species", "pos", "forces", "energy", "dsid")}, 5.0,
                             oracle.build_edges)
    st = {k: (np.zeros_like(v), np.zeros_like(v)) for k, v in [("s", sh)] + [(f"h{k}", hd[k]) for k in hd]}
    losses = []
    for t in range(1, 6):
        E, F, c = oracle.forward(h, sh, hd, b)
        L, dE, dF = oracle.loss(b, E, F)
        losses.append(L)
        gs, gh = oracle.backward(h, sh, hd, b, c, dE, dF)
        oracle.adamw(sh, gs, *st["s"], t)
        for k in hd:
            oracle.adamw(hd[k], gh[k], *st[f"h{k}"], t)
    assert np.allclose(losses, g["losses"], rtol=1e-5, atol=0)
    assert O.rel_vec_error(sh, g["shared_after"]) < 1e-5
