"""Periodic neighbour lists.  The reference has no PBC
(hmtl/graph.hpp:44-76), so the pin is the builder's FP64 brute
force over lattice images (oracle ho_build_edges_pbc), itself checked here
against analytic coordination shells; the GPU cell list must reproduce its
edge set and images bit-exactly, and the model on periodic edges must match
the FP64 oracle (rel 1e-4) with the per-edge image shifts."""
import numpy as np
import pytest

import oracle as O

import paper_2506_21788_b200 as P

TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    O.build(ref=False)


@pytest.fixture(scope="module")
def orc():
    return O.Oracle()


def lattice(kind, a):
    if kind == "sc":
        return np.eye(3) * a, np.zeros((1, 3))
    if kind == "fcc":
        return np.eye(3) * a, np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]]) * a
    if kind == "bcc":
        return np.eye(3) * a, np.array([[0, 0, 0], [.5, .5, .5]]) * a


@pytest.mark.parametrize("kind,a,rc,coord", [
    ("sc", 3.0, 3.05, 6), ("sc", 3.0, 4.3, 18), ("sc", 3.0, 5.3, 26),
    ("fcc", 4.0, 2.9, 12), ("fcc", 4.0, 4.05, 18), ("bcc", 3.0, 2.7, 8), ("bcc", 3.0, 3.05, 14)])
def test_oracle_coordination_shells(orc, kind, a, rc, coord):
    cell, pos = lattice(kind, a)
    go, eo, dst, src, img, sh = orc.build_edges_pbc([len(pos)], pos, cell[None], rc)
    deg = np.bincount(dst, minlength=len(pos))
    assert np.all(deg == coord), deg


def random_crystals(rng, G, nmin, nmax, side, tilt=0.0, outside=False):
    n = rng.integers(nmin, nmax + 1, size=G)
    cells, pos = [], []
    for g in range(G):
        A = np.diag(rng.uniform(0.9, 1.1, 3) * side)
        A[1, 0] += tilt * side
        A[2, 0] += 0.5 * tilt * side
        A[2, 1] += 0.3 * tilt * side
        f = rng.random((n[g], 3))
        if outside:  # unwrapped coordinates: some atoms one or two cells away
            f += rng.integers(-2, 3, size=(n[g], 3))
        pos.append(f @ A)
        cells.append(A)
    return n.astype(np.int32), np.concatenate(pos), np.array(cells)


def test_oracle_pbc_reduces_to_open_boundaries_in_large_cells(orc):
    rng = np.random.default_rng(3)
    n, pos, cells = random_crystals(rng, 3, 10, 20, 6.0)
    big = cells * 10.0  # every periodic image is > rc away
    go, eo, dst, src, img, sh = orc.build_edges_pbc(n, pos, big, 5.0)
    go2, eo2, dst2, src2 = orc.build_edges(n, pos, 5.0)
    assert np.array_equal(dst, dst2) and np.array_equal(src, src2) and not img.any()


def samples_for(n, pos, species_seed=0):
    rng = np.random.default_rng(species_seed)
    G, N = len(n), int(n.sum())
    return P.Samples(n, rng.integers(0, 20, N).astype(np.uint8), pos, rng.normal(size=(N, 3)),
                     rng.normal(size=G), np.zeros(G, np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg4", "triclinic", "unwrapped", "small_cells"])
def test_gpu_cell_list_bit_exact_vs_oracle(orc, case):
    rng = np.random.default_rng({"cfg4": 1, "triclinic": 2, "unwrapped": 3, "small_cells": 4}[case])
    if case == "cfg4":  # cfg4-class: 200-300 atoms, rc 6, dense
        n, pos, cells = random_crystals(rng, 4, 200, 300, 14.5)
    elif case == "triclinic":
        n, pos, cells = random_crystals(rng, 4, 60, 120, 11.0, tilt=0.35)
    elif case == "unwrapped":
        n, pos, cells = random_crystals(rng, 3, 40, 90, 10.0, tilt=0.2, outside=True)
    else:  # cells smaller than the cutoff: several images of every atom, self images
        n, pos, cells = random_crystals(rng, 5, 1, 6, 3.5, tilt=0.1)
    rc = 6.0
    go, eo, dst, src, img, sh = orc.build_edges_pbc(n, pos, cells, rc)
    s = samples_for(n, pos)
    hp = P.ModelHyper(20, 2, 32, 32, 3, 1, rc)
    m = P.ModelT(hp, 7, [0], caps=P.Caps(len(n) + 1, int(n.sum()) + 8, len(dst) + 64))
    m.upload_pbc(s, cells)
    P.lib().hmtl_build_batch(m.ctx, None)
    b = m.edges()
    assert np.array_equal(b.edge_dst, dst) and np.array_equal(b.edge_src, src)
    assert np.array_equal(m.edge_images(), img)
    assert np.array_equal(b.edge_offset, eo)
    m.close()


@pytest.mark.gpu
def test_gpu_periodic_forward_backward_parity(orc):
    rng = np.random.default_rng(7)
    n, pos, cells = random_crystals(rng, 3, 30, 60, 8.0, tilt=0.2, outside=True)
    rc = 5.0
    s = samples_for(n, pos, 1)
    go, eo, dst, src, img, sh = orc.build_edges_pbc(n, pos, cells, rc)
    hp = P.ModelHyper(20, 2, 32, 32, 3, 1, rc)
    oh = O.Hyper(20, 2, 32, 32, 3, 1, rc)
    m = P.ModelT(hp, 7, [0], caps=P.Caps(len(n) + 1, int(n.sum()) + 8, len(dst) + 64))
    m.upload_pbc(s, cells)
    P.lib().hmtl_build_batch(m.ctx, None)
    pred = m.forward()
    b = dict(n_atoms=s.n_atoms, species=s.species, pos=s.positions, forces=s.forces, energy=s.energy,
             dsid=s.dataset_id, graph_offset=go, edge_offset=eo, edge_dst=dst, edge_src=src, edge_shift=sh)
    sh0 = orc.init_block(oh, 7, -1)
    heads = {0: orc.init_block(oh, 7, 0)}
    E, F, cache = orc.forward(oh, sh0, heads, b)
    assert O.rel_vec_error(pred.energy_per_atom, E) < TOL
    assert O.rel_vec_error(pred.forces, F) < TOL
    L, dE, dF = orc.loss(b, E, F)
    assert abs(m.loss() - L) / abs(L) < TOL
    g = m.backward()
    gs, gh = orc.backward(oh, sh0, heads, b, cache, dE, dF)
    assert O.rel_vec_error(g.shared, gs) < TOL and O.rel_vec_error(g.heads[0], gh[0]) < TOL
    # a lattice translation of any atom changes nothing but the edge images
    pos2 = pos.copy()
    pos2[5] += cells[0][1] - 2 * cells[0][2]
    m.upload_pbc(samples_for(n, pos2, 1), cells)
    P.lib().hmtl_build_batch(m.ctx, None)
    pred2 = m.forward()
    assert O.rel_vec_error(pred2.energy_per_atom, pred.energy_per_atom) < 1e-5
    assert O.rel_vec_error(pred2.forces, pred.forces) < 1e-5
    m.close()


@pytest.mark.gpu
def test_cfg4_shaped_periodic_crystal_parity(orc):
    """BASELINE config 4 shape (parity case): a periodic inorganic cell of ~200
    atoms at rc 6 with dense neighbour lists, hidden 256 (layers reduced to 2 so
    the FP64 oracle stays fast); forward and gradients within 1e-4."""
    rng = np.random.default_rng(44)
    n, pos, cells = random_crystals(rng, 1, 200, 200, 13.0, tilt=0.15)
    rc = 6.0
    s = samples_for(n, pos, 4)
    go, eo, dst, src, img, sh = orc.build_edges_pbc(n, pos, cells, rc)
    assert len(dst) / n.sum() > 60  # dense: ~80 neighbours per atom
    hp = P.ModelHyper(20, 2, 256, 256, 3, 1, rc)
    oh = O.Hyper(20, 2, 256, 256, 3, 1, rc)
    m = P.ModelT(hp, 7, [0], caps=P.Caps(2, int(n.sum()) + 8, len(dst) + 64))
    m.upload_pbc(s, cells)
    P.lib().hmtl_build_batch(m.ctx, None)
    b_ = m.edges()
    assert np.array_equal(b_.edge_dst, dst) and np.array_equal(b_.edge_src, src)
    pred = m.forward()
    b = dict(n_atoms=s.n_atoms, species=s.species, pos=s.positions, forces=s.forces, energy=s.energy,
             dsid=s.dataset_id, graph_offset=go, edge_offset=eo, edge_dst=dst, edge_src=src, edge_shift=sh)
    sh0 = orc.init_block(oh, 7, -1)
    heads = {0: orc.init_block(oh, 7, 0)}
    E, F, cache = orc.forward(oh, sh0, heads, b)
    assert O.rel_vec_error(pred.energy_per_atom, E) < TOL
    assert O.rel_vec_error(pred.forces, F) < TOL
    L, dE, dF = orc.loss(b, E, F)
    m.loss()
    g = m.backward()
    gs, gh = orc.backward(oh, sh0, heads, b, cache, dE, dF)
    assert O.rel_vec_error(g.shared, gs) < TOL and O.rel_vec_error(g.heads[0], gh[0]) < TOL
    m.close()
