"""Synthetic multi-source inputs and MTL-par placement (host side).

* default5_specs / generate_dataset: the reference's Morse-potential source
  generator (src/dataset.cpp:106-161, 213-239) re-stated in C++ inside
  libhmtl_b200 (csrc/host.cpp); bit-identical to the reference
  (tests/test_host.py checks it against tests/golden/dataset5.npz).
* head_placement: head -> rank shares for uneven meshes (generalises the
  N x M Mesh of hmtl/mesh.hpp:21-31).
* mtl_batch_counts: per-head structure counts of a per-GPU batch with a fixed
  edge budget per head "unit" (load imbalance).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import CSpec, check, lib
from .model import Samples


@dataclass
class DatasetSpec:
    dataset_id: int = 0
    elements: list = field(default_factory=lambda: [0, 1, 2, 3])
    n_min: int = 2
    n_max: int = 8
    alpha: float = 1.0
    sigma: float = 0.0
    mu: list = field(default_factory=lambda: [0.0] * 20)
    count: int = 1000
    structure_seed: int = -1
    name: str = ""

    def c(self) -> CSpec:
        s = CSpec()
        s.dataset_id = self.dataset_id
        s.n_elements = len(self.elements)
        for i, e in enumerate(self.elements):
            s.elements[i] = e
        s.n_min, s.n_max, s.alpha, s.sigma = self.n_min, self.n_max, self.alpha, self.sigma
        for i in range(20):
            s.mu[i] = self.mu[i]
        s.count, s.structure_seed = self.count, self.structure_seed
        return s


DEFAULT5_NAMES = ["organicA", "organicB", "organicC", "inorganicA", "inorganicB"]


def default5_specs() -> list:
    out = []
    for i in range(5):
        s = CSpec()
        check(lib().hmtl_default5_spec(i, C.byref(s)))
        out.append(DatasetSpec(s.dataset_id, list(s.elements[: s.n_elements]), s.n_min, s.n_max, s.alpha, s.sigma,
                               list(s.mu), s.count, s.structure_seed, DEFAULT5_NAMES[i]))
    return out


def generate_dataset(spec: DatasetSpec, seed: int, count: int | None = None) -> Samples:
    if count is not None:
        spec = DatasetSpec(**{**spec.__dict__, "count": count})
    cs = spec.c()
    G, N = C.c_int(), C.c_int()
    check(lib().hmtl_generate(C.byref(cs), seed, C.byref(G), C.byref(N), None, None, None, None, None, None))
    n = np.zeros(G.value, np.int32)
    sp = np.zeros(N.value, np.uint8)
    pos = np.zeros((N.value, 3))
    f = np.zeros((N.value, 3))
    e = np.zeros(G.value)
    ds = np.zeros(G.value, np.uint8)
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    check(lib().hmtl_generate(C.byref(cs), seed, C.byref(G), C.byref(N), P(n, C.c_int), P(sp, C.c_uint8),
                              P(pos, C.c_double), P(f, C.c_double), P(e, C.c_double), P(ds, C.c_uint8)))
    return Samples(n, sp, pos, f, e, ds)


def head_placement(world: int, weights) -> np.ndarray:
    """share[r, k]: fraction of head k's global per-step batch served by rank r."""
    w = np.ascontiguousarray(weights, np.float64)
    out = np.zeros((world, len(w)), np.float64)
    check(lib().hmtl_head_placement(world, len(w), w.ctypes.data_as(C.POINTER(C.c_double)),
                                    out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


# MTL-par weak-scaling mix: per-GPU edge budget split
# over heads in proportion to GPUS_PER_HEAD_AT_8 = {1,1,1,2,3}.
GPUS_PER_HEAD_AT_8 = (1, 1, 1, 2, 3)


def mtl_batch_counts(edges_per_struct, unit_edges: float, weights=GPUS_PER_HEAD_AT_8, multiple=(1, 1, 1, 2, 3)):
    """Per-head structure counts n_k of the 1-GPU batch: n_k ~ w_k * unit / (8 * e_k),
    rounded to a multiple that keeps every rank's share integral at 1/2/4/8 GPUs."""
    total_w = float(sum(weights))
    out = []
    for k, e in enumerate(edges_per_struct):
        n = weights[k] * unit_edges / (total_w * e)
        m = multiple[k] if k < len(multiple) else 1
        m = 3 if weights[k] == 3 else m
        out.append(max(m, int(round(n / m)) * m))
    return out
