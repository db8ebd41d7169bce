"""ctypes bindings for the CHECKERS (test infrastructure only).

* ``Oracle`` -- oracle/_build/libhmtl_oracle.so, the plain-C FP64 restatement
  (oracle/hmtl_oracle.c) of the reference hot path.
* ``Ref``    -- oracle/_ref/libhmtl_ref.so, the unmodified reference compiled
  from /root/reference by oracle/Makefile (+ oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhmtl_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhmtl_ref.so")


def build(ref: bool = True) -> None:
    """Compile the C restatement (always) and the reference (when its sources exist)."""
    targets = ["oracle"] + (["ref"] if ref and os.path.isdir("/root/reference/proj") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


@dataclass
class Hyper:
    """ModelHyper, /root/reference/proj/include/hmtl/model.hpp:17-37."""

    n_species: int = 20
    layers: int = 2
    hidden: int = 32
    head_width: int = 32
    head_depth: int = 3
    n_heads: int = 1
    cutoff: float = 5.0


class _CHyper(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_species", "layers", "hidden", "head_width", "head_depth", "n_heads")] + [
        ("cutoff", C.c_double)
    ]


def _chyper(h: Hyper) -> _CHyper:
    return _CHyper(h.n_species, h.layers, h.hidden, h.head_width, h.head_depth, h.n_heads, h.cutoff)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


_D = C.c_double
_I = C.c_int
_U8 = C.c_uint8


class _CBatch(C.Structure):
    _fields_ = [
        ("G", C.c_int), ("N", C.c_int), ("E", C.c_int),
        ("graph_offset", C.POINTER(_I)), ("edge_offset", C.POINTER(_I)),
        ("pos", C.POINTER(_D)), ("species", C.POINTER(_U8)),
        ("edge_dst", C.POINTER(_I)), ("edge_src", C.POINTER(_I)),
        ("dataset_id", C.POINTER(_U8)), ("edge_shift", C.POINTER(_D)),
    ]


class _CCache(C.Structure):
    _fields_ = [(n, C.POINTER(_D)) for n in
                ("h_in", "z1", "a1", "z2", "m", "agg", "vz1", "vp1", "h_final", "pooled", "ez", "fz", "s")]


CACHE_KEYS = ("h_in", "z1", "a1", "z2", "m", "agg", "vz1", "vp1", "h_final", "pooled", "ez", "fz", "s")


def alloc_cache(h: Hyper, G: int, N: int, E: int) -> dict:
    L, H, W, D = h.layers, h.hidden, h.head_width, h.head_depth
    shp = {
        "h_in": (L, N, H), "z1": (L, E, H), "a1": (L, E, H), "z2": (L, E, H), "m": (L, E, H),
        "agg": (L, N, H), "vz1": (L, N, H), "vp1": (L, N, H), "h_final": (N, H), "pooled": (G, H),
        "ez": (D, G, W), "fz": (D, E, W), "s": (E,),
    }
    return {k: np.zeros(v, np.float64) for k, v in shp.items()}


def _ccache(c: dict) -> _CCache:
    return _CCache(*[_p(c[k], _D) for k in CACHE_KEYS])


def batch_from_samples(s: dict, cutoff: float, edges_fn) -> dict:
    """Adds graph_offset/edge_offset/edge_dst/edge_src to a sample dict."""
    b = dict(s)
    n = np.ascontiguousarray(s["n_atoms"], np.int32)
    go, eo, dst, src = edges_fn(n, np.ascontiguousarray(s["pos"], np.float64), cutoff, s.get("species"))
    b.update(graph_offset=go, edge_offset=eo, edge_dst=dst, edge_src=src)
    return b


class Oracle:
    """FP64 C restatement (oracle/hmtl_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.ho_shared_size.restype = C.c_size_t
        L.ho_head_size.restype = C.c_size_t
        L.ho_seed_stream.restype = C.c_uint64
        L.ho_seed_stream.argtypes = [C.c_uint64, C.c_uint64]
        L.ho_init_block.argtypes = [C.POINTER(_CHyper), C.c_uint64, C.c_int, C.POINTER(_D)]
        L.ho_build_edges.restype = C.c_long
        L.ho_build_edges.argtypes = [C.c_int, C.POINTER(_I), C.POINTER(_D), C.c_double] + [C.POINTER(_I)] * 4
        L.ho_forward.argtypes = [C.POINTER(_CHyper), C.POINTER(_D), C.POINTER(C.POINTER(_D)),
                                 C.POINTER(_CBatch), C.POINTER(_CCache), C.POINTER(_D), C.POINTER(_D)]
        L.ho_backward.argtypes = [C.POINTER(_CHyper), C.POINTER(_D), C.POINTER(C.POINTER(_D)),
                                  C.POINTER(_CBatch), C.POINTER(_CCache), C.POINTER(_D), C.POINTER(_D),
                                  C.POINTER(_D), C.POINTER(C.POINTER(_D))]
        L.ho_loss.restype = C.c_double
        L.ho_loss.argtypes = [C.POINTER(_CBatch)] + [C.POINTER(_D)] * 4 + [C.c_double, C.c_double] + [C.POINTER(_D)] * 2
        L.ho_adamw.argtypes = [C.POINTER(_D)] * 4 + [C.c_size_t, C.c_long] + [C.c_double] * 5
        L.ho_layout_entries.restype = C.c_int
        L.ho_layout_entries.argtypes = [C.POINTER(_CHyper), C.c_int, C.c_int, C.c_char_p, C.c_size_t,
                                        C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]

    def shared_size(self, h: Hyper) -> int:
        return self.lib.ho_shared_size(C.byref(_chyper(h)))

    def head_size(self, h: Hyper) -> int:
        return self.lib.ho_head_size(C.byref(_chyper(h)))

    def layout(self, h: Hyper, shared: bool) -> list:
        ch = _chyper(h)
        n = self.lib.ho_layout_entries(C.byref(ch), int(shared), -1, None, 0, None, None, None)
        out = []
        for i in range(n):
            nm = C.create_string_buffer(64)
            r, c, o = C.c_size_t(), C.c_size_t(), C.c_size_t()
            self.lib.ho_layout_entries(C.byref(ch), int(shared), i, nm, 64, C.byref(r), C.byref(c), C.byref(o))
            out.append((nm.value.decode(), r.value, c.value, o.value))
        return out

    def init_block(self, h: Hyper, seed: int, which: int) -> np.ndarray:
        n = self.shared_size(h) if which < 0 else self.head_size(h)
        out = np.zeros(n, np.float64)
        self.lib.ho_init_block(C.byref(_chyper(h)), seed, which, _p(out, _D))
        return out

    def build_edges_pbc(self, n_atoms, pos, cells, cutoff):
        """Periodic neighbour list (builder's FP64 oracle): returns
        graph_offset, edge_offset, dst, src, img [E][3], shift [E][3]."""
        L = self.lib
        L.ho_build_edges_pbc.restype = C.c_long
        L.ho_build_edges_pbc.argtypes = [C.c_int, C.POINTER(_I), C.POINTER(_D), C.POINTER(_D), C.c_double] + \
            [C.POINTER(_I)] * 5 + [C.POINTER(_D)]
        n = np.ascontiguousarray(n_atoms, np.int32)
        p = np.ascontiguousarray(pos, np.float64).reshape(-1)
        cl = np.ascontiguousarray(cells, np.float64).reshape(-1)
        G = len(n)
        E = L.ho_build_edges_pbc(G, _p(n, _I), _p(p, _D), _p(cl, _D), cutoff, None, None, None, None, None, None)
        if E < 0:
            raise ValueError("pbc: empty graph" if E == -1 else "pbc: image range exceeded")
        go, eo = np.zeros(G + 1, np.int32), np.zeros(G + 1, np.int32)
        dst, src = np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1), np.int32)
        img, sh = np.zeros((max(E, 1), 3), np.int32), np.zeros((max(E, 1), 3), np.float64)
        L.ho_build_edges_pbc(G, _p(n, _I), _p(p, _D), _p(cl, _D), cutoff, _p(go, _I), _p(eo, _I), _p(dst, _I),
                             _p(src, _I), _p(img, _I), _p(sh, _D))
        return go, eo, dst[:E], src[:E], img[:E], sh[:E]

    def build_edges(self, n_atoms, pos, cutoff, species=None):
        n = np.ascontiguousarray(n_atoms, np.int32)
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        G = len(n)
        E = self.lib.ho_build_edges(G, _p(n, _I), _p(pos, _D), cutoff, None, None, None, None)
        if E < 0:
            raise ValueError("build_batch: empty graph rejected")
        go = np.zeros(G + 1, np.int32)
        eo = np.zeros(G + 1, np.int32)
        dst = np.zeros(max(E, 1), np.int32)
        src = np.zeros(max(E, 1), np.int32)
        self.lib.ho_build_edges(G, _p(n, _I), _p(pos, _D), cutoff, _p(go, _I), _p(eo, _I), _p(dst, _I), _p(src, _I))
        return go, eo, dst[:E], src[:E]

    def _cbatch(self, b: dict):
        keep = dict(
            go=np.ascontiguousarray(b["graph_offset"], np.int32), eo=np.ascontiguousarray(b["edge_offset"], np.int32),
            pos=np.ascontiguousarray(b["pos"], np.float64).reshape(-1), sp=np.ascontiguousarray(b["species"], np.uint8),
            dst=np.ascontiguousarray(b["edge_dst"], np.int32), src=np.ascontiguousarray(b["edge_src"], np.int32),
            ds=np.ascontiguousarray(b["dsid"], np.uint8),
        )
        if b.get("edge_shift") is not None:
            keep["sh"] = np.ascontiguousarray(b["edge_shift"], np.float64).reshape(-1)
        cb = _CBatch(len(keep["ds"]), len(keep["sp"]), len(keep["dst"]), _p(keep["go"], _I), _p(keep["eo"], _I),
                     _p(keep["pos"], _D), _p(keep["sp"], _U8), _p(keep["dst"], _I), _p(keep["src"], _I),
                     _p(keep["ds"], _U8), _p(keep["sh"], _D) if "sh" in keep else None)
        return cb, keep

    @staticmethod
    def _heads(h: Hyper, heads: dict):
        arrs = [np.ascontiguousarray(heads[k], np.float64) if k in heads else None for k in range(h.n_heads)]
        ptrs = (C.POINTER(_D) * h.n_heads)(*[_p(a, _D) if a is not None else None for a in arrs])
        return ptrs, arrs

    def forward(self, h: Hyper, shared, heads: dict, b: dict, cache: bool = True):
        cb, keep = self._cbatch(b)
        G, N, E = cb.G, cb.N, cb.E
        c = alloc_cache(h, G, N, E) if cache else None
        cc = _ccache(c) if cache else None
        sh = np.ascontiguousarray(shared, np.float64)
        hp, keep_h = self._heads(h, heads)
        energy = np.zeros(G, np.float64)
        forces = np.zeros(3 * N, np.float64)
        rc = self.lib.ho_forward(C.byref(_chyper(h)), _p(sh, _D), hp, C.byref(cb),
                                 C.byref(cc) if cache else None, _p(energy, _D), _p(forces, _D))
        if rc != 0:
            raise RuntimeError(f"oracle forward rc={rc}")
        return energy, forces.reshape(N, 3), c

    def backward(self, h: Hyper, shared, heads: dict, b: dict, cache: dict, dE, dF):
        cb, keep = self._cbatch(b)
        sh = np.ascontiguousarray(shared, np.float64)
        hp, keep_h = self._heads(h, heads)
        gs = np.zeros(self.shared_size(h), np.float64)
        gh = {k: np.zeros(self.head_size(h), np.float64) for k in heads}
        ghp = (C.POINTER(_D) * h.n_heads)(*[_p(gh[k], _D) if k in gh else None for k in range(h.n_heads)])
        cc = _ccache(cache)
        dE = np.ascontiguousarray(dE, np.float64)
        dF = np.ascontiguousarray(dF, np.float64).reshape(-1)
        rc = self.lib.ho_backward(C.byref(_chyper(h)), _p(sh, _D), hp, C.byref(cb), C.byref(cc), _p(dE, _D),
                                  _p(dF, _D), _p(gs, _D), ghp)
        if rc != 0:
            raise RuntimeError(f"oracle backward rc={rc}")
        return gs, gh

    def loss(self, b: dict, energy, forces, w_e=1.0, w_f=1.0):
        cb, keep = self._cbatch(b)
        e = np.ascontiguousarray(energy, np.float64)
        f = np.ascontiguousarray(forces, np.float64).reshape(-1)
        le = np.ascontiguousarray(b["energy"], np.float64)
        lf = np.ascontiguousarray(b["forces"], np.float64).reshape(-1)
        dE = np.zeros(cb.G, np.float64)
        dF = np.zeros(3 * cb.N, np.float64)
        L = self.lib.ho_loss(C.byref(cb), _p(e, _D), _p(f, _D), _p(le, _D), _p(lf, _D), w_e, w_f, _p(dE, _D), _p(dF, _D))
        return L, dE, dF

    def adamw(self, p, g, m, v, step, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01):
        for a in (p, g, m, v):
            assert a.dtype == np.float64 and a.flags.c_contiguous
        self.lib.ho_adamw(_p(p, _D), _p(g, _D), _p(m, _D), _p(v, _D), p.size, step, lr, b1, b2, eps, wd)


class _RefCache(_CCache):
    pass


class Ref:
    """The unmodified reference (oracle/_ref/libhmtl_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_default5_spec.argtypes = [C.c_int, C.POINTER(_U8), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I),
                                        C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), C.POINTER(C.c_uint64)]
        L.ref_dataset_generate.restype = C.c_void_p
        L.ref_dataset_generate.argtypes = [C.c_int, C.POINTER(_U8), C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_double, C.POINTER(_D), C.c_uint64, C.c_int64, C.c_uint64]
        for f in ("ref_dataset_count", "ref_dataset_atoms"):
            getattr(L, f).restype = C.c_uint64
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_dataset_export.argtypes = [C.c_void_p, C.POINTER(_I), C.POINTER(_U8), C.POINTER(_D), C.POINTER(_D),
                                         C.POINTER(_D), C.POINTER(_U8)]
        L.ref_dataset_free.argtypes = [C.c_void_p]
        L.ref_build_batch.restype = C.c_long
        L.ref_build_batch.argtypes = [C.c_int, C.POINTER(_I), C.POINTER(_U8), C.POINTER(_D), C.c_double] + [C.POINTER(_I)] * 4
        L.ref_model_new.restype = C.c_void_p
        L.ref_model_new.argtypes = [C.POINTER(_CHyper), C.c_uint64, C.POINTER(_I), C.c_int, C.c_int]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_shared_size.restype = C.c_uint64
        L.ref_model_shared_size.argtypes = [C.c_void_p]
        L.ref_model_head_size.restype = C.c_uint64
        L.ref_model_head_size.argtypes = [C.c_void_p]
        L.ref_model_get_block.argtypes = [C.c_void_p, C.c_int, C.POINTER(_D)]
        L.ref_model_set_block.argtypes = [C.c_void_p, C.c_int, C.POINTER(_D)]
        L.ref_forward_backward.argtypes = [C.c_void_p, C.c_int, C.POINTER(_I), C.POINTER(_U8), C.POINTER(_D),
                                           C.POINTER(_U8), C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), C.POINTER(_D),
                                           C.POINTER(_D), C.POINTER(C.POINTER(_D)), C.POINTER(_CCache)]
        L.ref_trainer_new.restype = C.c_void_p
        L.ref_trainer_new.argtypes = [C.c_void_p] + [C.c_double] * 7
        L.ref_trainer_free.argtypes = [C.c_void_p]
        L.ref_train_step.restype = C.c_double
        L.ref_train_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(_I), C.POINTER(_U8), C.POINTER(_D),
                                     C.POINTER(_D), C.POINTER(_D), C.POINTER(_U8), C.c_int]

    def err(self) -> str:
        return self.lib.ref_last_error().decode()

    def write_samples(self, path: str, dataset_id: int, aligned: int, s: dict) -> None:
        """The reference's write_sample_file (src/sample_io.cpp:104-120)."""
        L = self.lib
        L.ref_write_samples.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_I), C.POINTER(_U8),
                                        C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), C.POINTER(_U8)]
        n = np.ascontiguousarray(s["n_atoms"], np.int32)
        sp = np.ascontiguousarray(s["species"], np.uint8)
        pos = np.ascontiguousarray(s["pos"], np.float64)
        en = np.ascontiguousarray(s["energy"], np.float64)
        fo = np.ascontiguousarray(s["forces"], np.float64)
        ds = np.ascontiguousarray(s["dsid"], np.uint8)
        if L.ref_write_samples(path.encode(), dataset_id, aligned, len(n), _p(n, _I), _p(sp, _U8), _p(pos, _D),
                               _p(en, _D), _p(fo, _D), _p(ds, _U8)) != 0:
            raise RuntimeError(self.err())

    def shuffle_epoch(self, counts: dict, n_groups: int, replicas: int, mode: int, seed: int, b_local: int,
                      rank: int):
        """The reference's shuffle_epoch (src/datastore.cpp:47-97) for one rank of Mesh{n_groups, replicas}."""
        L = self.lib
        L.ref_shuffle_epoch.restype = C.c_long
        L.ref_shuffle_epoch.argtypes = [C.POINTER(_U8), C.POINTER(C.c_uint64), C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_uint64, C.c_int, C.c_int, C.POINTER(_U8), C.POINTER(C.c_uint64),
                                        C.POINTER(_I)]
        ids = np.array(sorted(counts), np.uint8)
        cnt = np.array([counts[int(k)] for k in ids], np.uint64)
        cap = int(cnt.sum()) + 1
        ds, ix, st = np.zeros(cap, np.uint8), np.zeros(cap, np.uint64), _I()
        n = L.ref_shuffle_epoch(_p(ids, _U8), cnt.ctypes.data_as(C.POINTER(C.c_uint64)), len(ids), n_groups,
                                replicas, mode, seed, b_local, rank, _p(ds, _U8),
                                ix.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(st))
        if n < 0:
            raise RuntimeError(self.err())
        return st.value, ds[:n], ix[:n]

    def align_energies(self, files, ref_id: int, out_files):
        """The reference's align_energies (src/dataset.cpp:306-356): ({id: offsets[20]}, skipped)."""
        L = self.lib
        L.ref_align_energies.argtypes = [C.POINTER(C.c_char_p), C.c_int, C.c_int, C.POINTER(C.c_char_p),
                                         C.POINTER(_U8), C.POINTER(_D), C.POINTER(_U8), C.POINTER(_I)]
        n = len(files)
        fa = (C.c_char_p * n)(*[f.encode() for f in files])
        oa = (C.c_char_p * n)(*[f.encode() for f in out_files])
        ids, off = np.zeros(n, np.uint8), np.zeros(n * 20, np.float64)
        sk, ns = np.zeros(n * 20 + 1, np.uint8), _I()
        if L.ref_align_energies(fa, n, ref_id, oa, _p(ids, _U8), _p(off, _D), _p(sk, _U8), C.byref(ns)) != 0:
            raise RuntimeError(self.err())
        return {int(i): off[20 * j:20 * j + 20] for j, i in enumerate(ids)}, list(sk[:ns.value])

    def make_partition(self, counts: dict, n_groups: int, replicas: int, mode: int) -> dict:
        """The reference's make_partition (src/datastore.cpp:25-45) on Mesh{n_groups, replicas}:
        {dataset id: [(serving rank, begin, end), ...]}."""
        L = self.lib
        L.ref_make_partition.restype = C.c_long
        L.ref_make_partition.argtypes = [C.POINTER(_U8), C.POINTER(C.c_uint64), C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(_I), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(_I)]
        ids = np.array(sorted(counts), np.uint8)
        cnt = np.array([counts[int(k)] for k in ids], np.uint64)
        cap = len(ids) * n_groups * replicas + 1
        sv, b, e, ns = np.zeros(cap, np.int32), np.zeros(cap, np.uint64), np.zeros(cap, np.uint64), np.zeros(len(ids), np.int32)
        u64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
        n = L.ref_make_partition(_p(ids, _U8), u64(cnt), len(ids), n_groups, replicas, mode, _p(sv, _I), u64(b), u64(e),
                                 _p(ns, _I))
        if n < 0:
            raise RuntimeError(self.err())
        out, k = {}, 0
        for i, d in enumerate(ids):
            out[int(d)] = [(int(sv[k + j]), int(b[k + j]), int(e[k + j])) for j in range(ns[i])]
            k += ns[i]
        return out

    def default5_spec(self, i: int) -> dict:
        el = (_U8 * 32)()
        ne, nmin, nmax = _I(), _I(), _I()
        a, s = _D(), _D()
        mu = (_D * 20)()
        cnt = C.c_uint64()
        if self.lib.ref_default5_spec(i, el, C.byref(ne), C.byref(nmin), C.byref(nmax), C.byref(a), C.byref(s), mu,
                                      C.byref(cnt)) != 0:
            raise IndexError(i)
        return dict(dataset_id=i, elements=list(el[: ne.value]), n_min=nmin.value, n_max=nmax.value, alpha=a.value,
                    sigma=s.value, mu=list(mu), count=cnt.value)

    def generate(self, spec: dict, seed: int, count: int | None = None) -> dict:
        el = np.ascontiguousarray(spec["elements"], np.uint8)
        mu = np.ascontiguousarray(spec.get("mu", [0.0] * 20), np.float64)
        h = self.lib.ref_dataset_generate(spec["dataset_id"], _p(el, _U8), len(el), spec["n_min"], spec["n_max"],
                                          spec["alpha"], spec["sigma"], _p(mu, _D),
                                          count if count is not None else spec["count"],
                                          spec.get("structure_seed", -1), seed)
        if not h:
            raise RuntimeError(self.err())
        G = self.lib.ref_dataset_count(h)
        N = self.lib.ref_dataset_atoms(h)
        out = dict(n_atoms=np.zeros(G, np.int32), species=np.zeros(N, np.uint8), pos=np.zeros((N, 3)),
                   forces=np.zeros((N, 3)), energy=np.zeros(G), dsid=np.zeros(G, np.uint8))
        self.lib.ref_dataset_export(h, _p(out["n_atoms"], _I), _p(out["species"], _U8), _p(out["pos"], _D),
                                    _p(out["forces"], _D), _p(out["energy"], _D), _p(out["dsid"], _U8))
        self.lib.ref_dataset_free(h)
        return out

    def build_edges(self, n_atoms, pos, cutoff, species=None):
        n = np.ascontiguousarray(n_atoms, np.int32)
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        sp = np.zeros(int(n.sum()), np.uint8) if species is None else np.ascontiguousarray(species, np.uint8)
        G = len(n)
        E = self.lib.ref_build_batch(G, _p(n, _I), _p(sp, _U8), _p(pos, _D), cutoff, None, None, None, None)
        if E < 0:
            raise ValueError(self.err())
        go = np.zeros(G + 1, np.int32)
        eo = np.zeros(G + 1, np.int32)
        dst = np.zeros(max(E, 1), np.int32)
        src = np.zeros(max(E, 1), np.int32)
        self.lib.ref_build_batch(G, _p(n, _I), _p(sp, _U8), _p(pos, _D), cutoff, _p(go, _I), _p(eo, _I), _p(dst, _I),
                                 _p(src, _I))
        return go, eo, dst[:E], src[:E]


class RefModel:
    """ModelT<double|float> of the reference."""

    def __init__(self, ref: Ref, h: Hyper, seed: int, owned: list, dbl: bool = True):
        self.ref, self.h, self.owned = ref, h, list(owned)
        o = np.ascontiguousarray(owned, np.int32)
        self.ptr = ref.lib.ref_model_new(C.byref(_chyper(h)), seed, _p(o, _I), len(o), int(dbl))
        if not self.ptr:
            raise RuntimeError(ref.err())

    def __del__(self):
        if getattr(self, "ptr", None):
            self.ref.lib.ref_model_free(self.ptr)

    def save_checkpoint(self, path: str) -> None:
        """The reference's save_checkpoint (src/model_io.cpp:62-84); FP64 model with all heads."""
        L = self.ref.lib
        L.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
        if L.ref_save_checkpoint(self.ptr, path.encode()) != 0:
            raise RuntimeError(self.ref.err())

    def block(self, which: int) -> np.ndarray:
        n = self.ref.lib.ref_model_shared_size(self.ptr) if which < 0 else self.ref.lib.ref_model_head_size(self.ptr)
        out = np.zeros(n, np.float64)
        if self.ref.lib.ref_model_get_block(self.ptr, which, _p(out, _D)) != 0:
            raise RuntimeError(self.ref.err())
        return out

    def set_block(self, which: int, v) -> None:
        v = np.ascontiguousarray(v, np.float64)
        self.ref.lib.ref_model_set_block(self.ptr, which, _p(v, _D))

    def run(self, b: dict, E: int, dE=None, dF=None, cache: bool = True):
        """forward (and backward when dE/dF given); b needs n_atoms/species/pos/dsid."""
        n = np.ascontiguousarray(b["n_atoms"], np.int32)
        sp = np.ascontiguousarray(b["species"], np.uint8)
        pos = np.ascontiguousarray(b["pos"], np.float64).reshape(-1)
        ds = np.ascontiguousarray(b["dsid"], np.uint8)
        G, N = len(n), len(sp)
        energy, forces = np.zeros(G), np.zeros(3 * N)
        c = alloc_cache(self.h, G, N, E) if cache else None
        cc = _ccache(c) if cache else None
        gs = gh = None
        ghp = None
        if dE is not None:
            dE = np.ascontiguousarray(dE, np.float64)
            dF = np.ascontiguousarray(dF, np.float64).reshape(-1)
            gs = np.zeros(self.ref.lib.ref_model_shared_size(self.ptr))
            gh = {k: np.zeros(self.ref.lib.ref_model_head_size(self.ptr)) for k in self.owned}
            ghp = (C.POINTER(_D) * self.h.n_heads)(*[_p(gh[k], _D) if k in gh else None for k in range(self.h.n_heads)])
        rc = self.ref.lib.ref_forward_backward(self.ptr, G, _p(n, _I), _p(sp, _U8), _p(pos, _D), _p(ds, _U8),
                                               _p(dE, _D), _p(dF, _D), _p(energy, _D), _p(forces, _D),
                                               _p(gs, _D), ghp, C.byref(cc) if cache else None)
        if rc != 0:
            raise RuntimeError(f"reference rc={rc}: {self.ref.err()}")
        return dict(energy=energy, forces=forces.reshape(N, 3), cache=c, g_shared=gs, g_heads=gh)


class RefTrainer:
    """Reference CPU training step (ModelT<float> + SPEC loss/AdamW), thread-parallel."""

    def __init__(self, ref: Ref, model: RefModel, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01, w_e=1.0, w_f=1.0):
        self.ref, self.model = ref, model
        self.ptr = ref.lib.ref_trainer_new(model.ptr, lr, b1, b2, eps, wd, w_e, w_f)
        if not self.ptr:
            raise RuntimeError(ref.err())

    def __del__(self):
        if getattr(self, "ptr", None):
            self.ref.lib.ref_trainer_free(self.ptr)

    def step(self, s: dict, threads: int = 1) -> float:
        n = np.ascontiguousarray(s["n_atoms"], np.int32)
        sp = np.ascontiguousarray(s["species"], np.uint8)
        pos = np.ascontiguousarray(s["pos"], np.float64).reshape(-1)
        f = np.ascontiguousarray(s["forces"], np.float64).reshape(-1)
        e = np.ascontiguousarray(s["energy"], np.float64)
        ds = np.ascontiguousarray(s["dsid"], np.uint8)
        L = self.ref.lib.ref_train_step(self.ptr, len(n), _p(n, _I), _p(sp, _U8), _p(pos, _D), _p(f, _D), _p(e, _D),
                                        _p(ds, _U8), threads)
        if L != L:
            raise RuntimeError(self.ref.err())
        return L


def rel_vec_error(a, b, floor=1e-12) -> float:
    """||a-b|| / max(||a||, ||b||, floor) -- tests/oracles.hpp:62-74 of the reference."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), np.linalg.norm(b), floor))
