"""Python mirror of the reference's C++ API for the hot path, backed by the
B200 C ABI (include/hmtl_b200.h).  Names follow the reference:

  ModelHyper            hmtl/model.hpp:17-37
  shared_layout/head_layout  hmtl/model.hpp:56-90
  ModelT (float)        hmtl/model.hpp:155-242  (forward :196-197, backward :198-201)
  build_batch           hmtl/graph.hpp:46-83    (runs on the GPU)
  PredictionT / GradientBufferT  hmtl/model.hpp:92-115
  classify_regime / memory_footprint  hmtl/model.hpp:246-263

Host numpy arrays in, host numpy arrays out; the device keeps the batch, the
forward cache and the parameters.  Errors raise HmtlError with the
reference's ErrorCode.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import CCaps, CHyper, CSamples, CTrainCfg, HmtlError, check, lib

__all__ = [
    "ModelHyper", "Samples", "Caps", "ModelT", "PredictionT", "GradientBufferT", "GraphBatch", "TrainConfig",
    "shared_layout", "head_layout", "classify_regime", "memory_footprint", "HmtlError",
]


@dataclass
class ModelHyper:
    n_species: int = 20
    layers: int = 2
    hidden: int = 32
    head_width: int = 32
    head_depth: int = 3
    n_heads: int = 1
    cutoff: float = 5.0

    @staticmethod
    def paper_preset(n_heads: int) -> "ModelHyper":
        """4 x 866 encoder, 3-layer 889-unit heads (hmtl/model.hpp:28-36)."""
        return ModelHyper(layers=4, hidden=866, head_width=889, head_depth=3, n_heads=n_heads)

    def c(self) -> CHyper:
        return CHyper(self.n_species, self.layers, self.hidden, self.head_width, self.head_depth, self.n_heads,
                      self.cutoff)


def _layout(hp: ModelHyper, shared: bool):
    ch = hp.c()
    n = lib().hmtl_layout_entry(C.byref(ch), int(shared), -1, None, 0, None, None, None)
    out = []
    for i in range(n):
        nm = C.create_string_buffer(64)
        r, c, o = C.c_size_t(), C.c_size_t(), C.c_size_t()
        lib().hmtl_layout_entry(C.byref(ch), int(shared), i, nm, 64, C.byref(r), C.byref(c), C.byref(o))
        out.append((nm.value.decode(), r.value, c.value, o.value))
    return out


def shared_layout(hp: ModelHyper):
    return _layout(hp, True)


def head_layout(hp: ModelHyper):
    return _layout(hp, False)


def classify_regime(p_s: int, p_h: int, n_h: int) -> int:
    """1, 2, 3 = ParallelRegime::case1..case3 (hmtl/model.hpp:249-255)."""
    r = lib().hmtl_classify_regime(p_s, p_h, n_h)
    if r < 0:
        raise HmtlError(-r, lib().hmtl_last_error().decode())
    return r


def memory_footprint(p_s: int, p_h: int, n_h: int, mode: str) -> int:
    return lib().hmtl_memory_footprint(p_s, p_h, n_h, {"serial": 0, "base": 1, "taskpar": 2}[mode])


@dataclass
class Samples:
    """A list of AtomisticSample (hmtl/graph.hpp:13-21), struct-of-arrays."""

    n_atoms: np.ndarray  # [G] int32
    species: np.ndarray  # [N] uint8
    positions: np.ndarray  # [N,3] float64
    forces: np.ndarray  # [N,3] float64
    energy: np.ndarray  # [G] float64 (energy per atom)
    dataset_id: np.ndarray  # [G] uint8

    def __post_init__(self):
        self.n_atoms = np.ascontiguousarray(self.n_atoms, np.int32)
        self.species = np.ascontiguousarray(self.species, np.uint8)
        self.positions = np.ascontiguousarray(self.positions, np.float64).reshape(-1, 3)
        self.forces = np.ascontiguousarray(self.forces, np.float64).reshape(-1, 3)
        self.energy = np.ascontiguousarray(self.energy, np.float64)
        self.dataset_id = np.ascontiguousarray(self.dataset_id, np.uint8)

    @property
    def G(self) -> int:
        return len(self.n_atoms)

    @property
    def N(self) -> int:
        return len(self.species)

    def edge_bound(self) -> int:
        n = self.n_atoms.astype(np.int64)
        return int((n * (n - 1)).sum())

    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.n_atoms)]).astype(np.int64)

    def take(self, idx) -> "Samples":
        off = self.offsets()
        idx = list(idx)
        cat = lambda a: np.concatenate([a[off[i]:off[i + 1]] for i in idx]) if idx else a[:0]
        return Samples(self.n_atoms[idx], cat(self.species), cat(self.positions), cat(self.forces), self.energy[idx],
                       self.dataset_id[idx])

    @staticmethod
    def concat(parts) -> "Samples":
        return Samples(*[np.concatenate([getattr(p, f) for p in parts]) for f in
                         ("n_atoms", "species", "positions", "forces", "energy", "dataset_id")])

    def as_c(self) -> CSamples:
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        return CSamples(self.G, self.N, P(self.n_atoms, C.c_int), P(self.species, C.c_uint8),
                        P(self.positions, C.c_double), P(self.forces, C.c_double), P(self.energy, C.c_double),
                        P(self.dataset_id, C.c_uint8))


@dataclass
class Caps:
    max_graphs: int
    max_nodes: int
    max_edges: int

    @staticmethod
    def for_samples(s: Samples, slack: float = 1.0) -> "Caps":
        return Caps(max(1, int(s.G * slack)), max(1, int(s.N * slack)), max(1, int(s.edge_bound() * slack)))

    @staticmethod
    def for_periodic(s: Samples, cells, cutoff: float, slack: float = 1.5) -> "Caps":
        """Edge capacity for periodic structures, where the image
        count, not n(n-1), bounds a row: n x (density x 4/3 pi rc^3 x slack + 16)."""
        cells = np.asarray(cells, np.float64).reshape(s.G, 3, 3)
        vol = np.abs(np.linalg.det(cells))
        n = s.n_atoms.astype(np.float64)
        per_atom = n / np.maximum(vol, 1e-12) * (4.0 / 3.0) * np.pi * cutoff ** 3
        e = int(np.ceil((n * (per_atom * slack + 16.0)).sum()))
        return Caps(max(1, s.G), max(1, s.N), max(1, e, s.edge_bound()))

    def covers(self, s: Samples) -> bool:
        return s.G <= self.max_graphs and s.N <= self.max_nodes and s.edge_bound() <= self.max_edges

    def union(self, o: "Caps") -> "Caps":
        return Caps(max(self.max_graphs, o.max_graphs), max(self.max_nodes, o.max_nodes),
                    max(self.max_edges, o.max_edges))


@dataclass
class PredictionT:
    energy_per_atom: np.ndarray  # [G]
    forces: np.ndarray  # [N,3]


@dataclass
class GradientBufferT:
    shared: np.ndarray
    heads: dict = field(default_factory=dict)


@dataclass
class GraphBatch:
    """Edge view of GraphBatchT (hmtl/graph.hpp:27-42) as built on the device."""

    n_graphs: int
    graph_offset: np.ndarray
    edge_offset: np.ndarray
    edge_dst: np.ndarray
    edge_src: np.ndarray

    def n_edges(self) -> int:
        return len(self.edge_dst)


@dataclass
class TrainConfig:
    """TrainConfig + AdamW defaults."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01
    w_energy: float = 1.0
    w_force: float = 1.0
    use_graph: bool = True

    def c(self) -> CTrainCfg:
        return CTrainCfg(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, self.w_energy, self.w_force,
                         int(self.use_graph))


class ModelT:
    """ModelT<float> living on one B200 (hmtl/model.hpp:155-242)."""

    def __init__(self, hp: ModelHyper, seed: int, owned_heads, caps: Caps | None = None, device: int = 0):
        self.hp, self.seed, self.device = hp, int(seed), int(device)
        self.owned = sorted(int(k) for k in owned_heads)
        self.caps = caps or Caps(64, 4096, 1 << 17)
        self._ctx = None
        self._create(self.caps)
        self._G = self._N = 0

    # ---- context management
    def _create(self, caps: Caps, params=None):
        ctx = C.c_void_p()
        owned = (C.c_int * len(self.owned))(*self.owned)
        cc = CCaps(caps.max_graphs, caps.max_nodes, caps.max_edges)
        check(lib().hmtl_ctx_create(self.device, C.byref(self.hp.c()), self.seed, owned, len(self.owned),
                                    C.byref(cc), C.byref(ctx)))
        self._ctx = ctx
        self.caps = caps
        if params is not None:
            for k, v in params.items():
                check(lib().hmtl_set_block(self._ctx, k, _fp(v)))

    def reserve(self, s: Samples, need: Caps | None = None) -> None:
        """Grow the device capacities to fit `s` (or `need`) in place (hmtl_ctx_reserve):
        parameters, AdamW state, step counter and an attached communicator all survive."""
        if need is None:
            if self.caps.covers(s):
                return
            need = Caps.for_samples(s, 1.25)
        elif self.caps.union(need) == self.caps:
            return
        caps = self.caps.union(need)
        check(lib().hmtl_ctx_reserve(self._ctx, C.byref(CCaps(caps.max_graphs, caps.max_nodes, caps.max_edges))))
        self.caps = caps

    def close(self):
        if self._ctx is not None:
            lib().hmtl_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self):
        return self._ctx

    # ---- census (hmtl/model.hpp:169-180)
    def shared_size(self) -> int:
        return lib().hmtl_shared_size(C.byref(self.hp.c()))

    def head_size(self) -> int:
        return lib().hmtl_head_size(C.byref(self.hp.c()))

    def owns_head(self, k: int) -> bool:
        return k in self.owned

    def n_owned_heads(self) -> int:
        return len(self.owned)

    def param_count(self) -> int:
        return self.shared_size() + len(self.owned) * self.head_size()

    # ---- blocks (hmtl/model.hpp:182-187)
    def _get(self, fn, which, n):
        out = np.zeros(n, np.float32)
        check(fn(self._ctx, which, _fp(out)))
        return out

    def shared_block(self) -> np.ndarray:
        return self._get(lib().hmtl_get_block, -1, self.shared_size())

    def head_block(self, k: int) -> np.ndarray:
        return self._get(lib().hmtl_get_block, k, self.head_size())

    def set_shared_block(self, v) -> None:
        check(lib().hmtl_set_block(self._ctx, -1, _fp(np.ascontiguousarray(v, np.float32))))

    def set_head_block(self, k: int, v) -> None:
        check(lib().hmtl_set_block(self._ctx, k, _fp(np.ascontiguousarray(v, np.float32))))

    # ---- step pieces
    def upload(self, s: Samples, stream=None) -> None:
        self.reserve(s)
        self._keep = s
        check(lib().hmtl_batch_upload(self._ctx, C.byref(s.as_c()), stream))
        self._G, self._N = s.G, s.N

    def upload_pbc(self, s: Samples, cells, stream=None) -> None:
        """Periodic batch: samples + lattice cells[G][3][3] (rows a1..a3)."""
        self.reserve(s, Caps.for_samples(s, 1.25).union(Caps.for_periodic(s, cells, self.hp.cutoff)))
        self._keep = s
        self._cells = np.ascontiguousarray(cells, np.float64).reshape(s.G, 9)
        check(lib().hmtl_batch_upload_pbc(self._ctx, C.byref(s.as_c()),
                                          self._cells.ctypes.data_as(C.POINTER(C.c_double)), stream))
        self._G, self._N = s.G, s.N

    def edge_images(self) -> np.ndarray:
        """[E][3] lattice image of every edge's source (zeros for open boundaries)."""
        E = C.c_int()
        check(lib().hmtl_batch_edges(self._ctx, C.byref(E), None, None, None))
        img = np.zeros((max(E.value, 1), 3), np.int32)
        check(lib().hmtl_batch_edge_images(self._ctx, _ip(img)))
        return img[:E.value]

    def build_batch(self, s: Samples) -> GraphBatch:
        """build_batch<float> on the device; returns the edge view (syncs)."""
        self.upload(s)
        check(lib().hmtl_build_batch(self._ctx, None))
        return self.edges()

    def edges(self) -> GraphBatch:
        E = C.c_int()
        check(lib().hmtl_batch_edges(self._ctx, C.byref(E), None, None, None))
        dst = np.zeros(max(E.value, 1), np.int32)
        src = np.zeros(max(E.value, 1), np.int32)
        eo = np.zeros(self._G + 1, np.int32)
        check(lib().hmtl_batch_edges(self._ctx, C.byref(E), _ip(dst), _ip(src), _ip(eo)))
        go = np.concatenate([[0], np.cumsum(self._keep.n_atoms)]).astype(np.int32)
        return GraphBatch(self._G, go, eo, dst[:E.value], src[:E.value])

    def forward(self, s: Samples | None = None) -> PredictionT:
        """ModelT::forward (hmtl/model.hpp:338-488).  With `s`, uploads and builds the batch first."""
        if s is not None:
            self.upload(s)
            check(lib().hmtl_build_batch(self._ctx, None))
        check(lib().hmtl_forward(self._ctx, None))
        e = np.zeros(self._G, np.float32)
        f = np.zeros(3 * self._N, np.float32)
        check(lib().hmtl_predictions(self._ctx, _fp(e), _fp(f)))
        return PredictionT(e, f.reshape(-1, 3))

    def predictions(self) -> PredictionT:
        """PredictionT of the last forward on the device (e.g. inside a train step), no recompute."""
        e = np.zeros(self._G, np.float32)
        f = np.zeros(3 * self._N, np.float32)
        check(lib().hmtl_predictions(self._ctx, _fp(e), _fp(f)))
        return PredictionT(e, f.reshape(-1, 3))

    def loss(self, w_energy: float = 1.0, w_force: float = 1.0) -> float:
        """SPEC loss on the device (also leaves dE/dF on the device for backward(None, None))."""
        check(lib().hmtl_loss(self._ctx, w_energy, w_force, None))
        L = C.c_float()
        check(lib().hmtl_read_loss(self._ctx, C.byref(L)))
        return float(L.value)

    def backward(self, d_energy=None, d_forces=None) -> GradientBufferT:
        """ModelT::backward (hmtl/model.hpp:490-625) for the last forward."""
        if d_energy is None:
            check(lib().hmtl_backward(self._ctx, None, None, None))
        else:
            de = np.ascontiguousarray(d_energy, np.float32)
            df = np.ascontiguousarray(d_forces, np.float32).reshape(-1)
            if de.size != self._G or df.size != 3 * self._N:
                raise HmtlError(1, "model: upstream shape mismatch")
            check(lib().hmtl_backward(self._ctx, _fp(de), _fp(df), None))
        return self.grads()

    def grads(self) -> GradientBufferT:
        g = GradientBufferT(self._get(lib().hmtl_get_grad, -1, self.shared_size()))
        for k in self.owned:
            g.heads[k] = self._get(lib().hmtl_get_grad, k, self.head_size())
        return g

    def debug(self, name: str, layer: int = 0) -> np.ndarray:
        n = C.c_size_t()
        check(lib().hmtl_debug_fetch(self._ctx, name.encode(), layer, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.float32)
        check(lib().hmtl_debug_fetch(self._ctx, name.encode(), layer, _fp(out), out.size, C.byref(n)))
        return out[: n.value]

    def comm_init(self, uid: bytes, world: int, rank: int) -> None:
        """NCCL world communicator + per-head sub-groups (hmtl/mesh.hpp:322-334)."""
        check(lib().hmtl_comm_init(self._ctx, (C.c_uint8 * 128)(*bytes(uid)), world, rank))

    def save_checkpoint(self, path: str, with_optimizer: bool = True) -> None:
        """HMTP checkpoint (save_checkpoint, src/model_io.cpp:62-84) + AdamW resume section."""
        check(lib().hmtl_checkpoint_save(self._ctx, path.encode(), int(with_optimizer)))

    def load_checkpoint(self, path: str) -> None:
        """Load the owned blocks (+ optimizer state when present) from a full HMTP checkpoint."""
        check(lib().hmtl_checkpoint_load(self._ctx, path.encode()))

    def adamw(self, cfg: TrainConfig) -> None:
        check(lib().hmtl_adamw(self._ctx, C.byref(cfg.c()), None))

    def post_loss(self, slot: int, stream=None) -> None:
        """Enqueue the D2H read of this step's loss into pinned ring slot `slot` (no sync)."""
        check(lib().hmtl_loss_post(self._ctx, slot, stream))

    def wait_loss(self, slot: int) -> float:
        """Block on ring slot `slot` only; the loss posted there (errors as read_loss)."""
        L = C.c_float()
        check(lib().hmtl_loss_wait(self._ctx, slot, C.byref(L)))
        return float(L.value)

    def train_step(self, s: Samples | None, cfg: TrainConfig, stream=None, read_loss: bool = True):
        """train_step -- uploads `s` (if given) and runs the whole
        stream-ordered step; returns the loss (syncs) when read_loss."""
        if s is not None:
            self.upload(s, stream)
        check(lib().hmtl_train_step(self._ctx, C.byref(cfg.c()), stream))
        if read_loss:
            L = C.c_float()
            check(lib().hmtl_read_loss(self._ctx, C.byref(L)))
            return float(L.value)
        return None


def nbr_build(s: Samples, cutoff: float, device: int = 0) -> dict:
    """build_batch's edge set without a model (hmtl_nbr_build; hmtl/graph.hpp:46-83):
    edge_dst/edge_src[E], edge_offset[G+1], row_ptr[N+1] (CSR by dst), rev[E]."""
    E = C.c_int()
    cap = s.edge_bound()
    out = {"edge_dst": np.zeros(max(cap, 1), np.int32), "edge_src": np.zeros(max(cap, 1), np.int32),
           "edge_offset": np.zeros(s.G + 1, np.int32), "row_ptr": np.zeros(s.N + 1, np.int32),
           "rev": np.zeros(max(cap, 1), np.int32)}
    check(lib().hmtl_nbr_build(device, C.byref(s.as_c()), float(cutoff), cap, C.byref(E), _ip(out["edge_dst"]),
                               _ip(out["edge_src"]), _ip(out["edge_offset"]), _ip(out["row_ptr"]), _ip(out["rev"])))
    for k in ("edge_dst", "edge_src", "rev"):
        out[k] = out[k][:E.value]
    return out


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


# ---------------------------------------------------------------- data plane
def align_energies(files, ref_dataset_id: int, out_files, device: int = 0):
    """align_energies (hmtl/dataset.hpp:62-70, src/dataset.cpp:263-356) on the GPU:
    HMTD files in, aligned HMTD files out; returns ({dataset id: offsets[20]}, skipped)."""
    n = len(files)
    fa = (C.c_char_p * n)(*[str(f).encode() for f in files])
    oa = (C.c_char_p * len(out_files))(*[str(f).encode() for f in out_files])
    if len(out_files) != n:
        raise ValueError("align: out file count mismatch")
    ids, off = np.zeros(n, np.uint8), np.zeros(n * 20, np.float64)
    sk, ns = np.zeros(n * 20 + 1, np.uint8), C.c_int()
    check(lib().hmtl_align_energies(device, fa, n, ref_dataset_id, oa, ids.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    off.ctypes.data_as(C.POINTER(C.c_double)), n,
                                    sk.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(ns)))
    return {int(i): off[20 * j:20 * j + 20] for j, i in enumerate(ids)}, [int(x) for x in sk[:ns.value]]


def comm_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 makes it; ship it to the others out of band)."""
    b = (C.c_uint8 * 128)()
    check(lib().hmtl_comm_unique_id(b))
    return bytes(b)


def shard_range(count: int, n: int, i: int) -> tuple:
    """balanced_split(count, n)[i] (src/datastore.cpp:11-23): [begin, end)."""
    b, e = C.c_uint64(), C.c_uint64()
    check(lib().hmtl_shard_range(count, n, i, C.byref(b), C.byref(e)))
    return b.value, e.value


def make_partition(counts: dict, world: int, mode: str = "base", members: dict | None = None) -> dict:
    """make_partition (src/datastore.cpp:25-45): {dataset id: (count, serving ranks
    ascending, [(begin, end) per serving rank])}.  base: every rank serves every
    dataset; taskpar: the dataset's head group (members[id], any placement)."""
    out = {}
    for d in sorted(counts):
        if mode == "taskpar":
            if members is None or d not in members:
                raise ValueError(f"taskpar: dataset id {d} has no head sub-group")
            serving = sorted(int(r) for r in members[d])
        else:
            serving = list(range(world))
        out[int(d)] = (int(counts[d]), serving, [shard_range(int(counts[d]), len(serving), i) for i in range(len(serving))])
    return out


def epoch_plan(mode: str, counts: dict, world: int, seed: int, b_local: int, rank: int,
               members: dict | None = None):
    """shuffle_epoch (hmtl/datastore.hpp:48-75, src/datastore.cpp:47-97) for one rank:
    returns (steps, ds[steps*b_local] u8, idx[steps*b_local] u64).  mode 'base' or
    'taskpar'; members = {dataset id: ascending serving ranks} (taskpar)."""
    ids = np.array(sorted(counts), np.uint8)
    cnt = np.array([counts[int(k)] for k in ids], np.uint64)
    m = 1 if mode == "taskpar" else 0
    if m:
        if members is None:
            raise ValueError("taskpar needs the serving group of every dataset")
        off = np.zeros(len(ids) + 1, np.int32)
        flat = []
        for i, k in enumerate(ids):
            grp = sorted(int(r) for r in members.get(int(k), []))
            flat += grp
            off[i + 1] = off[i] + len(grp)
        mem = np.array(flat or [0], np.int32)
        mp, op = _ip(mem), _ip(off)
    else:
        mp = op = None
    u8 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint8))
    u64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
    steps, n = C.c_int(), C.c_size_t()
    check(lib().hmtl_epoch_plan(m, u8(ids), u64(cnt), len(ids), mp, op, world, seed, b_local, rank, None, None, 0,
                                C.byref(steps), C.byref(n)))
    ds = np.zeros(max(n.value, 1), np.uint8)
    ix = np.zeros(max(n.value, 1), np.uint64)
    check(lib().hmtl_epoch_plan(m, u8(ids), u64(cnt), len(ids), mp, op, world, seed, b_local, rank, u8(ds), u64(ix),
                                ds.size, C.byref(steps), C.byref(n)))
    return steps.value, ds[: n.value], ix[: n.value]


def checkpoint_write(path: str, hp: ModelHyper, shared, heads) -> None:
    """save_checkpoint (src/model_io.cpp:62-84) of host blocks (FP32, stored as f64)."""
    sh = np.ascontiguousarray(shared, np.float32)
    hd = np.ascontiguousarray(np.concatenate([np.asarray(h, np.float32) for h in heads]), np.float32)
    check(lib().hmtl_checkpoint_write(path.encode(), C.byref(hp.c()), _fp(sh), _fp(hd), None))


def checkpoint_hyper(path: str) -> tuple:
    """(ModelHyper, has_optimizer_section) of an HMTP file."""
    h, o = CHyper(), C.c_int()
    check(lib().hmtl_checkpoint_read_hyper(path.encode(), C.byref(h), C.byref(o)))
    return ModelHyper(h.n_species, h.layers, h.hidden, h.head_width, h.head_depth, h.n_heads, h.cutoff), bool(o.value)


def hmtd_write(path: str, dataset_id: int, aligned: int, s: Samples) -> None:
    """write_sample_file (src/sample_io.cpp:104-120), byte-compatible with the reference."""
    check(lib().hmtl_hmtd_write(path.encode(), dataset_id, aligned, C.byref(s.as_c())))


def hmtd_header(path: str) -> tuple:
    """read_sample_header (src/sample_io.cpp:173-189): (dataset_id, aligned, count)."""
    d, a, n = C.c_uint8(), C.c_uint8(), C.c_uint64()
    check(lib().hmtl_hmtd_read_header(path.encode(), C.byref(d), C.byref(a), C.byref(n)))
    return int(d.value), int(a.value), int(n.value)


class SampleStore:
    """Device-resident sample pool (DataStore, hmtl/datastore.hpp:77-115): upload once,
    bind a plan's batch into a model's arena by a device gather."""

    def __init__(self, pool: Samples | None, device: int = 0, _handle=None):
        self._pool = pool  # keeps the host arrays alive for the upload
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        check(lib().hmtl_store_create(device, C.byref(pool.as_c()), C.byref(h)))
        self._h = h

    @staticmethod
    def from_hmtd(paths, device: int = 0) -> "SampleStore":
        """HMTD files straight to HBM: CRC check and parse on the GPU."""
        arr = (C.c_char_p * len(paths))(*[p.encode() for p in paths])
        h = C.c_void_p()
        check(lib().hmtl_store_from_hmtd(device, arr, len(paths), C.byref(h)))
        return SampleStore(None, device, _handle=h)

    def counts(self) -> dict:
        n = C.c_int()
        check(lib().hmtl_store_counts(self._h, None, None, 0, C.byref(n)))
        ids = np.zeros(max(n.value, 1), np.uint8)
        cnt = np.zeros(max(n.value, 1), np.uint64)
        check(lib().hmtl_store_counts(self._h, ids.ctypes.data_as(C.POINTER(C.c_uint8)),
                                      cnt.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
        return {int(i): int(c) for i, c in zip(ids[: n.value], cnt[: n.value])}

    def bind(self, model: "ModelT", ds, idx, stream=None) -> None:
        ds = np.ascontiguousarray(ds, np.uint8)
        idx = np.ascontiguousarray(idx, np.uint64)
        check(lib().hmtl_store_bind(model.ctx, self._h, ds.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    idx.ctypes.data_as(C.POINTER(C.c_uint64)), len(ds), stream))
        self._bound(model)

    @staticmethod
    def sharded(model: "ModelT", shard: Samples, partition: dict) -> "SampleStore":
        """This rank's shard only (DataStore, src/datastore.cpp:99-145); collective
        over the model's communicator.  partition = {dataset id: (count, serving
        ranks ascending)}; shard = the samples of this rank's ranges, dataset by
        dataset in ascending id order (see shard_range)."""
        ids = np.array(sorted(partition), np.uint8)
        counts = np.array([partition[int(i)][0] for i in ids], np.uint64)
        mem = [list(partition[int(i)][1]) for i in ids]
        members = np.array([r for m in mem for r in m] or [0], np.int32)
        off = np.zeros(len(ids) + 1, np.int32)
        off[1:] = np.cumsum([len(m) for m in mem])
        h = C.c_void_p()
        check(lib().hmtl_store_create_sharded(model.ctx, C.byref(shard.as_c()), ids.ctypes.data_as(C.POINTER(C.c_uint8)),
                                              counts.ctypes.data_as(C.POINTER(C.c_uint64)),
                                              members.ctypes.data_as(C.POINTER(C.c_int)),
                                              off.ctypes.data_as(C.POINTER(C.c_int)), len(ids), C.byref(h)))
        st = SampleStore(None, model.device, _handle=h)
        st._pool = shard
        return st

    def download(self) -> Samples:
        """The pool back in host memory (store order)."""
        G, N = C.c_int(), C.c_longlong()
        check(lib().hmtl_store_shape(self._h, C.byref(G), C.byref(N)))
        na, sp = np.zeros(G.value, np.int32), np.zeros(N.value, np.uint8)
        pos, frc = np.zeros(3 * N.value), np.zeros(3 * N.value)
        en, ds = np.zeros(G.value), np.zeros(G.value, np.uint8)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        u8 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint8))
        check(lib().hmtl_store_download(self._h, na.ctypes.data_as(C.POINTER(C.c_int)), u8(sp), dp(pos), dp(frc),
                                        dp(en), u8(ds)))
        return Samples(na, sp, pos, frc, en, ds)

    def align(self, ref_dataset_id: int):
        """Energy alignment of the pool in place (align_energies, src/dataset.cpp:306-356):
        returns ({dataset id: offsets[20]}, skipped elements)."""
        n = len(self.counts())
        ids, off = np.zeros(n, np.uint8), np.zeros(n * 20, np.float64)
        sk, ns = np.zeros(n * 20 + 1, np.uint8), C.c_int()
        check(lib().hmtl_store_align(self._h, ref_dataset_id, ids.ctypes.data_as(C.POINTER(C.c_uint8)),
                                     off.ctypes.data_as(C.POINTER(C.c_double)), n,
                                     sk.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(ns)))
        return {int(i): off[20 * j:20 * j + 20] for j, i in enumerate(ids)}, [int(x) for x in sk[:ns.value]]

    def fetch(self, model: "ModelT", plan_ds, plan_idx, stream=None) -> None:
        """fetch_samples(plan, step) (src/datastore.cpp:192-248): plan_ds/plan_idx are
        this step's [world, b_local] plan rows of every rank; collective."""
        ds = np.ascontiguousarray(plan_ds, np.uint8)
        idx = np.ascontiguousarray(plan_idx, np.uint64)
        check(lib().hmtl_store_fetch(model.ctx, self._h, ds.ctypes.data_as(C.POINTER(C.c_uint8)),
                                     idx.ctypes.data_as(C.POINTER(C.c_uint64)), ds.shape[-1], stream))
        self._bound(model)

    @staticmethod
    def _bound(model: "ModelT") -> None:  # the model's host view of the batch the device now holds
        G, N = C.c_int(), C.c_int()
        check(lib().hmtl_batch_shape(model.ctx, C.byref(G), C.byref(N)))
        model._G, model._N = G.value, N.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().hmtl_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
