"""Training-step parity: SPEC loss/AdamW on the B200 vs the
FP64 oracle trainer, including the 100-step loss curve (north star)."""
import numpy as np
import pytest

import oracle as O

import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data
from paper_2506_21788_b200.model import Samples

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    O.build(ref=False)
    if P.lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")


def batch(counts, seed=1234):
    specs = data.default5_specs()
    return Samples.concat([data.generate_dataset(sp, seed + k, count=c) for k, (sp, c) in enumerate(zip(specs, counts)) if c])


class OracleTrainer:
    def __init__(self, o, oh, seed, owned):
        self.o, self.oh = o, oh
        self.sh = o.init_block(oh, seed, -1)
        self.heads = {k: o.init_block(oh, seed, k) for k in owned}
        self.st = {"s": (np.zeros_like(self.sh), np.zeros_like(self.sh))}
        for k in owned:
            self.st[k] = (np.zeros_like(self.heads[k]), np.zeros_like(self.heads[k]))
        self.t = 0

    def step(self, s: Samples, cutoff=5.0):
        b = O.batch_from_samples(dict(n_atoms=s.n_atoms, species=s.species, pos=s.positions, forces=s.forces,
                                      energy=s.energy, dsid=s.dataset_id), cutoff, self.o.build_edges)
        E, F, c = self.o.forward(self.oh, self.sh, self.heads, b)
        L, dE, dF = self.o.loss(b, E, F)
        gs, gh = self.o.backward(self.oh, self.sh, self.heads, b, c, dE, dF)
        self.t += 1
        self.o.adamw(self.sh, gs, *self.st["s"], self.t)
        for k in self.heads:
            self.o.adamw(self.heads[k], gh[k], *self.st[k], self.t)
        return L


def test_adamw_one_step_matches_oracle():
    o = O.Oracle()
    hp = P.ModelHyper(20, 2, 16, 16, 3, 5, 5.0)
    oh = O.Hyper(20, 2, 16, 16, 3, 5, 5.0)
    s = batch((3, 2, 2, 1, 1))
    m = P.ModelT(hp, 7, range(5))
    ot = OracleTrainer(o, oh, 7, range(5))
    cfg = P.TrainConfig(use_graph=False)
    L = m.train_step(s, cfg)
    Lo = ot.step(s)
    assert abs(L - Lo) / Lo < 1e-5
    assert O.rel_vec_error(m.shared_block(), ot.sh) < 1e-6
    for k in range(5):
        assert O.rel_vec_error(m.head_block(k), ot.heads[k]) < 1e-6


def test_cuda_graph_step_equals_eager_step():
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    s1, s2 = batch((3, 2, 2, 1, 1), 1), batch((4, 1, 3, 2, 1), 2)
    caps = P.Caps.for_samples(s1).union(P.Caps.for_samples(s2))
    res = []
    for g in (False, True):
        m = P.ModelT(hp, 7, range(5), caps=caps)
        cfg = P.TrainConfig(use_graph=g)
        Ls = [m.train_step(x, cfg) for x in (s1, s2, s1, s2)]
        res.append((Ls, m.shared_block()))
        m.close()
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])


def test_pipelined_steps_equal_synchronous_steps():
    """The trainer-loop pipeline (double-buffered pinned staging: batch i+1 packed and
    launched before step i's loss is read from the pinned result ring) gives the
    synchronous loop's losses and parameters bit for bit."""
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    xs = [batch((3, 2, 2, 1, 1), 1), batch((4, 1, 3, 2, 1), 2), batch((2, 2, 2, 2, 2), 3)]
    caps = P.Caps.for_samples(xs[0]).union(P.Caps.for_samples(xs[1])).union(P.Caps.for_samples(xs[2]))
    cfg = P.TrainConfig(use_graph=True)
    seq = xs * 3
    m = P.ModelT(hp, 7, range(5), caps=caps)
    sync = [m.train_step(x, cfg) for x in seq]
    ref = m.shared_block()
    m.close()
    m = P.ModelT(hp, 7, range(5), caps=caps)
    piped = []
    for i, x in enumerate(seq):
        m.train_step(x, cfg, read_loss=False)
        m.post_loss(i)
        if i:
            piped.append(m.wait_loss(i - 1))
    piped.append(m.wait_loss(len(seq) - 1))
    assert piped == sync
    assert np.array_equal(m.shared_block(), ref)
    m.close()


def test_loss_curve_100_steps_matches_fp64_oracle():
    """Loss curves over 100 steps (north star).  Same batches, same seeds; the
    FP32 B200 path vs the FP64 restatement of the reference."""
    o = O.Oracle()
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    oh = O.Hyper(20, 2, 32, 32, 3, 5, 5.0)
    batches = [batch((3, 2, 2, 1, 1), 100 + i) for i in range(4)]
    caps = P.Caps(64, 1024, max(b.edge_bound() for b in batches))
    m = P.ModelT(hp, 7, range(5), caps=caps)
    ot = OracleTrainer(o, oh, 7, range(5))
    cfg = P.TrainConfig(use_graph=True)
    g, ref = [], []
    for step in range(100):
        b = batches[step % 4]
        g.append(m.train_step(b, cfg))
        ref.append(ot.step(b))
    g, ref = np.array(g), np.array(ref)
    relerr = np.abs(g - ref) / np.abs(ref)
    print("max rel loss deviation over 100 steps:", relerr.max(), "final", g[-1], ref[-1])
    assert ref[-1] < ref[0]  # it trains
    assert relerr.max() < 1e-3
    assert O.rel_vec_error(m.shared_block(), ot.sh) < 1e-3


@pytest.mark.parametrize("H,L", [(128, 3), (64, 2)])
def test_fused_graph_steps_match_oracle(H, L, monkeypatch):
    """Steps 2+ of a graph-mode trainer run the fused node chains (chain.cuh),
    the side-stream weight gradients and the batched B images: every step's
    loss and the parameters after 3 AdamW steps must match the FP64 trainer
    (FP32 tolerance), and the unfused single-stream engine closely."""
    o = O.Oracle()
    hp = P.ModelHyper(20, L, H, H, 3, 5, 5.0)
    oh = O.Hyper(20, L, H, H, 3, 5, 5.0)
    batches = [batch((4, 3, 3, 2, 1), 300 + i) for i in range(3)]
    caps = P.Caps(64, 2048, max(b.edge_bound() for b in batches))
    cfg = P.TrainConfig(use_graph=True)
    m = P.ModelT(hp, 7, range(5), caps=caps)
    ot = OracleTrainer(o, oh, 7, range(5))
    for b in batches:
        # FP64 gradients at the device's current parameters (isolates the engine's
        # error from the FP32-vs-FP64 trajectory drift of earlier AdamW steps)
        ob = O.batch_from_samples(dict(n_atoms=b.n_atoms, species=b.species, pos=b.positions, forces=b.forces,
                                       energy=b.energy, dsid=b.dataset_id), 5.0, o.build_edges)
        psh = m.shared_block().astype(np.float64)
        phd = {k: m.head_block(k).astype(np.float64) for k in range(5)}
        E, F, cache = o.forward(oh, psh, phd, ob)
        _, dE, dF = o.loss(ob, E, F)
        gs, gh = o.backward(oh, psh, phd, ob, cache, dE, dF)
        L_dev, L_ref = m.train_step(b, cfg), ot.step(b)
        assert abs(L_dev - L_ref) / abs(L_ref) < 1e-5
        g = m.debug("grads")  # this step's gradients (fused engine from step 2 on)
        PS = gs.size
        assert O.rel_vec_error(g[:PS], gs) < 1e-4
        for k in range(5):
            assert O.rel_vec_error(g[PS + k * gh[k].size:PS + (k + 1) * gh[k].size], gh[k]) < 1e-4, k
    fused = m.shared_block()
    assert O.rel_vec_error(fused, ot.sh) < 1e-3  # trajectory drift bound, as the 100-step test
    fused_heads = [m.head_block(k) for k in range(5)]
    m.close()
    monkeypatch.setenv("HMTL_NO_CHAIN", "1")
    monkeypatch.setenv("HMTL_SINGLE_STREAM", "1")
    u = P.ModelT(hp, 7, range(5), caps=caps)
    for b in batches:
        u.train_step(b, cfg)
    unfused = u.shared_block()
    for k in range(5):
        assert np.array_equal(fused_heads[k], u.head_block(k))
    u.close()
    print("fused vs oracle", O.rel_vec_error(fused, ot.sh), "unfused vs oracle", O.rel_vec_error(unfused, ot.sh),
          "fused vs unfused", O.rel_vec_error(fused, unfused))
    assert np.array_equal(fused, unfused)  # fusion and streams change no bit
