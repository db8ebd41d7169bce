"""HMTP checkpoints with optimizer state: the reference's
format (src/model_io.cpp:7-13, 62-118) byte for byte, plus a trailing AdamW
section the reference's reader ignores, for exact resume."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()


def ref_ckpt():
    g = np.load(os.path.join(GOLDEN, "ckpt.npz"))
    hv = g["hyper"]
    hp = P.ModelHyper(int(hv[0]), int(hv[1]), int(hv[2]), int(hv[3]), int(hv[4]), int(hv[5]), 5.0)
    return hp, g["shared"], [g[f"head{k}"] for k in range(hp.n_heads)]


def test_writer_byte_identical_to_reference(tmp_path):
    hp, sh, heads = ref_ckpt()
    out = str(tmp_path / "ours.hmtp")
    P.checkpoint_write(out, hp, sh, heads)
    assert open(out, "rb").read() == open(os.path.join(GOLDEN, "ckpt_ref.hmtp"), "rb").read()


def test_read_hyper_and_errors(tmp_path):
    hp, has_opt = P.checkpoint_hyper(os.path.join(GOLDEN, "ckpt_ref.hmtp"))
    assert (hp.layers, hp.hidden, hp.n_heads, has_opt) == (2, 16, 3, False)
    bad = tmp_path / "bad.hmtp"
    bad.write_bytes(b"HMTPxxxx")
    with pytest.raises(P.HmtlError):
        P.checkpoint_hyper(str(bad))
    raw = open(os.path.join(GOLDEN, "ckpt_ref.hmtp"), "rb").read()
    (tmp_path / "short.hmtp").write_bytes(raw[:-100])
    with pytest.raises(P.HmtlError, match="short read"):
        P.checkpoint_hyper(str(tmp_path / "short.hmtp"))


@pytest.mark.gpu
def test_load_reference_checkpoint_and_mtl_par_subset():
    hp, sh, heads = ref_ckpt()
    m = P.ModelT(hp, 1, range(3))
    m.load_checkpoint(os.path.join(GOLDEN, "ckpt_ref.hmtp"))
    assert np.array_equal(m.shared_block(), sh)
    for k in range(3):
        assert np.array_equal(m.head_block(k), heads[k])
    m.close()
    r = P.ModelT(hp, 1, [2])  # an MTL-par rank owning head 2 only
    r.load_checkpoint(os.path.join(GOLDEN, "ckpt_ref.hmtp"))
    assert np.array_equal(r.head_block(2), heads[2]) and np.array_equal(r.shared_block(), sh)
    with pytest.raises(P.HmtlError, match="need all head blocks"):
        r.save_checkpoint("/tmp/never.hmtp")
    r.close()


@pytest.mark.gpu
def test_exact_resume_with_optimizer_state(tmp_path):
    """train 3 steps, checkpoint (+AdamW), resume in a fresh context, 2 more steps
    == 5 uninterrupted steps, bit for bit; the file still loads as a plain
    (reference) checkpoint."""
    hp = P.ModelHyper(20, 2, 32, 32, 3, 5, 5.0)
    specs = data.default5_specs()
    batches = [P.Samples.concat([data.generate_dataset(sp, 500 + 10 * i + k, count=c)
                                 for k, (sp, c) in enumerate(zip(specs, (4, 3, 3, 2, 1)))]) for i in range(5)]
    caps = P.Caps.for_samples(batches[0])
    for b in batches[1:]:
        caps = caps.union(P.Caps.for_samples(b))
    cfg = P.TrainConfig(use_graph=True)
    a = P.ModelT(hp, 7, range(5), caps=caps)
    La = [a.train_step(b, cfg) for b in batches]
    b_ = P.ModelT(hp, 7, range(5), caps=caps)
    Lb = [b_.train_step(b, cfg) for b in batches[:3]]
    path = str(tmp_path / "r.hmtp")
    b_.save_checkpoint(path)
    b_.close()
    assert P.checkpoint_hyper(path)[1]
    c = P.ModelT(hp, 99, range(5), caps=caps)  # different init seed: everything comes from the file
    c.load_checkpoint(path)
    Lc = [c.train_step(b, cfg) for b in batches[3:]]
    assert La == Lb + Lc
    assert np.array_equal(a.shared_block(), c.shared_block())
    for k in range(5):
        assert np.array_equal(a.head_block(k), c.head_block(k))
    a.close(), c.close()
