"""Small end-to-end workload for compute-sanitizer (tools/gpu/sanitize.sh): the
neighbour list, forward, SPEC loss, backward and AdamW of a 5-head batch --
eager steps, then CUDA-graph steps -- plus a periodic (cell-list) batch and the
standalone neighbour list.  Every kernel family of the training step runs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import paper_2506_21788_b200 as P  # noqa: E402
from paper_2506_21788_b200 import data  # noqa: E402
from paper_2506_21788_b200.model import Samples  # noqa: E402


def main():
    specs = data.default5_specs()
    s = Samples.concat([data.generate_dataset(sp, 1234 + k, count=c) for k, (sp, c) in
                        enumerate(zip(specs, (10, 6, 6, 4, 3)))])
    hp = P.ModelHyper(20, 2, 128, 128, 3, 5, 5.0)
    m = P.ModelT(hp, 7, range(5), caps=P.Caps.for_samples(s))
    for g in (False, False, True, True, True):
        L = m.train_step(s, P.TrainConfig(use_graph=g))
    m.forward(s)
    m.loss()
    m.backward()
    e = P.nbr_build(s, 5.0)
    # periodic batch through the cell list
    rng = np.random.default_rng(1)
    n = np.array([40, 40], np.int32)
    pos = rng.uniform(0, 7.0, size=(80, 3))
    ps = Samples(n, np.zeros(80, np.uint8), pos, np.zeros((80, 3)), np.zeros(2), np.zeros(2, np.uint8))
    mp = P.ModelT(P.ModelHyper(20, 2, 32, 32, 3, 1, 5.0), 7, [0])
    mp.upload_pbc(ps, np.tile(np.eye(3) * 7.0, (2, 1, 1)))
    Lp = mp.train_step(None, P.TrainConfig(use_graph=False))
    print("ok loss", L, "edges", len(e["edge_dst"]), "pbc loss", Lp)


if __name__ == "__main__":
    main()
