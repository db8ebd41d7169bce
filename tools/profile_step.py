"""Run a few eager training steps of the bench workload (for ncu / compute-sanitizer).

  python tools/profile_step.py [--steps 2] [--graph]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import bench  # noqa: E402
import paper_2506_21788_b200 as P  # noqa: E402
from paper_2506_21788_b200._lib import check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    heads, batches, _ = bench.rank_batches(0, 1)
    caps = P.Caps.for_samples(batches[0])
    for b in batches[1:]:
        caps = caps.union(P.Caps.for_samples(b))
    m = P.ModelT(P.ModelHyper(**bench.HYPER), 7, heads, caps=caps)
    cfg = P.TrainConfig(use_graph=a.graph)
    for i in range(a.steps):
        L = m.train_step(batches[i % len(batches)], cfg)
    print("loss", L)
    m.close()


if __name__ == "__main__":
    main()
