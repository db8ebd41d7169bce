"""CPU checks of the benchmark's workloads and measurement plumbing (no GPU):
the product's generator reproduces the reference's own generator (oracle/_ref)
on every workload's sources, the reference arm never maps the product library,
and kernel names map to the right roofline scopes."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

import bench

REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhmtl_ref.so")
need_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built here")


@need_ref
@pytest.mark.parametrize("workload", sorted(bench.WORKLOADS))
def test_product_generator_matches_reference_generator(workload):
    pd5, pgen = bench.product_generator()
    rd5, rgen = bench.reference_generator()
    ps, rs = bench.sources(workload, pd5), bench.sources(workload, rd5)
    assert len(ps) == len(rs) == len(bench.WORKLOADS[workload]["weights"])
    for k, (a, b) in enumerate(zip(ps, rs)):
        n = 2 if workload == "cfg4" else 5
        x, y = pgen(a, 1234 + k, n), rgen(b, 1234 + k, n)
        for f in bench.Batch.FIELDS:
            assert np.array_equal(getattr(x, f), getattr(y, f)), (workload, k, f)
    if workload == "cfg4":
        assert 200 <= x.n_atoms.min() and x.n_atoms.max() <= 300


@need_ref
def test_reference_arm_does_not_map_the_product_library():
    code = ("import sys; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','1','--ref-budget','2',"
            "'--workload','cfg2']; sys.path.insert(0, %r); import bench; bench.main(); "
            "print('MAPS', any('libhmtl_b200' in l for l in open('/proc/self/maps')))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "MAPS False" in out.stdout
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][0]
    import json

    d = json.loads(line)
    assert d["impl"] == "reference" and d["config"]["workload"] == "cfg2" and d["cpu_baseline"]["cpu_model"]
    assert d["parity"]["rel_dev"] < 1e-4


def test_kernel_scopes_keep_split_k_reduces_apart():
    names = set()
    for row in csv.reader(open(os.path.join(ROOT, "profiles", "r01_launches.csv"))):
        if len(row) > 5 and row[0].isdigit():
            names.add(row[4])
    assert names
    for n in names:
        sc = bench.scope_of(n)
        if "split_reduce_kernel" in n:
            assert sc == "bwd.wgrad_splitk_reduce", n
        if sc in ("bwd.edge_w2grad", "bwd.node_w2grad", "bwd.node_w1grad", "bwd.edge_w1ab_grad", "bwd.force_edge_wgrad"):
            assert "tc_red" in n and "split_reduce" not in n, n


def test_workload_configs_identical_across_arms():
    class B:
        G, N = 276, 3509

    a = bench.workload_config("mtl5-weak", B, 56706)
    b = bench.workload_config("mtl5-weak", B, 56706)
    assert a == b and a["per_gpu_batch"] == {"structures": 276, "edges": 56706, "nodes": 3509}
    assert bench.batch_counts("mtl5-weak") == [102, 58, 74, 24, 18]
