"""Checked build (compute-sanitizer is closed on this GPU pool; profiles/r02/sanitizer.md):
libhmtl_b200 compiled with -DHMTL_CHECKED validates, on the device and every step, every
index structure the step's gather / scatter / GEMM kernels dereference (edge endpoints,
CSR rows, reverse edges, per-graph ranges, head permutations, sizes vs capacities) and
traps on a violation.  The parity, training, error-semantics and fused-path suites run
against it in a subprocess (HMTL_LIB) -- including the edge-capacity overflow and
non-finite cases -- so an out-of-range index anywhere in those paths fails here."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
CHECKED = os.path.join(ROOT, "abuild", "checked", "libhmtl_b200.so")


def test_gpu_suites_under_checked_build():
    import paper_2506_21788_b200 as P

    if P.lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")
    mk = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2506_21788_b200", "csrc"),
                         f"OUT={CHECKED}", f"OBJ={os.path.join(ROOT, 'abuild', 'checked', 'obj')}",
                         "EXTRA=-DHMTL_CHECKED"], capture_output=True, text=True, timeout=1800)
    assert mk.returncode == 0, mk.stderr[-2000:]
    suites = ["tests/test_gpu_parity.py", "tests/test_gpu_train.py", "tests/test_gpu_errors.py",
              "tests/test_pbc.py", "tests/test_gpu_parity_measured.py::test_mtl5_bench_batch_train_step_parity"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", *suites], cwd=ROOT,
                       capture_output=True, text=True, timeout=1800, env=dict(os.environ, HMTL_LIB=CHECKED))
    print(r.stdout[-1500:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "HMTL_CHECKED" not in r.stdout + r.stderr
