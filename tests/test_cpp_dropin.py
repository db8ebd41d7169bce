"""The C++ drop-in header (include/hmtl_b200.hpp): compile the reference-style
test program here (CPU), run it on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

import paper_2506_21788_b200 as P

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2506_21788_b200")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_bin():
    P.build()
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
                    f"-L{LIBDIR}", "-lhmtl_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_dropin_header_compiles_and_links():
    build_bin()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_reference_style_tests_pass_on_gpu():
    build_bin()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
