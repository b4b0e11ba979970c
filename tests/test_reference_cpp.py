"""The REFERENCE's own C++ unit tests (proj/tests/test_*.cpp), compiled
unchanged against this repo's C++ API and linked to libpbkd_b200.so
(tests/cpp/Makefile, doctest macros from tests/cpp/doctest.h).

They are built where /root/reference exists (this container; build()) and
travel to the GPU box as binaries.  Host-only suites run on the CPU; the
rest (train_block, run_parallel, block_forward/backward, finetune, ...) run
the GPU path.  Test cases that read the reference's bundled data files
(proj/data) are excluded where that tree is absent.
"""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "_build")
DATA = "/root/reference/proj/data"
NEEDS_DATA = ["bundled demonstration trace parses", "bundled profile parses to the expected weights",
              "cost table covers every block of a deep model"]
HOST_ONLY = ["test_dataset", "test_scheduler"]
GPU = ["test_distill", "test_runtime", "test_replacement", "test_weights_io", "test_model"]


def run(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs the reference sources: make -C tests/cpp)")
    args = [exe] + ([] if os.path.isdir(DATA) else [f"--test-case-exclude={n}" for n in NEEDS_DATA])
    p = subprocess.run(args, capture_output=True, text=True, timeout=1800)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    return p.stdout


@pytest.mark.parametrize("name", HOST_ONLY)
def test_reference_unit_tests_host(name):
    out = run(name)
    assert ", 0 failed;" in out


@pytest.mark.gpu
@pytest.mark.parametrize("name", GPU)
def test_reference_unit_tests_gpu(name):
    out = run(name)
    assert ", 0 failed;" in out
