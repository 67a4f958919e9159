"""Build the C++ drop-in test (tests/cpp/test_dropin.cpp) against the
in-tree CUDA library; run it on the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_binary():
    from oracle.pyoracle import build as build_oracle
    from paper_1610_03525_b200.build import build

    build()
    build_oracle()
    lib = os.path.join(ROOT, "paper_1610_03525_b200", "lib")
    cmd = ["g++", "-std=c++20", "-O2", "-o", BIN, os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-L", lib, "-lpolyterrain_b200", f"-Wl,-rpath,{lib}",
           os.path.join(ROOT, "oracle", "liboracle.so"), f"-Wl,-rpath,{os.path.join(ROOT, 'oracle')}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_dropin_header_compiles_and_links():
    build_binary()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu():
    build_binary()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
