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
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-lz"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_dropin_header_compiles_and_links():
    build_binary()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(tmp_path):
    build_binary()
    env = dict(os.environ, TG_OUT_DIR=str(tmp_path))
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600, env=env)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    # the C++ io.hpp files equal the reference writers on the same map
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libtgref.so")
    if os.path.exists(ref_so):
        import ctypes as C

        import numpy as np
        import torch

        from helpers import make_cfg
        from oracle.pyoracle import Reference
        from paper_1610_03525_b200 import _abi

        c = make_cfg(method=0, smoothstep=5, seed=5, resolution=1024, base_frequency=4, octaves=10)
        m = torch.empty((200, 300), dtype=torch.float32, device="cuda")
        assert _abi.load().tg_fbm_generate_rect_f32(C.byref(c), 0, 0, 300, 200, m.data_ptr(), 300, None) == 0
        torch.cuda.synchronize()
        host = m.cpu().numpy().astype(np.float64)
        ref = Reference()
        assert (tmp_path / "dropin_300x200.pgm").read_bytes() == ref.encode16(host, png=False)
        assert (tmp_path / "dropin_300x200.png").read_bytes() == ref.encode16(host, png=True)
