"""The GPU CLI (tools/terrain_b200_cli.cpp): builds here, runs on the box;
mirrors the reference CLI's subcommands and exit codes (terrain_cli.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "terrain_b200")


def build_cli():
    from paper_1610_03525_b200.build import build

    build()
    lib = os.path.join(ROOT, "paper_1610_03525_b200", "lib")
    cmd = ["g++", "-std=c++20", "-O2", "-o", BIN, os.path.join(ROOT, "tools", "terrain_b200_cli.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-L", lib, "-lpolyterrain_b200",
           f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-lz"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_cli_builds_and_rejects_bad_input():
    build_cli()
    assert subprocess.run([BIN], capture_output=True).returncode == 1
    assert subprocess.run([BIN, "frobnicate"], capture_output=True).returncode == 1
    r = subprocess.run([BIN, "generate", "--method", "simplex"], capture_output=True, text=True)
    assert r.returncode == 1 and "unknown method" in r.stderr
    assert subprocess.run([BIN, "generate", "--octaves", "0"], capture_output=True).returncode == 1


@pytest.mark.gpu
def test_cli_generate_analyze_bench(tmp_path):
    import numpy as np

    build_cli()
    out = tmp_path / "m"
    r = subprocess.run([BIN, "generate", "--size", "256", "--octaves", "6", "--seed", "7", "--smoothstep", "5",
                        "--out", str(out), "--format", "png"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    png = (tmp_path / "m.png").read_bytes()
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libtgref.so")
    if os.path.exists(ref_so):
        import ctypes as C

        import torch

        from helpers import make_cfg
        from oracle.pyoracle import Reference
        from paper_1610_03525_b200 import _abi

        c = make_cfg(seed=7, smoothstep=5, resolution=256, octaves=6)
        m = torch.empty((256, 256), dtype=torch.float32, device="cuda")
        assert _abi.load().tg_fbm_generate_rect_f32(C.byref(c), 0, 0, 256, 256, m.data_ptr(), 256, None) == 0
        torch.cuda.synchronize()
        assert png == Reference().encode16(m.cpu().numpy().astype(np.float64), png=True)
    r = subprocess.run([BIN, "generate", "--size", "64", "--origin", "5,0", "--extent", "16", "--out",
                        str(tmp_path / "x")], capture_output=True, text=True)
    assert r.returncode == 1  # misaligned origin (fbm.hpp:551-558)
    r = subprocess.run([BIN, "generate", "--size", "64", "--out", "/nonexistent_dir/x.pgm"], capture_output=True)
    assert r.returncode == 2
    r = subprocess.run([BIN, "analyze", "--size", "512", "--octaves", "8", "--seed", "42"], capture_output=True,
                       text=True)
    assert r.returncode == 0 and "box-count: R=512" in r.stdout and r.stdout.startswith("epsilon,count,length")
    r = subprocess.run([BIN, "bench", "--methods", "zg,perlin3", "--octaves", "4", "--sizes", "1024", "--reps", "5"],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "speedup perlin3" in r.stdout
