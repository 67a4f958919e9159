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


def test_cli_new_flags_rejected_cleanly_without_gpu():
    build_cli()
    r = subprocess.run([BIN, "analyze", "--crest"], capture_output=True, text=True)
    assert r.returncode == 1 and "crest" in r.stderr
    r = subprocess.run([BIN, "texture", "--kind", "plaid"], capture_output=True, text=True)
    assert r.returncode == 1 and "unknown texture kind" in r.stderr
    r = subprocess.run([BIN, "analyze", "--in", "/nonexistent.pgm"], capture_output=True, text=True)
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_texture_gradient_maps_sweep_in_and_bench_csvs(tmp_path):
    import numpy as np

    build_cli()
    # generate --gradient-maps writes <out>_grad / <out>_hess beside the map
    r = subprocess.run([BIN, "generate", "--size", "128", "--octaves", "5", "--out", str(tmp_path / "g"),
                        "--gradient-maps"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for n in ("g.pgm", "g_grad.pgm", "g_hess.pgm"):
        assert (tmp_path / n).read_bytes().startswith(b"P5")
    # texture subcommand
    for kind in ("marble", "wood", "cloud"):
        r = subprocess.run([BIN, "texture", "--kind", kind, "--size", "128", "--octaves", "4", "--out",
                            str(tmp_path / f"t_{kind}"), "--format", "png"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        assert (tmp_path / f"t_{kind}.png").read_bytes()[:8] == b"\x89PNG\r\n\x1a\n"
    # analyze --in: the written PGM analysed back equals analysing the generated map
    r = subprocess.run([BIN, "generate", "--size", "256", "--octaves", "7", "--seed", "5", "--out",
                        str(tmp_path / "a")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r_in = subprocess.run([BIN, "analyze", "--in", str(tmp_path / "a.pgm")], capture_output=True, text=True)
    assert r_in.returncode == 0, r_in.stderr
    counts_in = [ln.split(",")[1] for ln in r_in.stdout.splitlines()[1:7]]
    # the reference semantics: median of the quantised heights (monotone in the samples)
    raw = (tmp_path / "a.pgm").read_bytes()
    s = np.frombuffer(raw[-2 * 256 * 256:], dtype=">u2").astype(np.int64).reshape(256, 256)
    sea_s = np.sort(s.ravel())[s.size // 2]
    land = s >= sea_s
    pad = np.pad(land, 1, constant_values=True)
    coast = land & ~(pad[:-2, 1:-1] & pad[2:, 1:-1] & pad[1:-1, :-2] & pad[1:-1, 2:])
    want = [int(coast.reshape(256 // e, e, 256 // e, e).any(axis=(1, 3)).sum()) for e in (2, 4, 8, 16, 32, 64)]
    assert [int(c) for c in counts_in] == want
    # analyze --sweep
    r = subprocess.run([BIN, "analyze", "--sweep", "--size", "128", "--n-min", "2", "--n-max", "4",
                        "--persistences", "0.5,0.7", "--out", str(tmp_path / "sw.csv")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "sw.csv").read_text().splitlines()
    assert rows[0] == "octaves,persistence,dimension,r2" and len(rows) == 1 + 6
    # bench --csv / --speedup-csv and the cost model
    r = subprocess.run([BIN, "bench", "--methods", "zg,perlin3", "--octaves", "2,4,6", "--sizes", "256,512",
                        "--reps", "5", "--csv", str(tmp_path / "b.csv"), "--speedup-csv", str(tmp_path / "s.csv")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "b.csv").read_text().startswith(
        "method,octaves,resolution,repetitions,mean_seconds,median_seconds,min_seconds,stddev_seconds")
    assert (tmp_path / "s.csv").read_text().startswith("method,octaves,resolution,median_seconds,baseline_seconds")
    assert "cost model zg_paper" in r.stdout
