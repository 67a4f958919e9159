"""The host worker pool and widening kernels of the drop-in path
(csrc/hostpipe.cpp) on the CPU: tests/cpp/test_hostpipe.cpp, with the default
pool and with one / many workers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("hostpipe") / "test_hostpipe")
    cmd = ["g++", "-std=c++17", "-O2", "-pthread", "-Wall", "-o", out,
           os.path.join(ROOT, "tests", "cpp", "test_hostpipe.cpp"),
           os.path.join(ROOT, "paper_1610_03525_b200", "csrc", "hostpipe.cpp")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("threads", [None, "1", "3", "12"])
def test_hostpipe(binary, threads):
    env = dict(os.environ)
    env.pop("TG_HOST_THREADS", None)
    if threads:
        env["TG_HOST_THREADS"] = threads
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")


@pytest.mark.parametrize("isa", [{"TG_HOST_AVX512": "0"}, {"TG_HOST_AVX512": "0", "TG_HOST_AVX2": "0"}])
def test_hostpipe_without_avx512(binary, isa):
    """The AVX2 and SSE2 widening forms (hosts without AVX-512)."""
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, TG_HOST_THREADS="4", **isa))
    assert r.returncode == 0, r.stdout + r.stderr


def test_hostpipe_thread_sanitizer(tmp_path):
    """The pool's submit / join / burst protocol under ThreadSanitizer (the
    device side has no sanitizer on the GPU pool; the host side does)."""
    out = str(tmp_path / "test_hostpipe_tsan")
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-pthread", "-fsanitize=thread", "-o", out,
           os.path.join(ROOT, "tests", "cpp", "test_hostpipe.cpp"),
           os.path.join(ROOT, "paper_1610_03525_b200", "csrc", "hostpipe.cpp")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("ThreadSanitizer runtime not available: " + r.stderr[-200:])
    r = subprocess.run([out], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, TG_HOST_THREADS="6", TSAN_OPTIONS="halt_on_error=1"))
    assert r.returncode == 0 and "WARNING: ThreadSanitizer" not in r.stderr, r.stdout + r.stderr[-3000:]
