"""Build the in-tree CUDA C-ABI library for sm_100a.

    python -m paper_1610_03525_b200.build [--verbose]

Produces paper_1610_03525_b200/lib/libpolyterrain_b200.so with explicit
``-gencode arch=compute_100a,code=sm_100a`` (no torch arch list, no JIT
cache): the built file travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libpolyterrain_b200.so")
SOURCES = ["capi.cu", "fbm2d.cu", "simplex2d.cu", "perm2d.cu", "fbm3d.cu", "kernels.cu", "analysis.cu", "vgring.cu",
           "hostpipe.cpp", "terrain.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xcompiler", "-Wall"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "polyterrain_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          extra: list | None = None) -> str:
    """Compile SOURCES into `out` (default: the in-tree library)."""
    target = out or LIB
    if not force and out is None and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objdir = tempfile.mkdtemp(prefix="tgobj_", dir=LIB_DIR)  # private: concurrent builds of variants
    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *(extra or []), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        return src, obj, cmd, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        for src, obj, cmd, out in pool.map(compile_one, SOURCES):
            if verbose:
                print(" ".join(cmd))
            if out.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{out.stderr}")
            if verbose and out.stderr:
                print(out.stderr)
            objs.append(obj)
    os.makedirs(os.path.dirname(target), exist_ok=True)
    tmp = target + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lpthread", "-ldl"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"link failed:\n{out.stderr}")
    os.replace(tmp, target)
    for o in objs:
        os.remove(o)
    os.rmdir(objdir)
    return target


if __name__ == "__main__":
    # python -m paper_1610_03525_b200.build [--verbose] [--out PATH] [-DNAME=V ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else None
    extra = [a for a in argv if a.startswith("-D")]
    print(build(force=True, verbose="--verbose" in argv, out=out, extra=extra))
