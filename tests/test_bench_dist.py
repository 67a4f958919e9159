"""bench.py's multi-rank helpers under a real process group.

The N > 1 arm of bench.py cannot run on the one-GPU boxes, so its helpers are
driven here: the max-over-ranks reduction under gloo (two CPU ranks, the
TG_BENCH_SHARED_GPU branch) and, on the GPU box, under a one-rank NCCL group
(the branch the driver's scaling run takes).
"""
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port

GLOO_CHILD = textwrap.dedent("""
    import os, sys
    sys.path.insert(0, %r)
    os.environ["TG_BENCH_SHARED_GPU"] = "1"
    import torch, torch.distributed as dist
    import bench
    dist.init_process_group("gloo")
    t = torch.tensor([float(dist.get_rank() + 1)], dtype=torch.float64)
    bench._max_over_ranks(t)
    assert float(t.item()) == float(dist.get_world_size()), t
    dist.barrier()
    dist.destroy_process_group()
    print("ok")
""" % ROOT)


def test_max_over_ranks_gloo_two_ranks(tmp_path):
    script = tmp_path / "child.py"
    script.write_text(GLOO_CHILD)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.count("ok") == 2


NCCL_CHILD = textwrap.dedent("""
    import os, sys
    sys.path.insert(0, %r)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ["TG_TEST_PORT"], RANK="0", WORLD_SIZE="1",
                      LOCAL_RANK="0")
    os.environ.pop("TG_BENCH_SHARED_GPU", None)
    import torch, torch.distributed as dist
    import bench
    assert not bench.SHARED_GPU
    torch.cuda.set_device(0)
    bench._init_dist(0)                       # the N > 1 branch: NCCL process group
    t = torch.tensor([3.5], dtype=torch.float64, device="cuda")
    bench._max_over_ranks(t)                  # all-reduce MAX on the device
    assert float(t.item()) == 3.5
    comm = bench._stats_comm(torch.device("cuda", 0))   # native NCCL communicator from a broadcast id
    import numpy as np
    assert comm.allreduce(np.array([1, 2, 3], dtype=np.int64)).tolist() == [1, 2, 3]
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    print("ok")
""" % ROOT)


@pytest.mark.gpu
def test_bench_nccl_helpers_one_rank(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "child.py"
    script.write_text(NCCL_CHILD)
    out = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, TG_TEST_PORT=str(_free_port())))
    assert out.returncode == 0, out.stderr[-2000:]
    assert "ok" in out.stdout


REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e")


def _one_json_line(stdout: str) -> dict:
    import json

    lines = [ln for ln in stdout.split("\n") if ln.strip()]
    assert len(lines) == 1, f"stdout must hold exactly one line, got {len(lines)}: {stdout[:300]!r}"
    return json.loads(lines[0])


def test_reference_arm_prints_one_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libtgref.so")):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _one_json_line(out.stdout)
    assert d["impl"] == "reference" and all(k in d for k in REQUIRED) and "cpu_baseline" in d


@pytest.mark.gpu
def test_bench_prints_one_json_line_with_the_contract_keys():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _one_json_line(out.stdout)  # NCCL's version banner must not land on stdout
    assert all(k in d for k in REQUIRED + ("roofline", "gpu_launches", "clocks"))
    assert d["gpu_launches"] == 5 and d["e2e"]["d2h_bytes_per_step"] == 4096 * 4096 * 8
    assert d["cfg5_terrain"] and "error" not in d["cfg5_terrain"]
