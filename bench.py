#!/usr/bin/env python
"""Benchmark: fBm heightmap generation on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload (a "step"): one 4096 x 4096 fp32 fBm heightmap, zero-gradient
polynomial cell (zg_paper) with the quintic (C2) fade, 12 octaves,
lacunarity 2, persistence 0.5, base cell 512 px (f0 = 8); octaves 10-11 are
sub-pixel.  Synthetic by construction (no dataset: every sample is a pure
function of the seed and pixel).  At N GPUs each rank generates its own
config-2-sized 4096^2 chunk of a 32768^2 terrain with the same cell sizes
(weak scaling, no data-path collective).  After the timed region the
fractal-analysis pass (median sea level, coastline + box count, variogram)
runs once on each rank's map with the statistics all-reduced (NCCL).

Timing: W warm-up steps, then K steps back to back into 3 rotating output
buffers (3 x 64 MiB = 192 MiB > 126 MB L2, so every step's writes reach HBM),
bracketed by barrier + cuda.synchronize; CUDA events on the launching stream
around the K launches (mean launch duration = bracketed time / K); max over
ranks.  Clocks are sampled through NVML during the
timed region.  `e2e` times the reference-facing drop-in
(tg_fbm_generate_f64_host = generate_into(span<double>)) with the host copy
inside the timed region.  `cpu_baseline` / `--impl reference` time the
unmodified reference (oracle/_ref) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "heightmap samples·octaves/sec per GPU & 8 GPU; % of FP32/HBM roofline"
UNIT = "sample·octaves/s"
R, F0, OCTAVES = 4096, 8, 12
FLOPS_PER_SAMPLE_OCTAVE = 7  # zg: paper's 3 mul + 3 add + 1 accumulate
BYTES_PER_SAMPLE = 4         # one fp32 store per sample, no inputs


# TG_BENCH_SHARED_GPU=1: a logic smoke test of the N-rank code paths on a
# one-GPU box — every rank on cuda:0, gloo for the process group and a host
# all-reduce hook for the statistics instead of NCCL (no rank's kernels wait on
# another's).  Not a measurement: the ranks share one GPU.
SHARED_GPU = os.environ.get("TG_BENCH_SHARED_GPU", "0") == "1"


# The contract is ONE JSON line on stdout.  Libraries write there too (NCCL
# prints "NCCL version ..." on stdout when its first communicator comes up), so
# file descriptor 1 is pointed at stderr for the life of the process and the
# line goes out through a duplicate of the original stdout.
_REAL_STDOUT = None


def _own_stdout() -> None:
    global _REAL_STDOUT
    if _REAL_STDOUT is None:
        try:
            sys.stdout.flush()
            real = os.fdopen(os.dup(1), "w")
            os.dup2(2, 1)
        except OSError:  # no usable stderr: leave stdout as it is
            return
        _REAL_STDOUT = real
        sys.stdout = sys.stderr


def _emit(line: dict) -> None:
    out = _REAL_STDOUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _device_index(local: int) -> int:
    return 0 if SHARED_GPU else local


def _init_dist(local: int) -> None:
    import torch
    import torch.distributed as dist

    if SHARED_GPU:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def _max_over_ranks(t):
    """All-reduce MAX of a one-element tensor (on the device under NCCL)."""
    import torch.distributed as dist

    if SHARED_GPU:
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def _stats_comm(device):
    from paper_1610_03525_b200.shard import Comm

    return Comm() if SHARED_GPU else Comm.nccl(device=device)


def workload_cfg(world: int, rank: int):
    import paper_1610_03525_b200 as pt

    if world == 1:
        # config 2 exactly: a 4096^2 map, f0 = 8 (base cell 512 px)
        cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=R,
                           base_frequency=F0, octaves=OCTAVES, frequency_ratio=2.0,
                           persistence=0.5, base_amplitude=1.0)
        return cfg, (0, 0)
    # Weak scaling: rank r generates its own 4096^2 chunk of a 32768^2 terrain
    # with f0 = 64 (base cell 512 px): every octave has config 2's pixels per
    # cell (512 ... 1, then lattice-point octaves k = 2, 4), so per-rank work is
    # identical to config 2 for any N <= 64; no data-path collective.
    T = 32768
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=T,
                       base_frequency=F0 * T // R, octaves=OCTAVES, frequency_ratio=2.0,
                       persistence=0.5, base_amplitude=1.0)
    per_row = T // R
    return cfg, ((rank % per_row) * R, (rank // per_row) * R)


def analysis_pass(lib, ccfg, buf, stream_ptr, world, rank):
    """Time the fractal-analysis pass on the step's map:
    device radix-select median, fused coastline + box count, variogram over
    lags 1..2048; statistics all-reduced across ranks (NCCL at N > 1)."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_1610_03525_b200 import _abi
    from paper_1610_03525_b200.shard import Comm, distributed_upper_median

    comm = _stats_comm(torch.device("cuda", torch.cuda.current_device()))
    sizes = [2, 4, 8, 16, 32, 64]
    lags = [1 << i for i in range(12)]

    def hist(prefix, mask, shift, bits):
        out = np.zeros(1 << bits, dtype=np.uint64)
        assert lib.tg_histogram_f32(buf.data_ptr(), R, R, R, prefix, mask, shift, bits, out.ctypes.data,
                                    stream_ptr) == 0, _abi.last_error()
        return out.astype(np.int64)

    def once():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sea = distributed_upper_median(hist, R * R * world, comm)
        arr = (C.c_int32 * 6)(*sizes)
        cnt = (C.c_int64 * 6)()
        coast, land = C.c_int64(), C.c_int64()
        assert lib.tg_coastline_boxcount_band(buf.data_ptr(), R, R, R, 0, 0, sea, arr, 6, cnt, C.byref(coast),
                                              C.byref(land), stream_ptr) == 0, _abi.last_error()
        t1 = time.perf_counter()
        la = (C.c_int32 * len(lags))(*lags)
        ss = (C.c_double * (2 * len(lags)))()
        pr = (C.c_int64 * (2 * len(lags)))()
        assert lib.tg_variogram_f32(buf.data_ptr(), R, R, R, la, len(lags), ss, pr, stream_ptr) == 0, \
            _abi.last_error()
        t2 = time.perf_counter()
        red = comm.allreduce(np.array(list(cnt) + [coast.value, land.value], dtype=np.int64))
        comm.allreduce(np.array(ss[:]))
        t3 = time.perf_counter()
        return sea, red, (t0, t1, t2, t3)

    once()  # warm-up: module loading and scratch-pool growth stay out of the numbers
    sea, red, (t0, t1, t2, t3) = once()
    counts = [int(v) for v in red[:6]]
    lx = [math.log(s) for s in sizes]
    ly = [math.log(max(c, 1)) for c in counts]
    mx, my = sum(lx) / 6, sum(ly) / 6
    slope = sum((a - mx) * (b - my) for a, b in zip(lx, ly)) / sum((a - mx) ** 2 for a in lx)
    return {"median_coast_boxcount_ms": (t1 - t0) * 1e3, "variogram_ms": (t2 - t1) * 1e3,
            "allreduce_ms": (t3 - t2) * 1e3, "sea_level": sea, "box_counts": counts, "d_box": -slope,
            "note": "per-rank 4096^2 map, second (warm) pass; host wall clock incl. syncs; statistics all-reduced over ranks"}


T5, F05, OCT5 = 32768, 32, 16  # config 5: 32768^2, base cell 1024 px (f0 = 32), 16 octaves, zg_paper S5


def cfg5_terrain(lib, world: int, rank: int, steps: int = 3, analysis: bool = True):
    """Config 5 on the N ranks of this job: the 32768^2 terrain in N row bands
    (strong scaling: the terrain is fixed), each rank generating its band
    (CUDA events, max over ranks), then the fractal statistics of the whole
    terrain through the C-ABI driver tg_terrain_stats_band — band regenerated
    with halo / lookahead rows, radix-select median, coastline + box counts
    (eps 2..64), variogram over lags 1..4096 — reduced across ranks by the
    native NCCL communicator (tg_comm_init_nccl)."""
    import ctypes as C

    import torch

    import paper_1610_03525_b200 as pt
    from paper_1610_03525_b200 import _abi
    from paper_1610_03525_b200.shard import Comm, DeviceBackend, plan_band, terrain_stats

    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=T5, base_frequency=F05,
                       octaves=OCT5)
    ccfg = cfg.to_c()
    sizes, lags = [2, 4, 8, 16, 32, 64], [1 << i for i in range(13)]
    band = plan_band(T5, T5, world, rank, align=1024, max_lag=max(lags))
    # the band buffer of the analysis: halo row, owned rows, lookahead rows; the
    # generation step writes the owned rows in place (row offset halo_top)
    buf = torch.empty((band.gen_rows, T5), dtype=torch.float32, device=dev)
    own = buf.data_ptr() + 4 * band.halo_top * T5
    stream = torch.cuda.current_stream(dev).cuda_stream

    def gen():
        assert lib.tg_fbm_generate_rect_f32(C.byref(ccfg), 0, band.y0, T5, band.rows, own, T5,
                                            stream) == 0, _abi.last_error()

    gen()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        gen()
    e1.record()
    torch.cuda.synchronize()
    g = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        _max_over_ranks(g)
    gen_ms = float(g.item())
    res = {"workload": f"config 5: {T5}^2 zg_paper S5, {OCT5} octaves, base cell 1024 px, {world} row band(s)",
           "gen_ms": gen_ms, "sample_octaves_per_s": float(T5) * T5 * OCT5 / (gen_ms * 1e-3),
           "band_rows": band.rows, "scaling": "strong (fixed 32768^2 terrain)"}
    if not analysis:
        return res
    comm = _stats_comm(dev)
    be = DeviceBackend(cfg, device=dev, buffer=buf, owned_ready=True)
    terrain_stats(band, be, comm, sizes, lags)  # warm-up (module loading, selection buffers)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    st = terrain_stats(band, be, comm, sizes, lags)
    torch.cuda.synchronize()
    a = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        _max_over_ranks(a)
    comm.close()
    res.update({"analysis_ms": float(a.item()) * 1e3,
                "analysis_note": "tg_terrain_stats_band_buf per rank on the generated band (halo / lookahead rows "
                                 "regenerated, none at N=1; upper median, coastline + box count, variogram 13 lags "
                                 "x 2 axes), statistics all-reduced by NCCL; host wall clock, max over ranks",
                "sea_level": st.sea_level, "land_fraction": st.land_fraction, "box_counts": st.counts,
                "d_box": st.d_box, "hurst": st.hurst, "d_variogram": st.d_variogram})
    del buf
    return res


class ClockSampler:
    """NVML clocks + throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], 0
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        rs = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": rs, "samples": len(self.samples)}


def hashes_per_launch(res: int, f0: int, octaves: int, tw: int = 128, th: int = 64) -> int:
    """Lattice-corner hashes one config-2-shaped launch performs: every
    octave's corner grid per 128 x 64 tile (shared by the tile's pixels), one
    hash per pixel for the lattice-point (sub-pixel) octaves."""
    tiles = (res // tw) * (res // th)
    total = 0
    for o in range(octaves):
        freq = f0 * 2 ** o
        if freq > res:
            total += res * res
            continue
        ppc = res // freq
        nx = tw // ppc + 1 if ppc <= tw else 2
        ny = th // ppc + 1 if ppc <= th else 2
        total += tiles * nx * ny
    return total


# Measured on B200 by tools/micro/pipe_rates.cu (warp-instructions per SMSP
# per cycle): IMAD 0.5, IMAD.WIDE.U32 / IMAD.HI.U32 0.25, SHF/LOP3 0.5,
# FFMA ~1.  One map-path lattice hash (lattice.cuh hash_top_word) is
# IMAD.WIDE + 2 IMAD + IMAD.HI + 2 IMAD = 16 IMAD-pipe cycles per warp.
IMAD_CYCLES_PER_WARP_HASH = 16
SMSP_PER_SM, N_SM = 4, 148


def integer_floor(hashes: int, launch_s: float, sm_mhz) -> dict:
    """The bound the bit-exact hash alone puts on a launch: its 64-bit
    multiplies on the IMAD pipe, all SMSPs busy, at the sampled SM clock; and
    the issue bound of the kernel's executed instruction count from the
    committed ncu capture."""
    mhz = float(sm_mhz or 1965.0)
    hash_s = hashes / 32.0 * IMAD_CYCLES_PER_WARP_HASH / (SMSP_PER_SM * N_SM) / (mhz * 1e6)
    out = {"hash_imad_floor_us": hash_s * 1e6, "frac_of_launch": hash_s / launch_s,
           "note": "hashes x 16 IMAD-pipe cycles per warp-hash / (592 SMSPs x clock); "
                   "rates from tools/micro/pipe_rates.cu"}
    inst = (traffic_summary() or {}).get("sm_inst_executed")
    if inst:
        issue_s = float(inst) / (SMSP_PER_SM * N_SM) / (mhz * 1e6)
        out.update({"issue_floor_us": issue_s * 1e6, "issue_frac_of_launch": issue_s / launch_s,
                    "issue_note": "ncu executed warp-instructions / (592 SMSPs x 1 issue/cycle x clock)"})
    return out


def measured_hbm_gbs() -> float:
    """HBM bandwidth from the driver-written MEASURED_PEAKS.json, else the
    B200 profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_bw_gbs"):
            if isinstance(d.get(k), (int, float)):
                return float(d[k])
    except Exception:
        pass
    return 6458.4


def traffic_summary():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return None


def traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_reference_run(steps: int, warmup: int, target_s: float | None = None, threads: int | None = None):
    """The unmodified reference (oracle/_ref/libtgref.so, bench::run_bench
    protocol, bench.hpp:54-78) on this host's cores.  zg with the quintic fade
    is not expressible in the reference FbmConfig: timed as the
    zg_paper S3 proxy (identical cost: the row LUT hides the fade order on
    fast octaves, and the two sub-pixel octaves sample lattice points)."""
    from oracle.pyoracle import Reference
    from paper_1610_03525_b200._abi import TgFbmConfig

    ref = Reference()
    cores = threads or os.cpu_count() or 1
    c = TgFbmConfig()
    c.seed, c.method, c.smoothstep, c.octaves, c.threads = 1, 0, 0, OCTAVES, cores
    c.resolution, c.base_frequency, c.frequency_ratio, c.persistence, c.base_amplitude = R, F0, 2.0, 0.5, 1.0
    if target_s is not None:  # size the sample to ~target_s of CPU work
        t0 = time.perf_counter()
        ref.run_bench(c, 3, 0)
        one = (time.perf_counter() - t0) / 3.0
        steps = int(max(3, min(50, target_s / max(one, 1e-6))))
        warmup = 1
    med, mn, mean = ref.run_bench(c, max(steps, 3), warmup)
    so = float(R * R * OCTAVES)
    return {"value": so / mean, "median_s": med, "min_s": mn, "mean_s": mean, "cores": cores,
            "reps": max(steps, 3), "cpu": _cpu_model()}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    r = cpu_reference_run(args.steps, args.warmup)
    sample = (f"reference bench::run_bench: {r['reps']} full {R}x{R}x{OCTAVES}-octave maps "
              f"(zg_paper S3 proxy for S5), threads={r['cores']} ({r['cpu']})")
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": r["reps"],
        "warmup": args.warmup, "ms_per_step": r["mean_s"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"config 2: {R}^2 zg_paper fBm, {OCTAVES} octaves, base cell 512 px",
                   "parallelism": f"cpu threads={r['cores']}"},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                         "sample": sample},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(line)


def run_cfg5_workload(args, rank: int, world: int, local: int) -> None:
    """--workload cfg5: the headline is config 5's generation — the 32768^2
    terrain (f0 = 32, 16 octaves, zg_paper S5) in N row bands, one per rank,
    K back-to-back band launches (CUDA events, max over ranks); value = the
    whole terrain's sample-octaves per second (strong scaling).  e2e: each
    rank's band through the drop-in generate_into(span<double>) as 4096^2
    chunks into pinned host memory.  Then the NCCL-reduced statistics."""
    import torch
    import torch.distributed as dist

    import paper_1610_03525_b200 as pt
    from paper_1610_03525_b200 import _abi
    from paper_1610_03525_b200.shard import plan_band

    local = _device_index(local)
    torch.cuda.set_device(local)
    if world > 1:
        _init_dist(local)
    lib = _abi.load()
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=T5, base_frequency=F05,
                       octaves=OCT5)
    ccfg = cfg.to_c()
    band = plan_band(T5, T5, world, rank, align=1024, max_lag=4096)
    peak_tflops = pt.ffma_peak_tflops()
    out = [torch.empty((band.rows, T5), dtype=torch.float32, device="cuda") for _ in range(2)]
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream

    def launch(i):
        if lib.tg_fbm_generate_rect_f32(C.byref(ccfg), 0, band.y0, T5, band.rows, out[i % 2].data_ptr(), T5, sp):
            raise RuntimeError(_abi.last_error())

    with torch.cuda.stream(stream):
        for i in range(max(args.warmup, 3)):
            launch(i)
    torch.cuda.synchronize()
    K = max(1, min(args.steps, 20))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for i in range(K):
                launch(i)
            ev[1].record(stream)
        torch.cuda.synchronize()
    t = torch.tensor([ev[0].elapsed_time(ev[1])], dtype=torch.float64, device="cuda")
    if world > 1:
        _max_over_ranks(t)
    total_ms = float(t.item())
    so_step = float(T5) * T5 * OCT5
    value = so_step * K / (total_ms * 1e-3)
    per_rank_s = total_ms * 1e-3 / K
    achieved = FLOPS_PER_SAMPLE_OCTAVE * band.rows * T5 * OCT5 / per_rank_s / 1e12
    del out
    torch.cuda.empty_cache()
    # e2e: the drop-in over the rank's band in 4096^2 chunks, pinned host doubles
    C4 = 4096
    host = torch.empty((C4, C4), dtype=torch.float64, pin_memory=True)
    chunks = [(x, y) for y in range(band.y0, band.y0 + band.rows, C4) for x in range(0, T5, C4)]
    for (x, y) in chunks[:2]:
        assert lib.tg_fbm_generate_f64_host(C.byref(ccfg), x, y, C4, host.data_ptr(), C4 * C4) == 0, _abi.last_error()
    if world > 1:
        dist.barrier()
    e2e_steps = 2
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        for (x, y) in chunks:
            assert lib.tg_fbm_generate_f64_host(C.byref(ccfg), x, y, C4, host.data_ptr(), C4 * C4) == 0
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        _max_over_ranks(te)
    e2e_value = so_step * e2e_steps / float(te.item())
    stats = cfg5_terrain(lib, world, rank, steps=1, analysis=not args.no_analysis)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": max(args.warmup, 3), "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config 5: {T5}x{T5} fp32 fBm, zg_paper C2 (S5), {OCT5} octaves, base cell "
                                   f"1024 px (f0 = 32), row bands over {world} GPU(s)",
                       "parallelism": f"{world} row bands (no data-path collective; statistics NCCL-reduced)",
                       "l2": f"2 rotating {band.rows * T5 * 4 >> 20} MiB band outputs (> 126 MB L2)"},
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": achieved / peak_tflops, "traffic": None,
                         "note": f"{FLOPS_PER_SAMPLE_OCTAVE} flop/sample-octave x the slowest rank's band"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": C.sizeof(ccfg) * len(chunks),
                    "d2h_bytes_per_step": band.rows * T5 * 8, "steps": e2e_steps,
                    "note": "tg_fbm_generate_f64_host (drop-in generate_into span<double>) per 4096^2 chunk of "
                            "each rank's band into pinned host memory; max over ranks"},
            "gpu_launches": K, "clocks": clk.summary(), "cpu_baseline": None,
            "cfg5_terrain": stats,
        }
        _emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-analysis", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg5"],
                    help="cfg2 (default): config 2 per rank (weak scaling); cfg5: the 32768^2 config-5 terrain "
                         "in N row bands (strong scaling) with NCCL-reduced statistics")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the config-5 terrain section of the cfg2 line")
    args = ap.parse_args()
    _own_stdout()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if args.workload == "cfg5":
        run_cfg5_workload(args, rank, world, local)
        return

    import torch
    import torch.distributed as dist

    import paper_1610_03525_b200 as pt
    from paper_1610_03525_b200 import _abi

    local = _device_index(local)
    torch.cuda.set_device(local)
    if world > 1:
        _init_dist(local)
    lib = _abi.load()
    cfg, origin = workload_cfg(world, rank)
    ccfg = cfg.to_c()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    bufs = [torch.empty((R, R), dtype=torch.float32, device="cuda") for _ in range(3)]

    def launch(i: int) -> None:
        st = lib.tg_fbm_generate_rect_f32(C.byref(ccfg), origin[0], origin[1], R, R, bufs[i % 3].data_ptr(), R, sp)
        if st != 0:
            raise RuntimeError(_abi.last_error())

    peak_tflops = pt.ffma_peak_tflops()
    with torch.cuda.stream(stream):
        for i in range(max(args.warmup, 3)):
            launch(i)
    torch.cuda.synchronize()

    K = args.steps
    # Events only around the K back-to-back launches (on their stream): an
    # event record between launches inserts a gap (~3 us per 60 us launch
    # measured), and the launches are serialised on the stream anyway, so the
    # mean launch duration is the bracketed time / K.
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for i in range(K):
                launch(i)
            ev[1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = ev[0].elapsed_time(ev[1])
    per_launch_ms = [total_ms / K]
    # Isolated launches (outside the timed region): the generation kernel is
    # launched with programmatic stream serialisation, so back-to-back launches
    # overlap one grid's tail with the next grid's hashing; report what a
    # single launch with an idle GPU before and after it takes as well.
    iso = []
    with torch.cuda.stream(stream):
        for i in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            torch.cuda._sleep(100000)  # ~50 us: e0 and the launch are queued before the GPU reaches e0
            e0.record(stream)
            launch(i)
            e1.record(stream)
            torch.cuda.synchronize()
            iso.append(e0.elapsed_time(e1))
    isolated_us = statistics.median(iso) * 1e3
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        _max_over_ranks(t)
    total_ms_max = float(t.item())

    so_per_step = float(R * R * OCTAVES)
    value = so_per_step * K * world / (total_ms_max * 1e-3)
    avg_launch_s = statistics.mean(per_launch_ms) * 1e-3
    achieved_tflops = FLOPS_PER_SAMPLE_OCTAVE * so_per_step / avg_launch_s / 1e12
    hbm_gbs = BYTES_PER_SAMPLE * R * R / avg_launch_s / 1e9

    # ---- end to end through the drop-in host API (generate_into(span<double>)) ----
    e2e_steps = args.e2e_steps or max(5, min(K, 20))
    host = torch.empty((R, R), dtype=torch.float64, pin_memory=True)
    for _ in range(3):
        st = lib.tg_fbm_generate_f64_host(C.byref(ccfg), origin[0], origin[1], R, host.data_ptr(), R * R)
        assert st == 0, _abi.last_error()
    if world > 1:
        dist.barrier()
    e2e_each = []
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        t1 = time.perf_counter()
        st = lib.tg_fbm_generate_f64_host(C.byref(ccfg), origin[0], origin[1], R, host.data_ptr(), R * R)
        assert st == 0, _abi.last_error()
        e2e_each.append(time.perf_counter() - t1)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        _max_over_ranks(te)
    e2e_value = so_per_step * e2e_steps * world / float(te.item())
    # the reference's callers pass a std::vector<double> (pageable): same call
    # into a pageable buffer, reported beside the pinned headline
    host_pg = torch.empty((R, R), dtype=torch.float64)
    pg_each = []
    for i in range(e2e_steps + 2):
        t1 = time.perf_counter()
        st = lib.tg_fbm_generate_f64_host(C.byref(ccfg), origin[0], origin[1], R, host_pg.data_ptr(), R * R)
        assert st == 0, _abi.last_error()
        if i >= 2:
            pg_each.append(time.perf_counter() - t1)
    del host_pg

    analysis = None
    if not args.no_analysis:
        try:
            analysis = analysis_pass(lib, ccfg, bufs[(K - 1) % 3], sp, world, rank)
        except Exception as e:  # pragma: no cover
            analysis = {"error": str(e)}
    terrain5 = None
    if not args.no_cfg5:
        del bufs
        torch.cuda.empty_cache()
        try:
            terrain5 = cfg5_terrain(lib, world, rank, steps=3, analysis=not args.no_analysis)
        except Exception as e:  # pragma: no cover
            terrain5 = {"error": str(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_run(0, 0, target_s=15.0)
            cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                   "sample": (f"reference bench::run_bench (oracle/_ref, unmodified headers): "
                              f"{r['reps']} full {R}^2 x {OCTAVES}-octave maps, zg_paper S3 proxy "
                              f"for S5, threads={r['cores']}, median {r['median_s']*1e3:.1f} ms, "
                              f"{r['cpu']}")}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
        try:  # bench.hpp:54-78 is also quoted single-threaded (the CLI forces threads = 1, terrain_cli.cpp:403)
            r1 = cpu_reference_run(0, 0, target_s=10.0, threads=1)
            cpu["threads_1"] = {"value": r1["value"], "cores": 1,
                                "sample": f"{r1['reps']} full {R}^2 x {OCTAVES}-octave maps, threads=1, median "
                                          f"{r1['median_s']*1e3:.1f} ms"}
        except Exception as e:  # pragma: no cover
            cpu["threads_1"] = {"value": None, "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": max(args.warmup, 3), "ms_per_step": total_ms_max / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config 2: {R}x{R} fp32 fBm, zg_paper C2 (S5), {OCTAVES} octaves, "
                                   f"lacunarity 2, persistence 0.5, base cell 512 px"
                                   + ("" if world == 1 else f"; one such chunk per rank of a 32768^2 terrain"),
                       "global_maps_per_step": world, "samples_per_step_per_gpu": R * R,
                       "parallelism": f"shard{world} (independent chunks, no data-path collective)",
                       "l2": "3 rotating 64 MiB outputs (192 MiB > 126 MB L2)"},
            "roofline": {"bound": "fp32", "achieved": achieved_tflops, "peak": peak_tflops,
                         "unit": "TFLOP/s", "frac": achieved_tflops / peak_tflops,
                         "traffic": traffic_from_profiles(),
                         "note": (f"{FLOPS_PER_SAMPLE_OCTAVE} flop/sample-octave (paper op count + accumulate) "
                                  f"x {int(so_per_step)} sample-octaves per launch / mean CUDA-event launch "
                                  f"time {avg_launch_s*1e6:.1f} us over the K back-to-back launches (programmatic "
                                  f"dependent launch overlaps each grid's tail with the next one's hashing; an "
                                  f"isolated launch takes {isolated_us:.1f} us, frac "
                                  f"{FLOPS_PER_SAMPLE_OCTAVE * so_per_step / (isolated_us * 1e-6) / 1e12 / peak_tflops:.3f}); "
                                  f"peak = FFMA-chain measured in-run (MEASURED_PEAKS.json has no FP32 entry)"),
                         "isolated_launch_us": isolated_us,
                         "hbm_write_gbs": hbm_gbs, "hbm_frac": hbm_gbs / measured_hbm_gbs(),
                         "hashes_per_launch": hashes_per_launch(R, F0, OCTAVES),
                         "hashes_per_s": hashes_per_launch(R, F0, OCTAVES) / avg_launch_s,
                         "pipes_pct_ncu": {k: (traffic_summary() or {}).get(k)
                                           for k in ("pipe_fma_pct", "pipe_alu_pct", "pipe_xu_pct")},
                         "issue_slots_busy_pct_ncu": (traffic_summary() or {}).get("issue_active_pct"),
                         "issue_note": "the bit-exact 64-bit lattice hash is integer work outside the 7-flop "
                                       "convention; issue-slot utilisation of the same kernel from the committed "
                                       "ncu capture (profiles/ncu_summary.json)",
                         "integer_floor": integer_floor(hashes_per_launch(R, F0, OCTAVES), avg_launch_s,
                                                        clk.summary().get("sm_mhz"))},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": C.sizeof(ccfg),
                    "d2h_bytes_per_step": R * R * 8, "steps": e2e_steps,
                    "ms_per_step_median": statistics.median(e2e_each) * 1e3,
                    "d2h_gbs": R * R * 8 / statistics.median(e2e_each) / 1e9,
                    "pageable_ms_per_step_median": statistics.median(pg_each) * 1e3,
                    "note": "tg_fbm_generate_f64_host (drop-in generate_into span<double>) into pinned host "
                            "memory; input is the config struct only; fp32 bands cross PCIe (64 MiB) and "
                            "are widened to the caller's doubles by the host pool inside the copies' shadow "
                            "(4 MiB bands, 8-slot pinned ring, asynchronous pool join; capi.cu generate_host); "
                            "the PCIe time of the 64 MiB is ~1.26 ms; pageable_ms: the same call into a "
                            "pageable buffer"},
            "gpu_launches": K,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "analysis": analysis,
            "cfg5_terrain": terrain5,
        }
        _emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
