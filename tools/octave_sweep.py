"""Octave-count sweep at 4096^2 (zg_paper S5, f0 = 8): the FP32-vs-HBM
roofline crossover SURVEY §8d asks for (PAPER.md:243's N sweep).

    python tools/octave_sweep.py [--out profiles/r01_octave_sweep.json]

For N = 1..16: mean CUDA-event time per launch (3 rotating 64 MiB outputs,
> L2), sample-octaves/s, achieved TFLOP/s at 7 flop/sample-octave against the
in-run FFMA peak, and HBM write GB/s against MEASURED_PEAKS.json.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    R = 4096
    sys.path.insert(0, ROOT)
    import bench

    peak = pt.ffma_peak_tflops()
    hbm = bench.measured_hbm_gbs()
    bufs = [torch.empty((R, R), dtype=torch.float32, device="cuda") for _ in range(3)]
    # write-only HBM bandwidth on the same buffers (torch fill_): the ceiling
    # of a kernel that only writes its 64 MiB output
    for i in range(10):
        bufs[i % 3].fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(200):
        bufs[i % 3].fill_(1.0)
    e1.record()
    torch.cuda.synchronize()
    wpeak = 4 * R * R / (e0.elapsed_time(e1) / 200 * 1e-3) / 1e9  # (fill_ launches stay ahead of the GPU)
    rows = []
    for n in range(1, 17):
        cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=R, base_frequency=8,
                           octaves=n)
        for i in range(5):
            pt.generate_into_device(cfg, (0, 0), R, bufs[i % 3])
        # device rate: the launches replayed from a CUDA graph (a Python loop of
        # C-ABI calls issues one launch per ~18 us, slower than the few-octave
        # kernels themselves)
        st = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(args.iters):
                pt.generate_into_device(cfg, (0, 0), R, bufs[i % 3], stream=st)
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / (3 * args.iters) * 1e-3
        so = R * R * n / s
        tf = 7 * so / 1e12
        gbs = 4 * R * R / s / 1e9
        rows.append({"octaves": n, "us": s * 1e6, "sample_octaves_per_s": so, "tflops": tf,
                     "fp32_frac": tf / peak, "hbm_write_gbs": gbs, "hbm_frac": gbs / hbm,
                     "write_frac_vs_fill": gbs / wpeak,
                     "hashes_per_sample": bench.hashes_per_launch(R, 8, n) / (R * R)})
        print(f"N={n:2d} {s*1e6:8.1f} us  {so/1e12:6.3f} T so/s  {tf:6.2f} TF ({tf/peak:5.1%})  "
              f"{gbs:7.1f} GB/s ({gbs/hbm:5.1%})", flush=True)
    res = {"workload": "4096^2 zg_paper S5, f0 = 8, ratio 2, persistence 0.5", "ffma_peak_tflops": peak,
           "hbm_peak_gbs": hbm, "write_fill_gbs": wpeak,
           "note": "device time per launch from CUDA-graph replays of `iters` launches (3 rotating 64 MiB outputs); hbm_frac against MEASURED_PEAKS.json hbm_gbs; write_frac_vs_fill against a torch fill_ of the "
                   "same 64 MiB buffers measured in this run (write-only ceiling)", "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
