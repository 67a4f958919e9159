"""Time the host-buffer entry points (drop-in generate_into) on config 2.

    python tools/time_e2e.py [--reps 20]
Prints median ms per call for f64/f32 into pinned and pageable buffers.
Host knobs come from the environment (TG_HOST_THREADS, TG_HOST_STREAM_STORES).
"""
import argparse
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--R", type=int, default=4096)
    args = ap.parse_args()
    import torch
    import paper_1610_03525_b200 as pt
    from paper_1610_03525_b200 import _abi

    lib = _abi.load()
    cfg = pt.FbmConfig(seed=42, method=pt.Method.zg_paper, smoothstep=5, octaves=12, resolution=args.R,
                       base_frequency=args.R // 512)
    ccfg = cfg.to_c()
    n = args.R * args.R
    res = {}
    for dt, fn in (("f64", lib.tg_fbm_generate_f64_host), ("f32", lib.tg_fbm_generate_f32_host)):
        for pinned in (True, False):
            t = torch.empty(n, dtype=torch.float64 if dt == "f64" else torch.float32, pin_memory=pinned)
            for _ in range(3):
                assert fn(C.byref(ccfg), 0, 0, args.R, t.data_ptr(), n) == 0, _abi.last_error()
            each = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                assert fn(C.byref(ccfg), 0, 0, args.R, t.data_ptr(), n) == 0
                each.append(time.perf_counter() - t0)
            res[f"{dt}_{'pinned' if pinned else 'pageable'}"] = round(statistics.median(each) * 1e3, 3)
    print("threads=%s stream_stores=%s" % (os.environ.get("TG_HOST_THREADS", "default"),
                                           os.environ.get("TG_HOST_STREAM_STORES", "1")), res, flush=True)


if __name__ == "__main__":
    main()
