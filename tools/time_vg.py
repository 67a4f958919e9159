"""Time the variogram on a config-5-shaped map (W x H, 13 power-of-two lags),
per axis (TG_VG_AXES=1 x, 2 y) and path (TG_VG_GENERIC), CUDA events around
the synchronous C-ABI call (device time incl. the small setup copies).

    python tools/time_vg.py [--w 32768] [--h 32768] [--reps 3]
"""
import argparse
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(a):
    import torch

    import paper_1610_03525_b200 as pt
    from paper_1610_03525_b200 import _abi

    lib = _abi.load()
    cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=32768, base_frequency=32, octaves=16)
    c = cfg.to_c()
    m = torch.empty((a.h, a.w), dtype=torch.float32, device="cuda")
    assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, a.w, a.h, m.data_ptr(), a.w, None) == 0
    lags = [1 << i for i in range(13)]
    arr = (C.c_int32 * 13)(*lags)
    ss = (C.c_double * 26)()
    pr = (C.c_int64 * 26)()
    ts = []
    for _ in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        assert lib.tg_variogram_f32(m.data_ptr(), a.w, a.h, a.w, arr, 13, ss, pr, None) == 0
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{os.environ.get('TAG', ''):24s} {min(ts[1:]):8.3f} ms  (gamma1 {ss[0] + ss[1]:.6e})")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--w", type=int, default=32768)
    ap.add_argument("--h", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--modes", default="ring,ring-x,ring-y,generic,generic-x,generic-y")
    a = ap.parse_args()
    if a.child:
        return child(a)
    envs = {"ring": {}, "ring-x": {"TG_VG_AXES": "1"}, "ring-y": {"TG_VG_AXES": "2"},
            "ring-conc": {"TG_VG_CONCURRENT": "1"},
            "generic": {"TG_VG_GENERIC": "1"}, "generic-x": {"TG_VG_GENERIC": "1", "TG_VG_AXES": "1"},
            "generic-y": {"TG_VG_GENERIC": "1", "TG_VG_AXES": "2"}}
    for mode in a.modes.split(","):
        env = dict(os.environ, TAG=mode, **envs[mode])
        subprocess.run([sys.executable, __file__, "--child", "--w", str(a.w), "--h", str(a.h), "--reps",
                        str(a.reps)], env=env, check=True)


if __name__ == "__main__":
    main()
