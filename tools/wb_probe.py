import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1610_03525_b200 as pt
R = 4096
bufs = [torch.empty((R, R), dtype=torch.float32, device="cuda") for _ in range(3)]
for n in (1, 4, 8, 12):
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=R, base_frequency=8, octaves=n)
    for i in range(5):
        pt.generate_into_device(cfg, (0, 0), R, bufs[i % 3])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(60):
        pt.generate_into_device(cfg, (0, 0), R, bufs[i % 3])
    e1.record(); torch.cuda.synchronize()
    loop = e0.elapsed_time(e1) / 60 * 1e3
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(30):
            pt.generate_into_device(cfg, (0, 0), R, bufs[i % 3], stream=s)
    g.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / 120 * 1e3
    t0 = time.perf_counter()
    for i in range(60):
        pt.generate_into_device(cfg, (0, 0), R, bufs[i % 3])
    host = (time.perf_counter() - t0) / 60 * 1e6
    torch.cuda.synchronize()
    print(f"octaves {n:2d}: python loop {loop:6.1f} us  graph {graph:6.1f} us  host call {host:6.1f} us  -> {4*R*R/graph/1e3:6.0f} GB/s")
