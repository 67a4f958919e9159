"""Generate every golden map one at a time in its own process
(CUDA_LAUNCH_BLOCKING=1) and report which ones fault or miss the tolerance."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json, ctypes as C
sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, ROOT)
import numpy as np, torch
from helpers import cfg_from_dict, height_tolerance
from paper_1610_03525_b200 import _abi
meta = json.load(open(os.path.join(ROOT, "tests/golden/maps.json")))[NAME]
ref = np.load(os.path.join(ROOT, "tests/golden/maps.npz"))[NAME]
c = cfg_from_dict(meta["cfg"]); (ox, oy), e = meta["origin"], meta["extent"]
out = torch.empty((e, e), dtype=torch.float32, device="cuda")
st = _abi.load().tg_fbm_generate_rect_f32(C.byref(c), ox, oy, e, e, out.data_ptr(), e, None)
torch.cuda.synchronize()
got = out.cpu().numpy().astype(np.float64)
err = float(np.max(np.abs(got - ref))); tol = height_tolerance(ref, c)
print("status", st, "err", err, "tol", tol, "OK" if err <= tol or meta["cfg"]["zero_lattice"] else "BAD")
'''
names = json.load(open(os.path.join(ROOT, "tests/golden/maps.json")))
for n in names:
    m = names[n]
    code = CHILD.replace("ROOT", repr(ROOT)).replace("NAME", repr(n))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
    last = (r.stdout.strip().split("\n") or [""])[-1] if r.returncode == 0 else "FAULT " + r.stderr.strip()[-160:]
    print(f"{n:40s} origin={m['origin']} ext={m['extent']} method={m['cfg'].get('method')} :: {last}", flush=True)
