"""Stall-sample breakdown per kernel phase of an ncu --import-source capture.

    python tools/sass_stalls.py SRC_CSV SYMBOL_SUBSTR [--src fbm2d.cu]
SRC_CSV: ncu -i REP --page source --csv --print-source sass.  Phases are
delimited by the marker comments of the source (as in tools/sass_phases.py).
"""
import collections
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src_csv, sym = sys.argv[1], sys.argv[2]
SRCF = sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv else "fbm2d.cu"
src = os.path.join(ROOT, "paper_1610_03525_b200", "csrc", SRCF)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                "--expt-relaxed-constexpr", "-cubin", "-o", "/tmp/_ks.cubin", src], check=True)
sass = subprocess.run(["nvdisasm", "-gi", "/tmp/_ks.cubin"], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, L in enumerate(sass) if L.startswith(".text.") and sym in L)
cur, m = None, {}
for L in sass[start + 1:]:
    if L.startswith(".text."):
        break
    g = re.search(r'File "(.*?)", line (\d+)', L)
    if g:
        cur = (os.path.basename(g.group(1)), int(g.group(2)))
        continue
    g = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", L)
    if g:
        m[int(g.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
iE = hdr.index("Instructions Executed")
st_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) > iE and r[iE].isdigit()]
base = int(data[0][0], 16)
text = open(src).read().split("\n")
marks = [(i + 1, L.strip()[:44]) for i, L in enumerate(text) if L.strip().startswith("// ----") or
         re.match(r"\s*// (\(a\)|\(b\)|\(c\)|power-of-two|ppc ==|lattice-point|everything else|ppc == 1)", L)]


def phase(ln):
    name = "pre"
    for a, n in marks:
        if a <= ln:
            name = f"{a}:{n}"
    return name


agg, ins = collections.defaultdict(collections.Counter), collections.Counter()
for r in data:
    loc = m.get(int(r[0], 16) - base)
    ph = phase(loc[1]) if loc and loc[0] == SRCF else "other"
    ins[ph] += int(r[iE])
    for i in st_cols:
        agg[ph][hdr[i][6:]] += int(r[i] or 0)
tot = sum(sum(c.values()) for c in agg.values())
for ph, c in sorted(agg.items(), key=lambda x: -sum(x[1].values())):
    s = sum(c.values())
    print(f"{ph[:48]:48s} samples {s / tot * 100:5.1f}%  instr {ins[ph] / 1e6:6.2f}M  " +
          " ".join(f"{k}:{v / s * 100:.0f}" for k, v in c.most_common(6)))
