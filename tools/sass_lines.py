"""Per-source-line executed instructions (and SASS) of an ncu capture for a line range.

    python tools/sass_lines.py SRC_CSV SYMBOL_SUBSTR FIRST LAST [--sass] [--src fbm3d.cu]
SRC_CSV: ncu -i REP --page source --csv --print-source sass; the in-tree
fbm2d.cu must be the source of the capture (line table from nvdisasm -gi).
"""
import collections
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src_csv, sym, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
SRCF = sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv else "fbm2d.cu"
src = os.path.join(ROOT, "paper_1610_03525_b200", "csrc", SRCF)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                "--expt-relaxed-constexpr", "-cubin", "-o", "/tmp/_k.cubin", src], check=True)
sass = subprocess.run(["nvdisasm", "-gi", "/tmp/_k.cubin"], capture_output=True, text=True).stdout.split("\n")
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
data = [r for r in rows[2:] if len(r) > iE and r[iE].isdigit()]
base = int(data[0][0], 16)
text = open(src).read().split("\n")
per = collections.Counter()
for r in data:
    loc = m.get(int(r[0], 16) - base)
    if loc and loc[0] == SRCF and lo <= loc[1] <= hi and int(r[iE]) > 0:
        per[loc[1]] += int(r[iE])
        if "--sass" in sys.argv:
            print(loc[1], r[iE], r[1][:90])
tot = sum(per.values())
print(f"lines {lo}-{hi}: {tot} warp instructions")
for ln in sorted(per):
    print(f"{per[ln]:9d} {ln:5d} {text[ln - 1].strip()[:100]}")
