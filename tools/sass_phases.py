"""Attribute an ncu capture's executed SASS instructions to kernel phases.

    python tools/sass_phases.py REPORT.ncu-rep CUBIN_SYMBOL_SUBSTR [--lines N]

Joins the report's per-instruction counts (source page, SASS view) with the
line table of the in-tree build (nvdisasm -gi on a -lineinfo cubin of
fbm2d.cu) by instruction offset, then sums by opcode and by source line.
Needs the capture to come from the same build as the current source.
"""
import collections
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, sym = sys.argv[1], sys.argv[2]
nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 30
src_name = sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv else "fbm2d.cu"
src_file = os.path.join(ROOT, "paper_1610_03525_b200", "csrc", src_name)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                "--expt-relaxed-constexpr", "-cubin", "-o", "/tmp/_k.cubin", src_file], check=True)
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
        m[int(g.group(1), 16)] = (cur, g.group(2))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.split("\n")))
hdr = rows[1]
iE, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > iE and r[iE].isdigit()]
base = int(data[0][0], 16)
byop, byline, st = collections.Counter(), collections.Counter(), collections.Counter()
fpline = collections.Counter()  # FFMA / FADD / FMUL per line (candidates for fp32x2 packing)
tot = 0
for r in data:
    n, s = int(r[iE]), int(r[iS] or 0)
    loc, ins = m.get(int(r[0], 16) - base, ((None, 0), "?"))
    op = r[1].strip().split()
    op = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    byop[op] += n
    byline[loc] += n
    st[loc] += s
    if op in ("FFMA", "FADD", "FMUL"):
        fpline[loc] += n
    tot += n
print("executed warp instructions:", tot)
print(" ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in byop.most_common(14)))
text = {f: open(os.path.join(ROOT, "paper_1610_03525_b200", "csrc", f)).read().split("\n")
        for f in (src_name, "lattice.cuh")}
for loc, v in byline.most_common(nlines):
    f, ln = loc
    s = text.get(f, [""] * (ln + 1))[ln - 1].strip()[:88] if f else "?"
    print(f"{v:9d} {v / tot * 100:5.1f}% st{st[loc]:5d} {str(f)[:6]}:{ln:4d} {s}")

if "--fp" in sys.argv:
    fpt = sum(fpline.values())
    print(f"scalar fp32 (FFMA/FADD/FMUL): {fpt} = {fpt / tot * 100:.1f}%")
    for loc, v in fpline.most_common(nlines):
        f, ln = loc
        s = text.get(f, [""] * (ln + 1))[ln - 1].strip()[:88] if f else "?"
        print(f"{v:9d} {v / tot * 100:5.1f}% {str(f)[:6]}:{ln:4d} {s}")

# --- optional: sum by kernel phase, delimited by marker comments in fbm2d.cu
if "--phases" in sys.argv:
    src = text["fbm2d.cu"]
    marks = [(i + 1, L.strip()[:60]) for i, L in enumerate(src) if L.strip().startswith("// ----") or
             re.match(r"\s*// (\(a\)|\(b\)|power-of-two|ppc ==|lattice-point|everything else|ppc == 1)", L)]
    def phase(ln):
        name = "pre"
        for a, n in marks:
            if a <= ln:
                name = f"{a}:{n}"
        return name
    agg = collections.Counter()
    for loc, v in byline.items():
        f, ln = loc
        agg[phase(ln) if f == "fbm2d.cu" else f"other:{f}"] += v
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v:9d} {v / tot * 100:5.1f}%  {k}")
