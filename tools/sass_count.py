"""Static SASS instruction counts of one kernel, per source line range.

    python tools/sass_count.py [--file fbm2d.cu] [--sym fbm2d_kernelILi0ELi5ELb1E] [-DNAME=V ...]
                               [--ranges A-B,C-D] [--ops]

Compiles the source to a -lineinfo cubin for sm_100a (same flags as the
library), disassembles it with nvdisasm -gi and prints the static number of
instructions of the kernel attributed to each source line range (default:
the whole kernel) plus, with --ops, the opcode mix.  Static counts are a
cheap, GPU-free proxy for the per-iteration cost of straight-line phases; the
executed counts come from ncu (tools/sass_phases.py).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
argv = sys.argv[1:]


def opt(name, default):
    return argv[argv.index(name) + 1] if name in argv else default


src = os.path.join(ROOT, "paper_1610_03525_b200", "csrc", opt("--file", "fbm2d.cu"))
sym = opt("--sym", "fbm2d_kernelILi0ELi5ELb1E")
defs = [a for a in argv if a.startswith("-D")]
cubin = "/tmp/_count_%d.cubin" % os.getpid()
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                "--expt-relaxed-constexpr", *defs, "-cubin", "-o", cubin, src], check=True)
sass = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.split("\n")
os.remove(cubin)
start = next(i for i, L in enumerate(sass) if L.startswith(".text.") and sym in L)
line, rows = None, []
for L in sass[start + 1:]:
    if L.startswith(".text."):
        break
    g = re.search(r'File "(.*?)", line (\d+)', L)
    if g:
        line = (os.path.basename(g.group(1)), int(g.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", L)
    if m:
        rows.append((line, m.group(2)))
ranges = []
for r in opt("--ranges", "").split(","):
    if r:
        a, b = r.split("-")
        ranges.append((int(a), int(b)))
base = os.path.basename(src)
print(f"{sym}: {len(rows)} instructions {' '.join(defs)}")
for a, b in ranges:
    sel = [op for (ln, op) in rows if ln and ln[0] == base and a <= ln[1] <= b]
    print(f"  lines {a}-{b}: {len(sel)}")
if "--ops" in argv:
    c = collections.Counter(op.split(".")[0] for _, op in rows)
    print("  " + " ".join(f"{k}:{v}" for k, v in c.most_common(25)))
