"""Summarise an ncu source page (cuda,sass csv) per CUDA source line:
instructions executed and stall samples.  Usage: ncu_lines.py mix.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur_file = ""
out = []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    out.append((ins, smp, f"{cur_file}:{r[0]}", r[1][:90]))
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
print(f"total warp-instr {tot_i}  samples {tot_s}")
for ins, smp, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100*ins/tot_i:5.1f}% ins {100*smp/tot_s:5.1f}% smp  {loc:16s} {src}")
