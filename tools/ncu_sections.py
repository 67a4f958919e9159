"""Group ncu per-line instruction counts into line ranges.
Usage: ncu_sections.py mix.csv file.cu name:start [name:start ...]  (ranges up to next start)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
marks = sorted((int(a.split(':')[1]), a.split(':')[0]) for a in sys.argv[3:])
hdr, cur, agg, tot = None, "", {}, 0
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    tot += ins
    if cur != target:
        key = cur
    else:
        ln = int(r[0])
        key = "pre"
        for s, n in marks:
            if ln >= s:
                key = n
    agg[key] = agg.get(key, 0) + ins
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:14s} {100*v/tot:5.1f}%  {v}")
