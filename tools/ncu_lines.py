"""Aggregate ncu warp-stall samples per CUDA source line.
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = {}
cur = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 6 or r[0] == "Line No":
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1][:100])
        agg.setdefault(cur, [0.0, 0.0])
        continue
    try:
        agg[cur][0] += float(r[4] or 0)
        agg[cur][1] += float(r[5] or 0)
    except (ValueError, KeyError, TypeError):
        pass
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
