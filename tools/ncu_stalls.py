"""Per-CUDA-line warp-stall breakdown from an ncu source page CSV.
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_stalls.py x.csv FILE LO HI"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want, lo, hi = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
hdr, fname, cur, agg, tot = None, "", None, {}, {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) // 2:
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1][:90])
        continue
    d = {h: r[k] for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    for h, v in d.items():
        try:
            x = float(v or 0)
        except ValueError:
            continue
        tot[h] = tot.get(h, 0) + x
        if cur and cur[0] == want and lo <= cur[1] <= hi:
            agg.setdefault(cur, {}).setdefault(h, 0)
            agg[cur][h] += x
T = sum(tot.values()) or 1
print("kernel total:", ", ".join(f"{h[6:]} {v / T * 100:.1f}%" for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]))
for k in sorted(agg):
    s = sum(agg[k].values())
    if s / T < 0.002:
        continue
    top = sorted(agg[k].items(), key=lambda kv: -kv[1])[:4]
    print(f"{s / T * 100:5.1f}% L{k[1]:4d} {k[2][:60]:60s} " + " ".join(f"{h[6:]}:{v / T * 100:.1f}" for h, v in top))
