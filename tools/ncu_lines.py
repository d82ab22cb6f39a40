"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA
source line: warp-stall samples and executed instructions.
  ncu -i REP --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_lines.py x.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.defaultdict(lambda: [0, 0, ""])
fname = "?"
cur = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ie:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        agg[cur][2] = r[1].strip()[:80]
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[si] or 0)
        agg[cur][1] += int(r[ie] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts}  instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / ts * 100:5.1f}% smp {v[1] / ti * 100:5.1f}% ins  {k[0]}:{k[1]}  {v[2]}")
