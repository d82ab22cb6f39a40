"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("asicp::", "")
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
unit = "ns"
print(f"total {tot/1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e6:10.3f} ms {100*t/tot:6.2f}%  {n:6d} launches  {t/n/1e3:9.2f} us/launch  {k}")
