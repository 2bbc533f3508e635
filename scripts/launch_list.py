"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel and grid.
    python scripts/launch_list.py gpurun_out/TAG/launches.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0] + " " + d.get("Grid Size", "")
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k:64s} n={n:5d} tot={t / 1e6:8.3f}ms share={t / tot:.3f} avg={t / n / 1e3:8.2f}us")
print(f"total {tot / 1e6:.3f} ms")
