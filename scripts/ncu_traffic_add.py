"""Add one workload's per-launch DRAM traffic of a kernel class to profiles/ncu_traffic.json:
the mean of dram__bytes_read.sum + dram__bytes_write.sum over the captured launches whose name
matches REGEX (an ncu --set full report, e.g. every sweep of one GMRES iteration).

    python scripts/ncu_traffic_add.py REPORT CONFIG CLASS REGEX "source note" [PER]

PER (default 1): kernel launches that make ONE launch of the class as bench.py counts it (the
wavefront's fork/join group of one preconditioner apply is one "launch" of cheb_sweep: PER = the
number of block kernels per apply); the figure is then the sum over each group.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, config, cls, rx, note = sys.argv[1:6]
per = int(sys.argv[6]) if len(sys.argv) > 6 else 1
out = (open(rep).read() if rep.endswith(".csv") else       # a report, or its --page raw --csv export
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(r, k):
    i = h.index(k)
    return float(r[i]) * scale[u[i]]


rd, wr, names = [], [], set()
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if re.search(rx, name):
        rd.append(val(r, "dram__bytes_read.sum"))
        wr.append(val(r, "dram__bytes_write.sum"))
        names.add(name.split("(")[0])
assert rd, "no matching launch"
assert len(rd) % per == 0, f"{len(rd)} launches is not a whole number of groups of {per}"
n = len(rd) // per
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
tr = json.load(open(path))
tr.setdefault(config, {})[cls] = {
    "dram_bytes_per_launch": (sum(rd) + sum(wr)) / n, "dram_read": sum(rd) / n, "dram_write": sum(wr) / n,
    "kernel": " | ".join(sorted(names)), "launches_averaged": n, "kernels_per_launch": per, "source": note}
json.dump(tr, open(path, "w"), indent=1)
print(config, cls, n, "launches", (sum(rd) + sum(wr)) / n / 1e9, "GB per launch")
