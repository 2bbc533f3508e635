"""Top stalled SASS instructions of the first kernel in an ncu report (experiment support).

    python scripts/ncu_hot.py REPORT [N] [kernel-index]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')[1:]
b = blocks[kidx]
lines = b.split("\n", 1)
print(lines[0][:150])
rows = list(csv.reader(io.StringIO(lines[1])))
h = rows[0]
iS, iA, iN = h.index("Source"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iN] or 0) for r in rows[1:] if len(r) > iN)
print("total samples", tot)
agg = {c: sum(float(r[h.index(c)] or 0) for r in rows[1:] if len(r) == len(h)) for c in cols}
print("by reason:", ", ".join(f"{k[6:]}={v / tot:.2f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
top = sorted((r for r in rows[1:] if len(r) == len(h)), key=lambda r: -float(r[iN] or 0))[:n]
for r in top:
    why = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{r[iA]:>6} {float(r[iN]) / tot:6.3f}  {r[iS][:60]:60s} " + " ".join(f"{w}={v:.0f}" for v, w in why if v))
