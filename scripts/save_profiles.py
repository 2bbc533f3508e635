"""Copy a gpu_bench_all.sh run into profiles/: bench JSON lines, the launch-list summary and
the ncu --set full summary (appended to profiles/r01_ncu_summary.md), and the per-class DRAM
traffic that bench.py reads (profiles/ncu_traffic.json).

    python scripts/save_profiles.py gpurun_out/r01e v4 "note"
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, ver = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
dst = os.path.join(ROOT, "profiles", f"r01_bench_{ver}")
os.makedirs(dst, exist_ok=True)
for f in ("b_head", "b_saddle", "b_2d256", "b_1d", "b_3d", "b_ref", "b_paper500"):
    p = os.path.join(src, f + ".json")
    if os.path.exists(p) and os.path.getsize(p):
        shutil.copy(p, dst)
ll = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_list.py"),
                     os.path.join(src, "launches.csv"), "12"], capture_output=True, text=True).stdout
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"),
                       os.path.join(src, "prof.ncu-rep")], capture_output=True, text=True).stdout
out = subprocess.run(["ncu", "-i", os.path.join(src, "prof.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(out)))
h, u = rr[0], rr[1]


def val(r, k):
    i = h.index(k)
    return float(r[i]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[i]]


cls = {"k_wave": "cheb_sweep", "k_fwd_upd": "forward_dft", "k_arnoldi": "arnoldi", "k_matvec": "matvec",
       "k_inverse": "inverse_dft"}
tr = {}
for r in rr[2:]:
    name = r[h.index("Kernel Name")]
    base = name.replace("void ", "").split("<")[0].split("(")[0].strip()
    for k, c in cls.items():
        if base.startswith(k):
            tr[c] = {"dram_bytes_per_launch": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                     "dram_read": val(r, "dram__bytes_read.sum"), "dram_write": val(r, "dram__bytes_write.sum"),
                     "kernel": name.split("(")[0],
                     "source": f"profiles/r01_ncu_summary.md ({ver} capture, one GMRES step of the headline)"}
json.dump({"headline": tr}, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
head = json.load(open(os.path.join(dst, "b_head.json")))
with open(os.path.join(ROOT, "profiles", "r01_ncu_summary.md"), "a") as f:
    f.write(f"\n## {ver}: headline 1024², ℓ=10, NC2 k=8 — {head['value']:.1f} its/s device, "
            f"{head['e2e']['value']:.1f} its/s end to end {note}\n\n")
    f.write("Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, 2 solves):\n```\n")
    f.write(ll + "```\n\n`ncu --set full --clock-control none`, one GMRES iteration:\n```\n" + summ + "```\n")
print(ll)
print(summ)
