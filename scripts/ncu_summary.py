"""Summarise an ncu report (raw page): per launch time, DRAM bytes, throughput, occupancy.
    python scripts/ncu_summary.py gpurun_out/TAG/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Kernel Name", "Block Size", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
idx = {w: hdr.index(w) for w in want if w in hdr}
units = rows[1]
for r in rows[2:]:
    d = {w: r[i] for w, i in idx.items()}
    t = float(d["gpu__time_duration.sum"])
    tu = units[idx["gpu__time_duration.sum"]]
    tus = t / 1000 if tu == "ns" else (t * 1000 if tu == "ms" else t)
    def mb(k):
        v = float(d[k]); u = units[idx[k]]
        return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    name = d["Kernel Name"].split("(")[0]
    extra = " ".join(f"{k.split('.')[0].split('__')[1][:14]}={d[k]}" for k in want[8:] if k in d)
    print(f"{name:32s} blk={d['Block Size']:12s} grid={d['Grid Size']:14s} t={tus:9.1f}us rd={rd:8.1f}MB wr={wr:8.1f}MB "
          f"GB/s={(rd + wr) / tus * 1e3:7.0f} dram%={float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):5.1f} "
          f"regs={d['launch__registers_per_thread']} {extra}")
