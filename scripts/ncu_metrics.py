"""Print the key counters of every kernel in an ncu report (experiment support).

    python scripts/ncu_metrics.py gpurun_out/TAG/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    print("--")
    for w in WANT:
        if w in h:
            print(f"  {w:70s} {v[h.index(w)]}")
    st = []
    for i, x in enumerate(h):
        if "issue_stalled" in x and x.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v[i]), x.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("  stalls:", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
