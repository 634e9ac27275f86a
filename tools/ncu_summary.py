"""Key metrics of every kernel in an `ncu --set full` report (text table)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ik, iid, imn, iv, iu = (hdr.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
want = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block"]
by = {}
for r in rows[1:]:
    if len(r) > iv and r[imn] in want:
        by.setdefault((r[iid], r[ik]), {})[r[imn]] = f"{r[iv]} {r[iu]}".strip()
for (i, k), m in by.items():
    print(f"[{i}] {k[:110]}")
    for w in want:
        if w in m:
            print(f"    {w:36s} {m[w]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_dmma.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
idx = {k: h.index(k) for k in keys if k in h}
units = rr[1] if len(rr) > 1 else []
ik2 = h.index("Kernel Name")
for r in rr[2:]:
    print(f"raw: {r[ik2][:60]}")
    for k, j in idx.items():
        print(f"    {k:70s} {r[j]} {units[j] if j < len(units) else ''}")
