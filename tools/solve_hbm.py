"""HBM rates of the solve sweeps from an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` launch list of tools/profile_solve.py: per kernel, launches, serialised time,
DRAM bytes and GB/s, and the fraction of the measured HBM copy bandwidth (MEASURED_PEAKS.json)."""
import collections
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6544.3) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6544.3
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]
ii, ik, im, iv = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(int(r[ii]), {"name": r[ik].split("(")[0].replace("<unnamed>::", "").replace("void ", "")})
    d[r[im]] = float(r[iv].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in L.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot_t = sum(a[1] for a in agg.values())
tot_b = sum(a[2] for a in agg.values())
print(f"HBM peak {peak:.0f} GB/s (MEASURED_PEAKS.json); serialised, cold-cache ncu times")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = a[2] / max(a[1], 1e-9)
    print(f"{a[1] / 1e6:9.3f} ms {a[0]:5d} launches {a[2] / 1e9:8.3f} GB {gbs:8.1f} GB/s ({gbs / peak:5.1%})  {k}")
print(f"total {tot_t / 1e6:.3f} ms, {tot_b / 1e9:.3f} GB, {tot_b / max(tot_t, 1e-9):.1f} GB/s "
      f"({tot_b / max(tot_t, 1e-9) / peak:.1%} of peak), {len(L)} launches")
