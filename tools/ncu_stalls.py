"""Stall reasons per CUDA source line of one kernel (ncu --set full --import-source on, -lineinfo)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
reasons = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {}
items = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[0].isdigit():
        continue
    vals = {hdr[j][6:]: int(r[j] or 0) for j in reasons if (r[j] or "0").isdigit()}
    s = sum(vals.values())
    if s == 0:
        continue
    for k, v in vals.items():
        tot[k] = tot.get(k, 0) + v
    items.append((s, int(r[0]), r[1].strip()[:80], vals))
T = sum(tot.values())
print("stall totals:", ", ".join(f"{k} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
for s, ln, src, vals in sorted(items, reverse=True)[:top]:
    top3 = ", ".join(f"{k} {v}" for k, v in sorted(vals.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100 * s / T:5.1f}% L{ln:4d} {src:80s} | {top3}")
