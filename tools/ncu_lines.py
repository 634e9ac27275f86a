"""Stall samples per CUDA source line of one kernel (needs -lineinfo + --import-source on)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
items = []
for r in rows:
    if len(r) > 6 and r[0].isdigit() and r[4].isdigit():
        items.append((int(r[4]), int(r[7]) if r[7].isdigit() else 0, int(r[0]), r[1].strip()[:110]))
tot = sum(i[0] for i in items)
print("total stall samples", tot)
for st, ex, ln, src in sorted(items, reverse=True)[:top]:
    print(f"{100 * st / max(tot, 1):5.1f}% {ex:10d}  L{ln:4d}  {src}")
