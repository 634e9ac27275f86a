"""Per-opcode instruction counts and stall samples of one kernel in an ncu report."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}",
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
isrc, iex, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
op, sm, lines = collections.Counter(), collections.Counter(), []
for r in rows[hi + 1:]:
    if len(r) <= iex or not r[iex].isdigit():
        continue
    ex, st, s = int(r[iex]), int(r[ist] or 0), r[isrc].strip()
    toks = s.split()
    o = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
    op[o.split(".")[0]] += ex
    sm[o.split(".")[0]] += st
    lines.append((st, ex, s))
print("total executed", sum(op.values()), " stall samples", sum(sm.values()))
for k, v in op.most_common(22):
    print(f"{k:12s} {v:12d}  stall={sm[k]}")
if len(sys.argv) > 3:
    for st, ex, s in sorted(lines, reverse=True)[: int(sys.argv[3])]:
        print(f"{st:7d} {ex:10d}  {s}")
