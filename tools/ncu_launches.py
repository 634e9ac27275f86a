"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel totals."""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ii, iname, igrid, ival = (hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Value"))
    return [(int(r[ii]), r[iname], r[igrid], float(r[ival].replace(",", ""))) for r in rows[1:]]


def summary(data):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, nm, grid, v in data:
        key = nm.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}% {v[0]:5d} launches  {k}")
    out.append(f"{tot / 1e6:9.3f} ms total, {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    data = load(sys.argv[1])
    if len(sys.argv) > 2 and sys.argv[2] == "half":   # second of two identical repetitions
        data = data[len(data) // 2:]
    print(summary(data))
    if len(sys.argv) > 3:
        for i, nm, grid, v in data:
            if sys.argv[3] in nm:
                print(f"{v/1e3:10.1f} us  {grid}  {nm[:90]}")
