#!/bin/bash
# round-2 closing run: integer-slice feasibility probe; ncu launch list of the bench command itself
# (C4, the default workload) after the same command has exited 0 without ncu
cd "$(dirname "$0")/.."
O=gpurun_out/aw
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python tools/ozaki_probe.py > $O/ozaki_probe.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_s2w1.json 2> $O/bench_s2w1.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file $O/bench_s2w1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_s2w1_ncu.log 2>&1
python - $O/bench_s2w1_launches.csv > $O/bench_s2w1_launch_kernels.txt <<'PY'
import csv, io, sys, collections
rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(sys.argv[1]) if l.startswith('"'))))]
h = rows[0]; rows = rows[1:]
ki, ni, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
acc = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r[ni] != "gpu__time_duration.sum": continue
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[ui], 1e-6)
    k = r[ki].split("(")[0]
    acc[k][0] += 1; acc[k][1] += v
tot = sum(v[1] for v in acc.values())
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 1 --no-cpu-baseline (C4; planner, warm-up, timed, probe and e2e steps all listed)")
print(f"# {sum(v[0] for v in acc.values())} launches, {tot:.1f} ms serialised")
for k, (n, ms) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{ms:12.3f} ms {100 * ms / tot:6.2f}% {n:7d} launches  {k}")
PY
rm -f $O/bench_s2w1_launches.csv.tmp
echo done
