#!/bin/bash
# round-2 final evidence v3 (3M products, grouped 64x64 tile, split-K planner candidates, W^-1 lookahead):
# smoke, full GPU suite, driver-style benches, one-step launch lists with DRAM bytes, ncu --set full of
# the C4 top merge GEMM and the complex leaf kernel; C2 block-step threshold probe
cd "$(dirname "$0")/.."
O=gpurun_out/final3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.txt 2>&1
S=$(date +%s); timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "wall $(( $(date +%s) - S )) s" > $O/bench_c4.wall
timeout 900 python bench.py --config 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
for C in 4 3 2; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/c${C}_launches.csv python tools/profile_step.py $C > $O/c${C}_ncu.log 2>&1
done
IDX=$(python - $O/c4_launches.csv <<'PY'
import csv, io, sys
rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(sys.argv[1]) if l.startswith('"'))))]
h = rows[0]; rows = rows[1:]
ki, ni, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
z = [float(r[vi].replace(",", "")) for r in rows if r[ni] == "gpu__time_duration.sum" and "zgemm_kernel" in r[ki]]
print(max(range(len(z)), key=lambda i: z[i]))
PY
)
echo "top zgemm index $IDX" > $O/idx.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zgemm_kernel \
    -s $IDX -c 1 -o $O/c4_top_zgemm python tools/profile_step.py 4 > $O/ncu_full_zgemm.log 2>&1
ncu -i $O/c4_top_zgemm.ncu-rep --page raw --csv > $O/c4_top_zgemm_raw.csv 2>/dev/null
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zgj_seq_kernel \
    -s 0 -c 1 -o $O/c4_leaf python tools/profile_step.py 4 > $O/ncu_full_leaf.log 2>&1
ncu -i $O/c4_leaf.ncu-rep --page raw --csv > $O/c4_leaf_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
timeout 300 python tools/knob_sweep.py 2 nat_bb_min 512 200 > $O/sweep_c2_bb.txt 2>&1
echo done
