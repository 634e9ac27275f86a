#!/bin/bash
# round-2 final evidence (after the 3M products and R^1 off at C4/C5): smoke, full GPU suite, driver-style benches (C4 headline with the driver's
# arguments, C3, C2), the reference arm, one-step launch lists with DRAM bytes (C4, C3, C2), ncu --set
# full captures of the C4 top merge GEMM and the complex leaf kernel, the C5 per-rank subtree
cd "$(dirname "$0")/.."
O=gpurun_out/final2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.txt 2>&1
S=$(date +%s); timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "wall $(( $(date +%s) - S )) s" > $O/bench_c4.wall
timeout 900 python bench.py --config 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_c4.json 2> $O/ref_c4.err
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
for C in 4 2; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/c${C}_solve_launches.csv python tools/profile_solve.py $C > $O/c${C}_solve.log 2>&1
done
timeout 1200 python tools/c5_rank_subtree.py 0 128 > $O/c5_rank0.json 2> $O/c5_rank0.err
timeout 300 python tools/leaf_trace_c3.py 32 > $O/leaf_trace_c3.txt 2>&1
echo done
