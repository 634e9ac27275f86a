#!/bin/bash
# round-2 evidence run (after the leaf and GEMM changes): full GPU suite, benches (C4 headline, C3, C2), launch lists with DRAM bytes,
# one ncu --set full capture each of the top merge GEMM and of the complex leaf kernel at C4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/s
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/s/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/s/bench_c4.json 2> gpurun_out/s/bench_c4.err
timeout 900 python bench.py --config 3 > gpurun_out/s/bench_c3.json 2> gpurun_out/s/bench_c3.err
timeout 600 python bench.py --config 2 --steps 10 > gpurun_out/s/bench_c2.json 2> gpurun_out/s/bench_c2.err
for C in 4 3 2; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/s/c${C}_launches.csv python tools/profile_step.py $C > gpurun_out/s/c${C}_ncu.log 2>&1
done
IDX=$(python - gpurun_out/s/c4_launches.csv <<'PY'
import csv, io, sys
rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(sys.argv[1]) if l.startswith('"'))))]
h = rows[0]; rows = rows[1:]
ki, ni, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
z = [float(r[vi].replace(",", "")) for r in rows if r[ni] == "gpu__time_duration.sum" and "zgemm_kernel" in r[ki]]
print(max(range(len(z)), key=lambda i: z[i]))
PY
)
echo "top zgemm index $IDX" > gpurun_out/s/idx.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zgemm_kernel \
    -s $IDX -c 1 -o gpurun_out/s/c4_top_zgemm python tools/profile_step.py 4 > gpurun_out/s/ncu_full_zgemm.log 2>&1
ncu -i gpurun_out/s/c4_top_zgemm.ncu-rep --page raw --csv > gpurun_out/s/c4_top_zgemm_raw.csv 2>/dev/null
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zgj_seq_kernel \
    -s 0 -c 1 -o gpurun_out/s/c4_leaf python tools/profile_step.py 4 > gpurun_out/s/ncu_full_leaf.log 2>&1
ncu -i gpurun_out/s/c4_leaf.ncu-rep --page raw --csv > gpurun_out/s/c4_leaf_raw.csv 2>/dev/null
ncu -i gpurun_out/s/c4_leaf.ncu-rep --page source --csv > gpurun_out/s/c4_leaf_source.csv 2>/dev/null
rm -f gpurun_out/s/*.ncu-rep
echo done
