#!/bin/bash
# Launch list of one planned build + solve of config $1, then one `ncu --set full` capture of
# that step's longest zgemm launch (dram bytes for the roofline's traffic key).
set -e
CFG=${1:-3}
OUT=gpurun_out/cap$CFG
mkdir -p $OUT
python tools/profile_step.py $CFG > $OUT/plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/profile_step.py $CFG > $OUT/ncu_list.log 2>&1
IDX=$(python - $OUT/launches.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
ki, ni, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
z = [float(r[vi].replace(",", "")) for r in rows if r[ni] == "gpu__time_duration.sum" and r[ki].startswith("void <unnamed>::zgemm_kernel")]
print(max(range(len(z)), key=lambda i: z[i]))
PY
)
echo "longest zgemm launch index $IDX" > $OUT/idx.txt
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zgemm_kernel \
    -s $IDX -c 1 -o $OUT/top_zgemm python tools/profile_step.py $CFG > $OUT/ncu_full.log 2>&1
ncu -i $OUT/top_zgemm.ncu-rep --page raw --csv > $OUT/top_zgemm_raw.csv
