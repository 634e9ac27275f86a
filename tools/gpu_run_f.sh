#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "zgemm_configs or natural or config2 or every_R" > gpurun_out/f_pytest.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/f_c4_launches.csv python tools/profile_step.py 4 > gpurun_out/f_c4_ncu.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config 2 > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.err
echo done
