#!/bin/bash
# round-2 GPU pass A: smoke, GPU tests, C4 bench, C4 launch list with DRAM bytes per launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/a_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/a_pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench_c4.json 2> gpurun_out/a_bench_c4.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/a_c4_launches.csv python tools/profile_step.py 4 > gpurun_out/a_c4_ncu.log 2>&1
echo done
