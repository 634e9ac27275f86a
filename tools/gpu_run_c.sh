#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c_smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rs > gpurun_out/c_pytest.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/c_bench_c4.json 2> gpurun_out/c_bench_c4.err
timeout 600 python tools/gemm_trace.py 4 > /dev/null 2> gpurun_out/c_trace_c4.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/c_c4_launches.csv python tools/profile_step.py 4 > gpurun_out/c_c4_ncu.log 2>&1
echo done
