#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/d_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rs -s \
  -k "natural or sharded or virtual or zgemm_configs or config4 or config3 or many_rhs or stream" > gpurun_out/d_pytest.txt 2>&1
timeout 600 python tools/gemm_tune16.py > gpurun_out/d_tune16.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/d_bench_c4.json 2> gpurun_out/d_bench_c4.err
timeout 600 python tools/gemm_trace.py 4 > /dev/null 2> gpurun_out/d_trace_c4.txt
echo done
