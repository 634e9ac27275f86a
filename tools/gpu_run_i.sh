#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/i_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "many_rhs or zgemm_configs or config2 or polynomial or torch_device or stream or virtual or every_R" > gpurun_out/i_pytest.txt 2>&1
timeout 600 python tools/gemm_tune16.py > gpurun_out/i_tune16.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/i_bench_c4.json 2> gpurun_out/i_bench_c4.err
timeout 600 python tools/gemm_trace.py 4 > /dev/null 2> gpurun_out/i_trace_c4.txt
echo done
