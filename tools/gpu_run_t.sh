#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/t/leaf_trace.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or plan_solve or config2 or every_R or many_rhs" > gpurun_out/t/pytest.txt 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/t/bench_c4.json 2> gpurun_out/t/bench_c4.err
echo done
