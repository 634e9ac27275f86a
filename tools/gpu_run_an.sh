#!/bin/bash
# split-K: tests, then the planned benches (the planner picks split-K where it is faster)
cd "$(dirname "$0")/.."
O=gpurun_out/an
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "split_k or plan_ or zgemm_configs or product_forms" > $O/pytest.txt 2>&1
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python tools/gemm_trace.py 3 --plan > $O/trace_c3.out 2> $O/trace_c3.txt
echo done
