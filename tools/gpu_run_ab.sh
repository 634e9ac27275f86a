#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or zinv or every_R or config2 or planned or natural" > gpurun_out/ab/pytest.txt 2>&1
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab/bench_c2.json 2> gpurun_out/ab/bench_c2.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab/bench_c3.json 2> gpurun_out/ab/bench_c3.err
echo done
