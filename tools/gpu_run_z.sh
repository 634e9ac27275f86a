#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/z
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/z/leaf_trace.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or every_R or config3_sampled" > gpurun_out/z/pytest.txt 2>&1
timeout 1200 python tools/c5_rank_subtree.py 0 128 > gpurun_out/z/c5_rank0.json 2> gpurun_out/z/c5_rank0.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/z/ref_c4.json 2> gpurun_out/z/ref_c4.err
echo done
