#!/bin/bash
# 3M in the complex leaf update: leaf parity, C3 leaf timeline both ways, C4/C3 sweeps, C4 bench
cd "$(dirname "$0")/.."
O=gpurun_out/ai
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "leaf or config3_sampled or every_R or zgemm_3m" > $O/pytest.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 gemm_3m=1 > $O/leaf_trace_3m.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 gemm_3m=0 > $O/leaf_trace_4m.txt 2>&1
timeout 600 python tools/knob_sweep.py 4 gemm_3m 1 0 > $O/sweep_c4.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 gemm_3m 1 0 > $O/sweep_c3.txt 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
echo done
