#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/w
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/w/leaf_trace_u32.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 leaf_upd32=0 > gpurun_out/w/leaf_trace_u16.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or zinv or config2 or every_R or plan or natural" > gpurun_out/w/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 leaf_upd32 1 0 > gpurun_out/w/sweep_c3.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 leaf_upd32 1 0 > gpurun_out/w/sweep_c4.txt 2>&1
echo done
