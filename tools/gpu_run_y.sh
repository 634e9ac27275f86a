#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/y
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rhs_chunks or torch_device or many_rhs or plan or gl_" > gpurun_out/y/pytest.txt 2>&1
timeout 1200 python tools/c5_rank_subtree.py 0 128 > gpurun_out/y/c5_rank0.json 2> gpurun_out/y/c5_rank0.err
echo done
