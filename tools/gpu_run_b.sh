#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rs -s \
  -k "virtual or sharded or stream or nccl or cache or config3_sampled or gl_boundary or natural or forced or schur" \
  > gpurun_out/b_pytest.txt 2>&1
timeout 900 python tools/poly_errors.py > gpurun_out/b_poly.txt 2>&1
echo done
