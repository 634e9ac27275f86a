#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/e_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rs -s \
  -k "natural or leaf_schur or config3_sampled or config4 or sharded or many_rhs or zgemm_configs or leaf_parity" > gpurun_out/e_pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 4 nat_bb_min 1024 448 224 > gpurun_out/e_sweep_c4.txt 2>&1
timeout 300 python tools/knob_sweep.py 2 nat_bb_min 1024 224 > gpurun_out/e_sweep_c2.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --config 3 > gpurun_out/e_bench_c3.json 2> gpurun_out/e_bench_c3.err
echo done
