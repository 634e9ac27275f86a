#!/bin/bash
# after retiring nat_b32 / nat_persist / gemm_3m=2: affected tests; host enqueue vs device time (C2, C3)
cd "$(dirname "$0")/.."
O=gpurun_out/at
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "natural or zgemm or product_forms or config2" > $O/pytest_sel.txt 2>&1
timeout 300 python tools/host_probe.py 2 1 > $O/host_c2.txt 2>&1
timeout 300 python tools/host_probe.py 2 16 > $O/host_c2_16.txt 2>&1
timeout 600 python tools/host_probe.py 3 > $O/host_c3.txt 2>&1
echo done
