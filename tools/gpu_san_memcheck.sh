#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1700 compute-sanitizer --tool memcheck --target-processes all --log-file gpurun_out/san_memcheck.log \
  python tools/sanitize_case.py > gpurun_out/san_memcheck_stdout.txt 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck_stdout.txt
