#!/bin/bash
# after 3M: C4 GEMM trace, complex leaf kernel stall lines (3M), C3/C2 bench lines
cd "$(dirname "$0")/.."
O=gpurun_out/ak
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python tools/gemm_trace.py 4 > $O/trace_c4.out 2> $O/trace_c4.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgj_seq_kernel -c 1 -o $O/leaf \
   python tools/leaf_trace_c3.py 32 > $O/ncu_leaf.log 2>&1
python tools/ncu_stalls.py $O/leaf.ncu-rep zgj_seq_kernel 40 > $O/leaf_stalls.txt 2>&1
python tools/ncu_lines.py $O/leaf.ncu-rep zgj_seq_kernel 60 > $O/leaf_lines.txt 2>&1
ncu -i $O/leaf.ncu-rep --page raw --csv > $O/leaf_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
echo done
