#!/bin/bash
# leaf kernel: Z prefetch, in-place natural-order elimination, cp.async epilogue loads; GEMM group 8 DRAM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/n/leaf_trace_c3.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or every_R or config2 or config3_sampled or polynomial or gl_edges" > gpurun_out/n/pytest.txt 2>&1
for G in 1 8; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:zgemm_kernel -c 3 \
  python tools/gemm_one.py 7168x14336x3584x1x1 gemm_group=$G > gpurun_out/n/ncu_one_g$G.txt 2>&1
done
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/n/bench_c3.json 2> gpurun_out/n/bench_c3.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/n/bench_c4.json 2> gpurun_out/n/bench_c4.err
echo done
