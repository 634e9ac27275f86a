mkdir -p gpurun_out/wrap
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/wrap/pytest_gpu.txt
timeout 400 python bench.py > gpurun_out/wrap/bench_c2.json 2> gpurun_out/wrap/bench_c2.err
timeout 600 python bench.py --config 3 > gpurun_out/wrap/bench_c3.json 2> gpurun_out/wrap/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wrap/c2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-plan > gpurun_out/wrap/ncu_launch.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wrap/c2_step_launches.csv python tools/profile_step.py 2 > gpurun_out/wrap/ncu_step.log 2>&1
HPS_PLAN=0 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:dgj_leaf|leaf_real_ops" -c 2 -o gpurun_out/wrap/c2_leaf_real_full python tools/trace_once.py 2 > gpurun_out/wrap/ncu_full.log 2>&1
HPS_LR_TRACE=1 HPS_PLAN=0 timeout 300 python tools/trace_once.py 2 2>&1 | grep leaf_real | tail -2 > gpurun_out/wrap/lr_trace.txt
cat gpurun_out/wrap/pytest_gpu.txt
