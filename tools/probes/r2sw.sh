# refresh BASELINE configs[2] (granularity sweep, Algorithm 1 on real timings) and configs[4] (12-layer stack)
timeout 1500 python tools/sweep.py granularity --out gpurun_out/r2sw_cfg3_granularity_sweep.json > gpurun_out/r2sw_cfg3.log 2>&1
timeout 600 python tools/bench_stack.py > gpurun_out/r2sw_stack.json 2> gpurun_out/r2sw_stack.err
tail -3 gpurun_out/r2sw_cfg3.log; cat gpurun_out/r2sw_stack.json
