# compute lanes gated on the chunk GEMM size: layer/graph tests, configs[3] step, memory sweep, default bench
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_graph.py -q -x > gpurun_out/r2lanes_tests.log 2>&1; tail -2 gpurun_out/r2lanes_tests.log
for r in 1 2; do timeout 300 python tools/cfg4_probe.py --n 8 >> gpurun_out/r2lanes_cfg4.jsonl 2>> gpurun_out/r2lanes.err; done
timeout 1400 python tools/sweep.py memory --out gpurun_out/r2lanes_cfg4_memory_sweep.json > gpurun_out/r2lanes_mem.log 2>&1
timeout 600 python bench.py > gpurun_out/r2lanes_bench.json 2>> gpurun_out/r2lanes.err
cut -c1-300 gpurun_out/r2lanes_cfg4.jsonl; cut -c1-200 gpurun_out/r2lanes_mem.log | tail -6; tail -1 gpurun_out/r2lanes_bench.json | cut -c1-200
