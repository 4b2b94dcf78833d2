# routing epilogue (tree top-k), per-kernel zero groups, warp dWg reduce, pair dWg: A/B, parity, bench
for i in 1 2; do
  MPM_LIB=_ab/libmpm_base.so python tools/hbm_probe.py 30 2>&1 | grep -E "gate_route|permute|combine_bwd|gate_bwd|gate_gather" | sed "s/^/base /"
  python tools/hbm_probe.py 30 2>&1 | grep -E "gate_route|permute|combine_bwd|gate_bwd|gate_gather" | sed "s/^/new /"
done > gpurun_out/r2w_hbm.txt
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_graph.py -x -q > gpurun_out/r2w_tests.log 2>&1; echo rc=$? >> gpurun_out/r2w_tests.log
for i in 1 2; do
python bench.py --no-memory-sweep --no-cpu-baseline > gpurun_out/r2w_bench_new_$i.json 2> /dev/null
MPM_LIB=_ab/libmpm_base.so python bench.py --no-memory-sweep --no-cpu-baseline > gpurun_out/r2w_bench_base_$i.json 2> /dev/null
done
python tools/kernel_timeline.py --n 1 > gpurun_out/r2w_timeline_n1.txt 2>&1
cat gpurun_out/r2w_hbm.txt; tail -2 gpurun_out/r2w_tests.log
