# routing in the gate GEMM's epilogue, warp dWg reduce, pair dWg, grouped zero rows: A/B, parity, bench
for i in 1 2; do
  MPM_LIB=_ab/libmpm_base.so python tools/hbm_probe.py 50 > gpurun_out/r2t_hbm_base_$i.txt 2>&1
  python tools/hbm_probe.py 50 > gpurun_out/r2t_hbm_new_$i.txt 2>&1
done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_graph.py -x -q > gpurun_out/r2t_tests.log 2>&1; echo rc=$? >> gpurun_out/r2t_tests.log
python bench.py --no-memory-sweep --no-cpu-baseline > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
MPM_LIB=_ab/libmpm_base.so python bench.py --no-memory-sweep --no-cpu-baseline > gpurun_out/r2t_bench_base.json 2> gpurun_out/r2t_bench_base.err
python tools/kernel_timeline.py --n 1 > gpurun_out/r2t_timeline_n1.txt 2>&1
tail -2 gpurun_out/r2t_tests.log
