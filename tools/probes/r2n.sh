set -x
python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r2n_kernels.log 2>&1; echo rc=$? >> gpurun_out/r2n_kernels.log
python tools/gemm_table.py --only cfg2_N1 --gemm fc2_wgrad,fc1_wgrad --sustained > gpurun_out/r2n_wgrad_ares.jsonl 2>&1
MPM_GEMM_ARES=0 python tools/gemm_table.py --only cfg2_N1 --gemm fc2_wgrad,fc1_wgrad --sustained > gpurun_out/r2n_wgrad_noares.jsonl 2>&1
python bench.py --no-memory-sweep --no-cpu-baseline > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
MPM_GEMM_ARES=0 python bench.py --no-memory-sweep --no-cpu-baseline > gpurun_out/r2n_bench_noares.json 2> gpurun_out/r2n_bench_noares.err
timeout 600 ncu --set full --clock-control none -k regex:"nvjet|gemm|umma" -o gpurun_out/r2n_cublas_vs_ours python tools/cublas_ncu_probe.py --only cfg2_N1 > gpurun_out/r2n_ncu.log 2>&1
tail -2 gpurun_out/r2n_kernels.log
