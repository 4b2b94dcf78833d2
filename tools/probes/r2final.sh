# round-2 validation of the current tree: full GPU suite, smoke, default bench, bench launch list
python -m pytest tests -m gpu -q > gpurun_out/r2fin7_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2fin7_pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/r2fin7_smoke.log 2>&1
python bench.py > gpurun_out/r2fin7_bench.json 2> gpurun_out/r2fin7_bench.err
MPM_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2fin7_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-memory-sweep --no-cpu-baseline > gpurun_out/r2fin7_bench_ncu.log 2>&1
python tools/ep_shape_probe.py > gpurun_out/r2fin7_n8_shape_chunking.jsonl 2> gpurun_out/r2fin7_n8.err
tail -2 gpurun_out/r2fin7_pytest_gpu.log
