# register-direct 256-bit output stores (incl. the ReLU-mask epilogues): never / auto (K <= 512) / always
run() { env $1 python tools/gemm_table.py --reps 20 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$2', d['shape'], d['gemm'], round(d['ours_us'], 1), round(d['cublas_us'], 1))"; }
for rep in 1 2 3; do
run "MPM_GEMM_DIRECT=0" never
run "X=0" auto
run "MPM_GEMM_DIRECT=1" always
done > gpurun_out/r2z2_direct.txt
for m in 0 1; do MPM_GEMM_DIRECT=$m python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/r2z2_tests_$m.log 2>&1; echo rc=$? >> gpurun_out/r2z2_tests_$m.log; done
python -m pytest tests/test_gpu_layer.py -q -x > gpurun_out/r2z2_tests_layer.log 2>&1; echo rc=$? >> gpurun_out/r2z2_tests_layer.log
for rep in 1 2; do
for v in "MPM_GEMM_DIRECT=0" "X=0" "MPM_GEMM_DIRECT=1"; do
  env $v python bench.py --no-memory-sweep --no-cpu-baseline 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6, 3), round(d['ms_per_step'], 4), round(d['roofline']['gemm_ms_per_step'], 4))"
done; done > gpurun_out/r2z2_bench.txt
tail -1 gpurun_out/r2z2_tests_*.log; cat gpurun_out/r2z2_bench.txt
