# 64-column TMEM loads in the wide epilogue: GEMM A/B against the previous build, parity, bench A/B
run() { env $1 python tools/gemm_table.py --reps 20 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$2', d['shape'], d['gemm'], round(d['ours_us'], 1), round(d['cublas_us'], 1))"; }
for rep in 1 2; do
run "MPM_LIB=_ab/libmpm_head.so" head
run "X=0" new
done > gpurun_out/r2l64.txt
python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/r2l64_tests.log 2>&1; echo rc=$? >> gpurun_out/r2l64_tests.log
for rep in 1 2; do
for v in "MPM_LIB=_ab/libmpm_head.so" "X=0"; do
  env $v python bench.py --no-memory-sweep --no-cpu-baseline 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6, 3), round(d['ms_per_step'], 4), round(d['roofline']['gemm_ms_per_step'], 4))"
done; done > gpurun_out/r2l64_bench.txt
tail -2 gpurun_out/r2l64_tests.log; cat gpurun_out/r2l64_bench.txt
