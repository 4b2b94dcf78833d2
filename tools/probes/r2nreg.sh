# expert GEMM register cap 168 (148 used) vs 136 vs 128: GEMMs alone and the step (the gather shares SMs
# with the first weight gradient; fewer GEMM registers leave it more room)
run() { env $1 python tools/gemm_table.py --reps 20 --only cfg2_N1 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$2', d['shape'], d['gemm'], round(d['ours_us'], 1), round(d['cublas_us'], 1))"; }
run "MPM_LIB=_ab/libmpm_head.so" head > gpurun_out/r2nreg_gemm.txt
run "MPM_LIB=_ab/libmpm_nreg128.so" nreg128 >> gpurun_out/r2nreg_gemm.txt
for rep in 1 2 3; do
for v in "MPM_LIB=_ab/libmpm_head.so" "MPM_LIB=_ab/libmpm_nreg136.so" "MPM_LIB=_ab/libmpm_nreg128.so"; do
  env $v python bench.py --no-memory-sweep --no-cpu-baseline 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6, 3), round(d['ms_per_step'], 4), round(d['roofline']['gemm_ms_per_step'], 4))"
done; done > gpurun_out/r2nreg_bench.txt
cat gpurun_out/r2nreg_bench.txt
