# L2 eviction hints on the operand loads and TMA L2 promotion: expert GEMM A/B (burst, L2 flushed)
run() { env $1 python tools/gemm_table.py --reps 20 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$2', d['shape'], d['gemm'], round(d['ours_us'], 1), round(d['cublas_us'], 1))"; }
for rep in 1 2; do
run "X=0" base
run "MPM_GEMM_L2HINT=21" hint21
run "MPM_GEMM_L2HINT=12" hint12
run "MPM_GEMM_L2HINT=22" hint22
run "MPM_TMA_PROMO=128" promo128
run "MPM_TMA_PROMO=0" promo0
done > gpurun_out/r2y_l2hints.txt
for rep in 1 2; do
for v in "X=0" "MPM_GEMM_L2HINT=21" "MPM_TMA_PROMO=128"; do
  env $v python bench.py --no-memory-sweep --no-cpu-baseline 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6, 3), round(d['ms_per_step'], 4), round(d['roofline']['gemm_ms_per_step'], 4))"
done; done > gpurun_out/r2y_bench.txt
cat gpurun_out/r2y_bench.txt
