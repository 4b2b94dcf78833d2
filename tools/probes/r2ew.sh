# 4 vs 8 epilogue warps on every expert GEMM (the ncu SASS profile shows the K=1024 fc1 forward's MMA
# issuer waiting on the accumulator-empty barrier: the epilogue paces those tiles)
run() { env $1 python tools/gemm_table.py --reps 20 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$2', d['shape'], d['gemm'], round(d['ours_us'], 1), round(d['cublas_us'], 1))"; }
for rep in 1 2 3; do
run "MPM_GEMM_EW=4" ew4
run "MPM_GEMM_EW=8" ew8
done > gpurun_out/r2ew.txt
cat gpurun_out/r2ew.txt | head -3
