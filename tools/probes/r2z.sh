# plain bf16 outputs stored straight from registers with 256-bit stores (no smem staging): GEMM A/B
run() { env $1 python tools/gemm_table.py --reps 20 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$2', d['shape'], d['gemm'], round(d['ours_us'], 1), round(d['cublas_us'], 1))"; }
for rep in 1 2 3; do
run "X=0" base
run "MPM_GEMM_DIRECT=1" direct
done > gpurun_out/r2z_direct.txt
python -m pytest tests/test_gpu_kernels.py -q -x -k "tcgen05 or valid" > gpurun_out/r2z_tests.log 2>&1; echo rc=$? >> gpurun_out/r2z_tests.log
MPM_GEMM_DIRECT=1 python -m pytest tests/test_gpu_kernels.py -q -x -k "tcgen05 or valid" >> gpurun_out/r2z_tests.log 2>&1; echo rc=$? >> gpurun_out/r2z_tests.log
tail -4 gpurun_out/r2z_tests.log
