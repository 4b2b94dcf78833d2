# routing epilogue with tree selection: A/B against the two-kernel route, then parity
for i in 1 2; do
  MPM_LIB=_ab/libmpm_base.so python tools/hbm_probe.py 30 2>&1 | grep -E "gate_route|permute|combine_bwd_gate|gate_bwd" | sed "s/^/base /"
  python tools/hbm_probe.py 30 2>&1 | grep -E "gate_route|permute|combine_bwd_gate|gate_bwd" | sed "s/^/new /"
done > gpurun_out/r2v_hbm.txt
python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r2v_tests.log 2>&1; echo rc=$? >> gpurun_out/r2v_tests.log
cat gpurun_out/r2v_hbm.txt; tail -3 gpurun_out/r2v_tests.log
