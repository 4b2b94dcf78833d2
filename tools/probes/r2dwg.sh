# dWg split reduce: coalesced block-per-128-columns form vs the warp-per-4-columns form (old lib)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x -k "gate or dwg or layer" > gpurun_out/r2dwg_tests.log 2>&1; tail -2 gpurun_out/r2dwg_tests.log
for r in 1 2 3; do
  echo "== old $r" >> gpurun_out/r2dwg.txt; MPM_LIB=$PWD/gpurun_ab_old_libmpm.so  # (the previous build, copied in before the call) timeout 300 python tools/hbm_probe.py 50 2>&1 | grep -E "gate_bwd_gemms|combine_bwd_gate" >> gpurun_out/r2dwg.txt
  echo "== new $r" >> gpurun_out/r2dwg.txt; timeout 300 python tools/hbm_probe.py 50 2>&1 | grep -E "gate_bwd_gemms|combine_bwd_gate" >> gpurun_out/r2dwg.txt
done
cat gpurun_out/r2dwg.txt
