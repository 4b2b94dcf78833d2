# combine_bwd_gate BN=192 gate tile, pair dWg, warp dWg reduce, grouped zero rows: kernel A/B (isolated) and parity
for i in 1 2; do
  MPM_LIB=_ab/libmpm_base.so python tools/hbm_probe.py 50 > gpurun_out/r2s_hbm_base_$i.txt 2>&1
  python tools/hbm_probe.py 50 > gpurun_out/r2s_hbm_new_$i.txt 2>&1
done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_graph.py -x -q > gpurun_out/r2s_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_tests.log
tail -2 gpurun_out/r2s_tests.log
