# epilogue cost A/B: the same GEMMs with parts of the epilogue compiled out (probe builds only)
B='from paper_2506_22175_b200 import build; build.build(force=True)'
for v in 0 1 2 3; do
  if [ $v = 0 ]; then MPM_NVCC_FLAGS= python -c "$B"; else MPM_NVCC_FLAGS=-DMPM_EPI_SKIP=$v python -c "$B"; fi > gpurun_out/r2skip_build$v.log 2>&1
  cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_skip$v.so
done
C=fc1_fwd,fc1_fwd_plain,fc2_fwd,fc2_dgrad,fc1_dgrad,fc2_wgrad
for r in 1 2; do for v in 0 1 2 3; do
  echo "== skip$v round$r" >> gpurun_out/r2skip.txt
  MPM_LIB=/tmp/libmpm_skip$v.so python tools/gemm_probe.py 30 $C >> gpurun_out/r2skip.txt 2>&1
done; done
cat gpurun_out/r2skip.txt
