# epilogue cost A/B, part 2: isolated (L2-flushed) and sustained (with SM clock) per-GEMM times for the
# full epilogue (skip0) and no epilogue (skip3), to separate power/clock from on-chip contention
B='from paper_2506_22175_b200 import build; build.build(force=True)'
for v in 0 3; do
  if [ $v = 0 ]; then MPM_NVCC_FLAGS= python -c "$B"; else MPM_NVCC_FLAGS=-DMPM_EPI_SKIP=$v python -c "$B"; fi > gpurun_out/r2skip_build$v.log 2>&1
  cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_skip$v.so
done
for r in 1 2; do for v in 0 3; do
  echo "== skip$v round$r" >> gpurun_out/r2skip2.txt
  MPM_LIB=/tmp/libmpm_skip$v.so python tools/gemm_table.py --sustained --only cfg2_N1 >> gpurun_out/r2skip2.txt 2>&1
done; done
cat gpurun_out/r2skip2.txt
