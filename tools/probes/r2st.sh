# configs[4] stack: current tree vs the session-start library on the same box (interleaved)
for i in 1 2; do
  MPM_LIB=_ab/libmpm_base.so timeout 600 python tools/bench_stack.py 2>/dev/null | sed "s/^/base /"
  timeout 600 python tools/bench_stack.py 2>/dev/null | sed "s/^/new /"
done > gpurun_out/r2st_stack_ab.txt
cat gpurun_out/r2st_stack_ab.txt | cut -c1-400
