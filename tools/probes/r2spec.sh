# A/B: epilogue-specialised expert GEMM kernels (compile-time epilogue) vs the generic runtime epilogue
B='from paper_2506_22175_b200 import build; build.build(force=True)'
MPM_NVCC_FLAGS=-DMPM_EPI_SPEC=0 python -c "$B" > gpurun_out/r2spec_build0.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_old.so
MPM_NVCC_FLAGS= python -c "$B" > gpurun_out/r2spec_build1.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_new.so
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > gpurun_out/r2spec_tests.log 2>&1; tail -2 gpurun_out/r2spec_tests.log
rm -f gpurun_out/r2spec.txt
for r in 1 2 3; do for v in old new; do
  echo "== $v round$r" >> gpurun_out/r2spec.txt
  MPM_LIB=/tmp/libmpm_$v.so timeout 300 python tools/gemm_table.py --sustained --only cfg2_N1 >> gpurun_out/r2spec.txt 2>&1
  MPM_LIB=/tmp/libmpm_$v.so timeout 300 python bench.py --no-memory-sweep --no-cpu-baseline --pipeline-n 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['gemm_ms_per_step'])" >> gpurun_out/r2spec.txt 2>&1
done; done
python - <<'P'
import json
for l in open('gpurun_out/r2spec.txt'):
    if l.startswith('{'):
        d=json.loads(l); print(d['gemm'], round(d['ours_us'],1), round(d['ours_sustained_us'],1))
    else: print(l.strip())
P
